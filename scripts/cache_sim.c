/* cache_sim.c — DRAM traffic of the X-row gathers of a CSR x dense SpMM for a
 * cache of `cap` X rows (scripts/c3_gather_bound.py):
 *   opt  : Belady's optimal replacement on the access sequence (the minimum any
 *          cache of that size can reach for this order of the gathers)
 *   lru  : least-recently-used on the same sequence
 *   pin  : the `cap` most referenced rows pinned, every other access a miss
 * Accesses are the colind stream in CSR order (rows ascending, each row's
 * columns ascending) — the order the SpMM kernels consume them in.
 * Build: gcc -O2 -o cache_sim cache_sim.c ; run: cache_sim colind.bin ncols cap...
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

typedef struct { int64_t key; int32_t col; } HeapItem;  /* max-heap on next use */

static void heap_push(HeapItem* h, int64_t* n, HeapItem it) {
  int64_t i = (*n)++;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (h[p].key >= it.key) break;
    h[i] = h[p];
    i = p;
  }
  h[i] = it;
}
static HeapItem heap_pop(HeapItem* h, int64_t* n) {
  HeapItem top = h[0], last = h[--(*n)];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    int64_t mk = last.key;
    if (l < *n && h[l].key > mk) { m = l; mk = h[l].key; }
    if (r < *n && h[r].key > mk) { m = r; }
    if (m == i) break;
    h[i] = h[m];
    i = m;
  }
  if (*n > 0) h[i] = last;
  return top;
}

int main(int argc, char** argv) {
  if (argc < 4) { fprintf(stderr, "usage: %s colind.bin ncols cap [cap...]\n", argv[0]); return 2; }
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 1;
  fseek(f, 0, SEEK_END);
  const int64_t n = ftell(f) / 4;
  fseek(f, 0, SEEK_SET);
  int32_t* a = malloc(n * 4);
  if (fread(a, 4, n, f) != (size_t)n) return 1;
  fclose(f);
  const int64_t ncols = atoll(argv[2]);
  /* next use of each access (Belady), frequencies (pin) */
  int64_t* nxt = malloc(n * 8);
  int64_t* last = malloc(ncols * 8);
  int64_t* cnt = calloc(ncols, 8);
  for (int64_t c = 0; c < ncols; ++c) last[c] = INT64_MAX;
  for (int64_t i = n - 1; i >= 0; --i) { nxt[i] = last[a[i]]; last[a[i]] = i; cnt[a[i]]++; }
  int64_t distinct = 0;
  for (int64_t c = 0; c < ncols; ++c) distinct += cnt[c] > 0;
  printf("{\"accesses\": %lld, \"distinct\": %lld, \"results\": [", (long long)n, (long long)distinct);
  for (int ai = 3; ai < argc; ++ai) {
    const int64_t cap = atoll(argv[ai]);
    /* ---- OPT */
    int64_t miss_opt = 0, hn = 0, incache = 0;
    HeapItem* heap = malloc((n + 1) * sizeof(HeapItem));
    int64_t* cur = malloc(ncols * 8);  /* current next-use key of a cached column, -1 absent */
    for (int64_t c = 0; c < ncols; ++c) cur[c] = -1;
    for (int64_t i = 0; i < n; ++i) {
      const int32_t c = a[i];
      if (cur[c] >= 0) {                 /* hit: re-key lazily */
        cur[c] = nxt[i];
        heap_push(heap, &hn, (HeapItem){nxt[i], c});
        continue;
      }
      ++miss_opt;
      if (incache == cap) {              /* evict the farthest next use (skip stale) */
        for (;;) {
          HeapItem t = heap_pop(heap, &hn);
          if (cur[t.col] == t.key) { cur[t.col] = -1; --incache; break; }
        }
      }
      cur[c] = nxt[i];
      ++incache;
      heap_push(heap, &hn, (HeapItem){nxt[i], c});
      if (hn > 4 * cap + 1024) {         /* compact stale heap entries */
        int64_t m = 0;
        for (int64_t q = 0; q < hn; ++q)
          if (cur[heap[q].col] == heap[q].key) heap[m++] = heap[q];
        int64_t hh = 0;
        for (int64_t q = 0; q < m; ++q) heap_push(heap, &hh, heap[q]);
        hn = hh;
      }
    }
    free(heap);
    /* ---- LRU: doubly linked list over columns */
    int32_t* prv = malloc(ncols * 4);
    int32_t* nx2 = malloc(ncols * 4);
    char* in = calloc(ncols, 1);
    int32_t head = -1, tail = -1;
    int64_t size = 0, miss_lru = 0;
    for (int64_t i = 0; i < n; ++i) {
      const int32_t c = a[i];
      if (in[c]) {
        if (head == c) continue;
        /* unlink */
        nx2[prv[c]] = nx2[c];
        if (nx2[c] >= 0) prv[nx2[c]] = prv[c]; else tail = prv[c];
      } else {
        ++miss_lru;
        if (size == cap) {
          const int32_t v = tail;
          tail = prv[v];
          if (tail >= 0) nx2[tail] = -1; else head = -1;
          in[v] = 0;
          --size;
        }
        in[c] = 1;
        ++size;
      }
      prv[c] = -1;
      nx2[c] = head;
      if (head >= 0) prv[head] = c;
      head = c;
      if (tail < 0) tail = c;
    }
    free(prv); free(nx2); free(in);
    /* ---- pin the cap most frequent */
    int64_t* hist = NULL;
    int64_t maxc = 0;
    for (int64_t c = 0; c < ncols; ++c) maxc = cnt[c] > maxc ? cnt[c] : maxc;
    hist = calloc(maxc + 1, 8);
    for (int64_t c = 0; c < ncols; ++c) hist[cnt[c]]++;
    int64_t left = cap, covered = 0, pinned = 0;
    for (int64_t v = maxc; v >= 1 && left > 0; --v) {
      const int64_t take = hist[v] < left ? hist[v] : left;
      covered += take * v;
      pinned += take;
      left -= take;
    }
    const int64_t miss_pin = (n - covered) + pinned;
    /* ---- LRU with reuse hints: an access whose next use is more than D
     * accesses away is (re)placed at the LRU end (an L2 evict_first load),
     * others at the MRU end; D = hint_dist * cap (HINT_D env, default 4) */
    const double hint_mult = getenv("HINT_D") ? atof(getenv("HINT_D")) : 4.0;
    const int64_t D = (int64_t)(hint_mult * (double)cap);
    int64_t miss_hint = 0;
    {
      int32_t* pv = malloc(ncols * 4);
      int32_t* nv = malloc(ncols * 4);
      char* inn = calloc(ncols, 1);
      int32_t hd = -1, tl = -1;
      int64_t sz = 0;
      for (int64_t i = 0; i < n; ++i) {
        const int32_t c = a[i];
        const int near = nxt[i] != INT64_MAX && nxt[i] - i <= D;
        if (inn[c]) {
          /* unlink c */
          if (pv[c] >= 0) nv[pv[c]] = nv[c]; else hd = nv[c];
          if (nv[c] >= 0) pv[nv[c]] = pv[c]; else tl = pv[c];
        } else {
          ++miss_hint;
          if (sz == cap) {
            const int32_t v = tl;
            tl = pv[v];
            if (tl >= 0) nv[tl] = -1; else hd = -1;
            inn[v] = 0;
            --sz;
          }
          inn[c] = 1;
          ++sz;
        }
        if (near || hd < 0) {  /* MRU end */
          pv[c] = -1; nv[c] = hd;
          if (hd >= 0) pv[hd] = c;
          hd = c;
          if (tl < 0) tl = c;
        } else {               /* LRU end */
          nv[c] = -1; pv[c] = tl;
          nv[tl] = c;
          tl = c;
        }
      }
      free(pv); free(nv); free(inn);
    }
    free(hist);
    free(cur);
    printf("%s{\"cap_rows\": %lld, \"miss_opt\": %lld, \"miss_lru\": %lld, \"miss_pin\": %lld, "
           "\"miss_hint\": %lld, \"hint_d\": %lld}",
           ai > 3 ? ", " : "", (long long)cap, (long long)miss_opt, (long long)miss_lru,
           (long long)miss_pin, (long long)miss_hint, (long long)D);
    fflush(stdout);
  }
  printf("]}\n");
  return 0;
}
