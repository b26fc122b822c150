"""Host-side (numpy) builders for test matrices: the benchmark stencils at small
sizes and ragged / power-law CSR structures with the edge cases the reference
tests exercise (empty rows, long rows, unsorted-free sorted columns)."""
from __future__ import annotations

import numpy as np


def stencil_csr(points: int, n: int):
    """5-point 2-D (diag 4) or 27-point 3-D (diag 26) stencil, natural order,
    ascending columns, off-diagonals -1; int64 rowptr, int32 colind, f64 values."""
    if points == 5:
        ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        ii, jj = ii.ravel(), jj.ravel()
        rows = ii * n + jj
        offs = [(-1, 0), (0, -1), (0, 0), (0, 1), (1, 0)]
        cols, keep, diag = [], [], []
        for di, dj in offs:
            ok = (ii + di >= 0) & (ii + di < n) & (jj + dj >= 0) & (jj + dj < n)
            cols.append((ii + di) * n + (jj + dj))
            keep.append(ok)
            diag.append(np.full(rows.shape, di == 0 and dj == 0))
    else:
        g = np.arange(n)
        ii, jj, kk = np.meshgrid(g, g, g, indexing="ij")
        ii, jj, kk = ii.ravel(), jj.ravel(), kk.ravel()
        rows = (ii * n + jj) * n + kk
        cols, keep, diag = [], [], []
        for di in (-1, 0, 1):
            for dj in (-1, 0, 1):
                for dk in (-1, 0, 1):
                    ok = ((ii + di >= 0) & (ii + di < n) & (jj + dj >= 0) & (jj + dj < n)
                          & (kk + dk >= 0) & (kk + dk < n))
                    cols.append(((ii + di) * n + (jj + dj)) * n + (kk + dk))
                    keep.append(ok)
                    diag.append(np.full(rows.shape, di == 0 and dj == 0 and dk == 0))
    C = np.stack(cols, 1)
    K = np.stack(keep, 1)
    D = np.stack(diag, 1)
    counts = K.sum(1)
    rowptr = np.zeros(rows.size + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum(counts)
    colind = C[K].astype(np.int32)
    values = np.where(D[K], 4.0 if points == 5 else 26.0, -1.0)
    return rowptr, colind, values


def ragged_csr(rng: np.random.Generator, nrows: int, ncols: int, *, max_len: int = 40,
               long_rows: dict | None = None, empty_every: int = 0, dtype=np.float64):
    """Random CSR with row lengths U[0, max_len), optional forced long rows
    {row: length} and forced empty rows; sorted unique columns per row."""
    counts = rng.integers(0, max_len, nrows)
    if empty_every:
        counts[::empty_every] = 0
    for r, L in (long_rows or {}).items():
        counts[r] = min(L, ncols)
    rowptr = np.zeros(nrows + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum(counts)
    parts = []
    for c in counts:
        if c == 0:
            continue
        if c * 4 > ncols:
            parts.append(np.sort(rng.choice(ncols, size=int(c), replace=False)))
        else:
            sel = np.unique(rng.integers(0, ncols, int(c) * 2))[: int(c)]
            while sel.size < c:
                sel = np.unique(np.concatenate([sel, rng.integers(0, ncols, int(c))]))[: int(c)]
            parts.append(np.sort(sel))
    colind = (np.concatenate(parts) if parts else np.zeros(0)).astype(np.int32)
    if np.issubdtype(dtype, np.integer):
        values = rng.integers(-50, 50, rowptr[-1]).astype(dtype)
    else:
        values = rng.uniform(-1.0, 1.0, rowptr[-1]).astype(dtype)
    return rowptr, colind, values


def powerlaw_csr(rng: np.random.Generator, nrows: int, mean: float = 10.0, alpha: float = 2.5,
                 max_len: int | None = None):
    """Chung-Lu style power-law CSR (SURVEY A.8 in miniature): Pareto(alpha)
    weights, columns drawn in proportion to the same weights, hubs permuted,
    per-row sorted and deduplicated."""
    w = (1.0 - rng.random(nrows)) ** (-1.0 / (alpha - 1.0))
    w = w / w.sum()
    total = int(mean * nrows)
    cdf = np.cumsum(w)
    r = np.minimum(np.searchsorted(cdf, rng.random(total) * cdf[-1]), nrows - 1)
    perm = rng.permutation(nrows)
    c = perm[np.minimum(np.searchsorted(cdf, rng.random(total) * cdf[-1]), nrows - 1)]
    r = perm[r]
    key = np.unique(r.astype(np.int64) * nrows + c)
    rows, cols = key // nrows, key % nrows
    counts = np.bincount(rows, minlength=nrows)
    rowptr = np.zeros(nrows + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum(counts)
    values = rng.uniform(-1.0, 1.0, rowptr[-1])
    return rowptr, cols.astype(np.int32), values
