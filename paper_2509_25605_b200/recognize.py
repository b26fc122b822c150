"""Hot-nest recognition: lowered LAPIS loop nests -> hand-written sm_100a kernels.

The reference pipeline turns sparse.spmv_csr, linalg.matmul / matvec /
batch_matmul, linalg.reduce and the SpMM / GCN loop nests into the Kokkos
nests of its golden IR (tests/golden/ir/*.mlir).  The
executor (runtime.py) offers every device nest to ``match`` first: a nest whose
dataflow is one of those kernels is run by the tuned kernel behind the C ABI
(include/lapis_b200.h) instead of a generated one.  Matching is structural:
each value the nest stores is rewritten into an expression tree over the
nest's index roles, constants, free scalars and loads from free memrefs, and
compared with the kernel's template (commutative ops in either order, widening
index casts transparent).  Anything that does not match exactly — other
inits, other combiners, extents the kernel would overrun — falls through to
the generated kernel, which reports the interpreter's errors.

Counters are the interpreter's (interp.py:597-602, 918-928): a recognised
nest adds the closed-form execution counts of its single / store / barrier
ops.  Library ops (kokkos.gemm / gemv, linalg.*, sparse.spmv_csr) count
nothing, as in the interpreter (their stores bypass _h_store).
"""
from __future__ import annotations

import ctypes as C
import struct

import torch

from . import _capi
from ._capi import check

_DT = {"f32": _capi.F32, "f64": _capi.F64, "i32": _capi.I32, "i64": _capi.I64,
       "index": _capi.I64}
_IDX_BYTES = {"i32": 4, "i64": 8, "index": 8}
_COMB = {"add": _capi.ADD, "mul": _capi.MUL, "min": _capi.MIN, "max": _capi.MAX}
_COMMUTATIVE = {"arith.addi", "arith.muli", "arith.addf", "arith.mulf"}


# ------------------------------------------------------------ expression trees
class Nest:
    """Index of one nest: which ops are inside, and the role of each index."""

    def __init__(self, top):
        from lapis.ir import walk
        self.top = top
        self.inside = set(id(o) for o in walk(top))
        self.roles: dict = {}

    def tree(self, v):
        if v in self.roles:
            return ("role", self.roles[v])
        op = v.defining_op()
        if op is not None and op.name == "arith.constant":   # wherever it is defined
            return ("const", v.type.kind, op.attrs["value"])
        if op is None or id(op) not in self.inside or op is self.top:
            return ("free", v)
        name = op.name
        if name == "memref.load":
            return ("load", self.tree(op.operands[0])) + tuple(self.tree(i) for i in op.operands[1:])
        if name == "arith.index_cast":
            src, dst = op.operands[0].type.kind, v.type.kind
            if _width(dst) >= _width(src):
                return self.tree(op.operands[0])
        args = tuple(self.tree(o) for o in op.operands)
        if name in _COMMUTATIVE:
            args = tuple(sorted(args, key=_key))
        return (name,) + args


def _outer(nest: "Nest", env, v):
    """Runtime value of a scalar the nest reads: host-computed values from the
    environment, constants wherever they are defined; None otherwise."""
    t = nest.tree(v)
    if t[0] == "const":
        return int(t[2]) if t[1] not in ("f32", "f64") else float(t[2])
    if t[0] == "free":
        return env[v]
    return None


def _width(kind: str) -> int:
    return {"i1": 1, "i32": 32, "i64": 64, "index": 64}.get(kind, 0)


def _is_zero(t, kind_ok=None) -> bool:
    if not (isinstance(t, tuple) and t and t[0] == "const"):
        return False
    kind, v = t[1], t[2]
    if kind_ok is not None and kind not in kind_ok:
        return False
    if kind in ("f32", "f64", "f16"):
        return struct.pack("<d", float(v)) == struct.pack("<d", 0.0)
    return int(v) == 0


def _const_int(t):
    if isinstance(t, tuple) and t[0] == "const" and t[1] in ("i32", "i64", "index"):
        return int(t[2])
    return None


def _free(t):
    return t[1] if isinstance(t, tuple) and t[0] == "free" else None


def _key(t) -> str:
    """Deterministic sort key of a tree (free values by identity)."""
    if isinstance(t, tuple):
        if t and t[0] == "free":
            return f"free#{id(t[1])}"
        return "(" + ",".join(_key(x) for x in t) + ")"
    return repr(t)


def _comm(op: str, a, b):
    return (op,) + tuple(sorted((a, b), key=_key))


def _body(region):
    """Non-trivial ops of a region: everything but constants, pure arithmetic
    and the terminator (those only matter through the trees)."""
    out = []
    for o in region.ops:
        if o.name in ("scf.yield", "kokkos.yield", "scf.reduce") or o.name.startswith("arith.") \
                or o.name in ("memref.load", "memref.dim"):
            continue
        out.append(o)
    return out


def _reduce_of(loop):
    """(combiner, contribution value) of a single-result reducing loop."""
    from lapis.dialect import classify_combiner
    term = loop.region(0).ops[-1]
    if term.name != "scf.reduce" or len(term.operands) != 1 or len(loop.results) != 1:
        return None, None
    return classify_combiner(term.regions[0]), term.operands[0]


def _single_store(op, level="perThread"):
    """The store inside `kokkos.single {level}` holding exactly one store."""
    if op.name != "kokkos.single" or op.attrs.get("level") != level:
        return None
    ops = [o for o in op.region(0).ops if o.name != "kokkos.yield"]
    if len(ops) != 1 or ops[0].name != "memref.store":
        return None
    return ops[0]


# ------------------------------------------------------------------ helpers
def _dev_ptr(m, view, op):
    t = m.device_storage(view.root, op)
    return t.data_ptr() + view.flat_offset() * t.element_size()


def _s(m):
    return C.c_void_p(m.stream.cuda_stream)


def _ld(view) -> int:
    return view.root.strides()[0] if len(view.root.extents) >= 2 else 1


def _count(m, category, op, n) -> None:
    if n:
        key = m.path(op)
        m.counters[category][key] = m.counters[category].get(key, 0) + int(n)


# --------------------------------------------------------------- library ops
def _gemm_mode(m, kind):
    if kind in ("i32", "i64", "index"):
        return _capi.GEMM_EXACT
    return _capi.GEMM_EXACT if m.exact else _capi.GEMM_AUTO


def _lib_matmul(m, op, env):
    a, b, c = (env[v] for v in op.operands[:3])
    (mm, kk), (kk2, nn) = a.shape, b.shape
    kind = c.root.kind
    if kind not in _DT or a.root.kind != kind or b.root.kind != kind:
        return None

    def call():
        check(_capi.lib().lapis_b200_gemm(mm, nn, kk, _dev_ptr(m, a, op), _ld(a), _dev_ptr(m, b, op),
                                          _ld(b), _dev_ptr(m, c, op), _ld(c), _DT[kind],
                                          _gemm_mode(m, kind), _s(m)), "gemm")
    return call


def _lib_matvec(m, op, env):
    a, x, y = (env[v] for v in op.operands[:3])
    mm, nn = a.shape
    kind = y.root.kind
    if kind not in _DT or a.root.kind != kind or x.root.kind != kind:
        return None

    def call():
        check(_capi.lib().lapis_b200_gemv(mm, nn, _dev_ptr(m, a, op), _ld(a), _dev_ptr(m, x, op),
                                          _dev_ptr(m, y, op), _DT[kind], _s(m)), "gemv")
    return call


def _contiguous(view) -> bool:
    r = view.root
    if view.shape == r.extents:
        return True
    # a window is contiguous when it spans whole trailing dims
    for d in range(1, len(r.extents)):
        if view.shape[d] != r.extents[d] or view.offsets[d] != 0:
            return False
    return True


def _lib_batch_matmul(m, op, env):
    a, b, c = (env[v] for v in op.operands[:3])
    nb, mm, kk = a.shape
    nn = b.shape[2]
    kind = c.root.kind
    if kind not in _DT or not all(_contiguous(v) for v in (a, b, c)):
        return None

    def call():
        check(_capi.lib().lapis_b200_batch_gemm(nb, mm, nn, kk, _dev_ptr(m, a, op),
                                                _dev_ptr(m, b, op), _dev_ptr(m, c, op), _DT[kind],
                                                _gemm_mode(m, kind), _s(m)), "batch_gemm")
    return call


def _lib_spmv(m, op, env):
    rowptr, colind, values, x, y = (env[v] for v in op.operands)
    nrows = rowptr.shape[0] - 1
    return _spmv_call(m, op, rowptr, colind, values, x, y, nrows, 0)


def _lib_reduce(m, op, env):
    src, dst = env[op.operands[0]], env[op.operands[1]]
    axes = list(op.attrs["axes"])
    if len(src.shape) != 2 or len(axes) != 1 or not _contiguous(src) or not _contiguous(dst):
        return None
    kind = src.root.kind
    if kind not in _DT:
        return None
    rows, cols = src.shape

    def call():
        check(_capi.lib().lapis_b200_reduce_2d(rows, cols, _dev_ptr(m, src, op), _dev_ptr(m, dst, op),
                                               axes[0], _COMB[op.attrs["combiner"]], _DT[kind],
                                               _s(m)), "reduce_2d")
    return call


# ------------------------------------------------------------------ SpMV/SpMM
_csr_ok_cache: dict = {}


def _spmv_call(m, op, rowptr, colind, values, x, y, nrows, vl_hint):
    kinds = (values.root.kind, x.root.kind, y.root.kind)
    if len(set(kinds)) != 1 or kinds[0] not in _DT:
        return None
    if rowptr.root.kind not in _IDX_BYTES or colind.root.kind not in _IDX_BYTES:
        return None
    if rowptr.shape[0] < nrows + 1 or y.shape[0] < nrows or nrows < 0:
        return None
    if m.exact and kinds[0] in ("f32", "f64"):
        return None   # the generated kernel is the reference order
    rp, ci = _dev_ptr(m, rowptr, op), _dev_ptr(m, colind, op)
    nnz = _csr_check(m, rowptr, colind, values, x.shape[0], nrows, rp, ci)
    if nnz is None:
        return None
    lib = _capi.lib()
    plan = _csr_plan(m, rowptr, nrows, nnz, rp)

    def call():
        # the plan picks the kernel from the row-length profile (DESIGN.md
        # section 4); the reference's VL hint is recorded, not obeyed
        check(lib.lapis_b200_spmv_csr_plan(plan, rp, _IDX_BYTES[rowptr.root.kind], ci,
                                           _IDX_BYTES[colind.root.kind], _dev_ptr(m, values, op),
                                           _dev_ptr(m, x, op), _dev_ptr(m, y, op), _DT[kinds[0]],
                                           _s(m)), "spmv_csr_plan")
    return call


def _csr_plan(m, rowptr, nrows, nnz, rp):
    key = ("plan", id(rowptr.root), rowptr.flat_offset(), nrows, m.version(rowptr.root))
    plan = m.csr_plans.get(key)
    if plan is None:
        h = C.c_void_p()
        check(_capi.lib().lapis_b200_csr_plan_create(nrows, nnz, rp, _IDX_BYTES[rowptr.root.kind],
                                                     _s(m), C.byref(h)), "csr_plan_create")
        plan = m.csr_plans[key] = h
    return plan


def _csr_check(m, rowptr, colind, values, ncols, nrows, rp, ci):
    """nnz of a structure the tuned kernels may run, or None: any entry range
    outside colind / values, column outside x, or decreasing rowptr goes to
    the generated kernel, which raises the interpreter's exact error (or runs
    the empty rows) — interp.py:269-276, 798-812."""
    key = (id(rowptr.root), id(colind.root), rowptr.flat_offset(), colind.flat_offset(), nrows,
           ncols, min(colind.shape[0], values.shape[0]), m.version(rowptr.root),
           m.version(colind.root))
    hit = m.csr_checked.get(key)
    if hit is not None:
        return hit if hit >= 0 else None
    out = (C.c_int64 * 4)()
    check(_capi.lib().lapis_b200_csr_check(nrows, rp, _IDX_BYTES[rowptr.root.kind], ci,
                                           _IDX_BYTES[colind.root.kind],
                                           min(colind.shape[0], values.shape[0]), ncols, out, _s(m)),
          "csr_check")
    nnz = int(out[3]) if out[0] == 0 else -1
    m.csr_checked[key] = nnz
    return nnz if nnz >= 0 else None


def _match_spmv_nest(m, op, env):
    """thread_parallel(i < N, VL) { b = rp[i]; len = rp[i+1] - b;
    s = threadvector(jj < len) init(0) add(vals[b+jj] * x[col[b+jj]]);
    single perThread { y[i] = s } } — golden IR spmv.mlir (spmv_lowering.py:21-77)."""
    from lapis.dialect import parallel_hint_operands, parallel_init_operands
    if parallel_init_operands(op):
        return None
    nest = Nest(op)
    i = op.region(0).args[0]
    nest.roles[i] = "i"
    ops = _body(op.region(0))
    if len(ops) != 2 or ops[0].name != "kokkos.range_parallel" or \
            ops[0].attrs.get("parallelLevel") != "threadvector":
        return None
    loop, single = ops
    store = _single_store(single)
    if not loop.results or store is None or store.operands[0] is not loop.results[0]:
        return None
    inits = parallel_init_operands(loop)
    if len(inits) != 1 or not _is_zero(nest.tree(inits[0])):
        return None
    comb, contrib = _reduce_of(loop)
    if comb != "add":
        return None
    jj = loop.region(0).args[0]
    nest.roles[jj] = "jj"
    if _body(loop.region(0)):
        return None
    # y[i] = s
    ytree = nest.tree(store.operands[1])
    if _free(ytree) is None or [nest.tree(v) for v in store.operands[2:]] != [("role", "i")]:
        return None
    # bound: rp[i+1] - rp[i]
    bt = nest.tree(loop.operands[0])
    if bt[0] != "arith.subi":
        return None
    hi, lo = bt[1], bt[2]
    if lo[0] != "load" or len(lo) != 3 or lo[2] != ("role", "i"):
        return None
    rp = _free(lo[1])
    one = None
    if hi[0] == "load" and len(hi) == 3 and _free(hi[1]) is rp and hi[2][0] == "arith.addi":
        one = [t for t in hi[2][1:] if t != ("role", "i")]
    if rp is None or not one or len(one) != 1 or _const_int(one[0]) != 1:
        return None
    # contribution: vals[j] * x[col[j]], j = rp[i] + jj
    jt = _comm("arith.addi", lo, ("role", "jj"))
    ct = nest.tree(contrib)
    if ct[0] not in ("arith.mulf", "arith.muli"):
        return None
    loads = ct[1:]
    vals = xv = colv = None
    for t in loads:
        if t[0] == "load" and len(t) == 3 and t[2] == jt:
            vals = _free(t[1])
        elif t[0] == "load" and len(t) == 3 and t[2][0] == "load" and len(t[2]) == 3 \
                and t[2][2] == jt:
            xv, colv = _free(t[1]), _free(t[2][1])
    if vals is None or xv is None or colv is None:
        return None
    n = int(_outer(nest, env, op.operands[0]))
    views = [env[v] for v in (rp, colv, vals, xv, _free(ytree))]
    if any(len(v.shape) != 1 for v in views):
        return None
    _, vlv = parallel_hint_operands(op)
    call = _spmv_call(m, op, *views, n, int(env[vlv]) if vlv is not None else 0)
    if call is None:
        return None

    def run():
        call()
        _count(m, "single", single, n)
        _count(m, "store", store, n)
    return run


def _match_spmm_nest(m, op, env):
    """thread_parallel(t < N*K, VL) { i = t / K; c = t - i*K; b = rp[i];
    s = threadvector(jj < rp[i+1]-b) add(vals[b+jj] * X[col[b+jj], c]);
    single { Y[i, c] = s } } — the lowered oracle/ir/spmm.mlir."""
    from lapis.dialect import parallel_init_operands
    if parallel_init_operands(op):
        return None
    nest = Nest(op)
    t = op.region(0).args[0]
    nest.roles[t] = "t"
    ops = _body(op.region(0))
    if len(ops) != 2 or ops[0].name != "kokkos.range_parallel" or \
            ops[0].attrs.get("parallelLevel") != "threadvector" or not ops[0].results:
        return None
    loop, single = ops
    store = _single_store(single)
    if store is None or store.operands[0] is not loop.results[0]:
        return None
    inits = parallel_init_operands(loop)
    if len(inits) != 1 or not _is_zero(nest.tree(inits[0])):
        return None
    comb, contrib = _reduce_of(loop)
    if comb != "add" or _body(loop.region(0)):
        return None
    nest.roles[loop.region(0).args[0]] = "jj"
    idx = [nest.tree(v) for v in store.operands[2:]]
    if len(idx) != 2 or idx[0][0] != "arith.divi" or idx[0][1] != ("role", "t"):
        return None
    kt = idx[0][2]
    kval = _free(kt)
    it = idx[0]
    ct_want = ("arith.subi", ("role", "t"), _comm("arith.muli", it, kt))
    if kval is None or idx[1] != ct_want:
        return None
    bt = nest.tree(loop.operands[0])
    if bt[0] != "arith.subi":
        return None
    hi, lo = bt[1], bt[2]
    if lo[0] != "load" or len(lo) != 3 or lo[2] != it:
        return None
    rp = _free(lo[1])
    if not (hi[0] == "load" and len(hi) == 3 and _free(hi[1]) is rp and hi[2][0] == "arith.addi"):
        return None
    one = [x for x in hi[2][1:] if x != it]
    if len(one) != 1 or _const_int(one[0]) != 1:
        return None
    jt = _comm("arith.addi", lo, ("role", "jj"))
    ctree = nest.tree(contrib)
    if ctree[0] not in ("arith.mulf", "arith.muli"):
        return None
    vals = xv = colv = None
    for x in ctree[1:]:
        if x[0] == "load" and len(x) == 3 and x[2] == jt:
            vals = _free(x[1])
        elif x[0] == "load" and len(x) == 4 and x[3] == idx[1] and x[2][0] == "load" \
                and len(x[2]) == 3 and x[2][2] == jt:
            xv, colv = _free(x[1]), _free(x[2][1])
    if vals is None or xv is None or colv is None:
        return None
    K = int(env[kval])
    total = int(_outer(nest, env, op.operands[0]))
    if K <= 0 or total % K:
        return None
    n = total // K
    rpv, colvv, valsv, X, Y = (env[v] for v in (rp, colv, vals, xv, _free(nest.tree(store.operands[1]))))
    kinds = {valsv.root.kind, X.root.kind, Y.root.kind}
    if len(kinds) != 1 or valsv.root.kind not in _DT or len(X.shape) != 2 or len(Y.shape) != 2:
        return None
    if rpv.shape[0] < n + 1 or Y.shape[0] < n or Y.shape[1] < K or X.shape[1] < K:
        return None
    if rpv.root.kind not in _IDX_BYTES or colvv.root.kind not in _IDX_BYTES:
        return None
    if m.exact and valsv.root.kind in ("f32", "f64"):
        return None
    kind = valsv.root.kind
    rpp, cip = _dev_ptr(m, rpv, op), _dev_ptr(m, colvv, op)
    nnz = _csr_check(m, rpv, colvv, valsv, X.shape[0], n, rpp, cip)
    if nnz is None:
        return None

    def run():
        check(_capi.lib().lapis_b200_spmm_csr(
            n, X.shape[0], nnz, K, rpp, _IDX_BYTES[rpv.root.kind], cip, _IDX_BYTES[colvv.root.kind],
            _dev_ptr(m, valsv, op), _dev_ptr(m, X, op), _ld(X), _dev_ptr(m, Y, op), _ld(Y),
            _DT[kind], _s(m)), "spmm_csr")
        _count(m, "single", single, total)
        _count(m, "store", store, total)
    return run


# ------------------------------------------------------------- dense nests
def _match_matmul_nest(m, op, env):
    """team_parallel(i < M, VL) { teamthread(j < N) { s = threadvector(k < K)
    init(0) add(A[i, k] * B[k, j]); single perThread { C[i, j] = s } };
    team_barrier } — golden cpp matmul_f64.hpp:23-38 (linalg_lowering.py:95-131)."""
    from lapis.dialect import parallel_init_operands
    if parallel_init_operands(op):
        return None
    nest = Nest(op)
    nest.roles[op.region(0).args[0]] = "i"
    ops = _body(op.region(0))
    if len(ops) != 2 or ops[0].name != "kokkos.range_parallel" or \
            ops[0].attrs.get("parallelLevel") != "teamthread" or ops[1].name != "kokkos.team_barrier":
        return None
    tt, barrier = ops
    if parallel_init_operands(tt):
        return None
    nest.roles[tt.region(0).args[0]] = "j"
    inner = _body(tt.region(0))
    if len(inner) != 2 or inner[0].name != "kokkos.range_parallel" or \
            inner[0].attrs.get("parallelLevel") != "threadvector" or not inner[0].results:
        return None
    loop, single = inner
    store = _single_store(single)
    if store is None or store.operands[0] is not loop.results[0]:
        return None
    inits = parallel_init_operands(loop)
    if len(inits) != 1 or not _is_zero(nest.tree(inits[0])):
        return None
    comb, contrib = _reduce_of(loop)
    if comb != "add" or _body(loop.region(0)):
        return None
    nest.roles[loop.region(0).args[0]] = "k"
    if [nest.tree(v) for v in store.operands[2:]] != [("role", "i"), ("role", "j")]:
        return None
    ct = nest.tree(contrib)
    if ct[0] not in ("arith.mulf", "arith.muli"):
        return None
    a = b = None
    for x in ct[1:]:
        if x[0] == "load" and x[2:] == (("role", "i"), ("role", "k")):
            a = _free(x[1])
        elif x[0] == "load" and x[2:] == (("role", "k"), ("role", "j")):
            b = _free(x[1])
    cv = _free(nest.tree(store.operands[1]))
    if a is None or b is None or cv is None:
        return None
    dims = [_outer(nest, env, v) for v in (op.operands[0], tt.operands[0], loop.operands[0])]
    if any(d is None for d in dims):
        return None
    M, N, K = (int(d) for d in dims)
    A, B, Cm = env[a], env[b], env[cv]
    kind = Cm.root.kind
    if kind not in _DT or A.root.kind != kind or B.root.kind != kind:
        return None
    if M > A.shape[0] or K > A.shape[1] or K > B.shape[0] or N > B.shape[1] or \
            M > Cm.shape[0] or N > Cm.shape[1] or min(M, N, K) < 0:
        return None
    if m.exact and kind in ("f32", "f64"):
        return None

    def run():
        if M and N:
            check(_capi.lib().lapis_b200_gemm(M, N, K, _dev_ptr(m, A, op), _ld(A), _dev_ptr(m, B, op),
                                              _ld(B), _dev_ptr(m, Cm, op), _ld(Cm), _DT[kind],
                                              _gemm_mode(m, kind), _s(m)), "gemm")
        _count(m, "single", single, M * N)
        _count(m, "store", store, M * N)
        _count(m, "barrier", barrier, M)
    return run


def _match_rowdot_nest(m, op, env):
    """thread_parallel(i < M, VL) { s = threadvector(j < N) init(I) comb(e);
    single perThread { y[i] = s } } with e = A[i, j] * x[j] (matvec,
    linalg_lowering.py:134-155) or e = src[i, j] / src[j, i] (linalg.reduce
    over the last / first axis, linalg_lowering.py:214-252)."""
    from lapis.dialect import parallel_init_operands
    if parallel_init_operands(op):
        return None
    nest = Nest(op)
    nest.roles[op.region(0).args[0]] = "i"
    ops = _body(op.region(0))
    if len(ops) != 2 or ops[0].name != "kokkos.range_parallel" or \
            ops[0].attrs.get("parallelLevel") != "threadvector" or not ops[0].results:
        return None
    loop, single = ops
    store = _single_store(single)
    if store is None or store.operands[0] is not loop.results[0]:
        return None
    inits = parallel_init_operands(loop)
    if len(inits) != 1:
        return None
    comb, contrib = _reduce_of(loop)
    if comb is None or _body(loop.region(0)):
        return None
    nest.roles[loop.region(0).args[0]] = "j"
    if [nest.tree(v) for v in store.operands[2:]] != [("role", "i")]:
        return None
    yv = _free(nest.tree(store.operands[1]))
    init_t = nest.tree(inits[0])
    ct = nest.tree(contrib)
    N = _outer(nest, env, loop.operands[0])
    if N is None:
        return None
    M, N = int(env[op.operands[0]]), int(N)
    Y = env[yv] if yv is not None else None
    if Y is None or M < 0 or N < 0 or M > Y.shape[0]:
        return None
    kind = Y.root.kind
    if kind not in _DT or (m.exact and kind in ("f32", "f64") and comb in ("add", "mul")):
        return None
    # matvec
    if comb == "add" and _is_zero(init_t) and ct[0] in ("arith.mulf", "arith.muli"):
        a = x = None
        for t in ct[1:]:
            if t[0] == "load" and t[2:] == (("role", "i"), ("role", "j")):
                a = _free(t[1])
            elif t[0] == "load" and t[2:] == (("role", "j"),):
                x = _free(t[1])
        if a is None or x is None:
            return None
        A, X = env[a], env[x]
        if A.root.kind != kind or X.root.kind != kind or M > A.shape[0] or N > A.shape[1] \
                or N > X.shape[0]:
            return None

        def run_mv():
            if M:
                check(_capi.lib().lapis_b200_gemv(M, N, _dev_ptr(m, A, op), _ld(A), _dev_ptr(m, X, op),
                                                  _dev_ptr(m, Y, op), _DT[kind], _s(m)), "gemv")
            _count(m, "single", single, M)
            _count(m, "store", store, M)
        return run_mv
    # axis reduce: the init must be the combiner identity (interp.py:186-195)
    if ct[0] != "load" or len(ct) != 4 or init_t[0] != "const" or \
            not _is_identity(init_t, comb, kind):
        return None
    src = _free(ct[1])
    if src is None:
        return None
    S = env[src]
    if S.root.kind != kind or not _contiguous(S) or S.shape != S.root.extents:
        return None
    if ct[2:] == (("role", "i"), ("role", "j")):
        axis, rows, cols = 1, M, N
    elif ct[2:] == (("role", "j"), ("role", "i")):
        axis, rows, cols = 0, N, M
    else:
        return None
    if S.shape != (rows, cols):
        return None

    def run_red():
        if M:
            check(_capi.lib().lapis_b200_reduce_2d(rows, cols, _dev_ptr(m, S, op), _dev_ptr(m, Y, op),
                                                   axis, _COMB[comb], _DT[kind], _s(m)), "reduce_2d")
        _count(m, "single", single, M)
        _count(m, "store", store, M)
    return run_red


def _is_identity(t, comb, kind) -> bool:
    v = t[2]
    if kind in ("f32", "f64"):
        want = {"add": 0.0, "mul": 1.0, "min": float("inf"), "max": float("-inf")}[comb]
        return struct.pack("<d", float(v)) == struct.pack("<d", want)
    w = 32 if kind == "i32" else 64
    want = {"add": 0, "mul": 1, "min": (1 << (w - 1)) - 1, "max": -(1 << (w - 1))}[comb]
    return int(v) == want


def _match_relu_nest(m, op, env):
    """range_parallel topmdrange (i, j) { x = T[i, j]; O[i, j] = x > 0 ? x : 0 }
    — the lowered linalg.elementwise ReLU of the GCN (oracle/ir/gcn_f32.mlir)."""
    if op.attrs.get("parallelLevel") not in ("toprange", "topmdrange"):
        return None
    from lapis.dialect import parallel_init_operands
    if parallel_init_operands(op):
        return None
    nest = Nest(op)
    args = op.region(0).args
    for d, a in enumerate(args):
        nest.roles[a] = f"d{d}"
    ops = _body(op.region(0))
    if len(ops) != 1 or ops[0].name != "memref.store":
        return None
    store = ops[0]
    roles = tuple(("role", f"d{d}") for d in range(len(args)))
    if tuple(nest.tree(v) for v in store.operands[2:]) != roles:
        return None
    vt = nest.tree(store.operands[0])
    if vt[0] != "arith.select":
        return None
    cond, a, b = vt[1], vt[2], vt[3]
    if not (a[0] == "load" and a[2:] == roles and _is_zero(b) and cond[0] == "arith.cmpf"):
        return None
    cmp_op = store.operands[0].defining_op().operands[0].defining_op()
    if cmp_op.attrs.get("predicate") != "ogt" or cond[1] != a or not _is_zero(cond[2]):
        return None
    src, dst = env[_free(a[1])], env[_free(nest.tree(store.operands[1]))]
    ext = tuple(int(_outer(nest, env, v)) for v in op.operands[:len(args)])
    if src.shape != ext or dst.shape != ext or not _contiguous(src) or not _contiguous(dst):
        return None
    kind = dst.root.kind
    if kind not in ("f32", "f64") or src.root.kind != kind:
        return None
    total = 1
    for e in ext:
        total *= e

    def run():
        if total:
            check(_capi.lib().lapis_b200_relu(total, _dev_ptr(m, src, op), _dev_ptr(m, dst, op),
                                              _DT[kind], _s(m)), "relu")
        _count(m, "store", store, total)
    return run


_LIBRARY = {
    "kokkos.gemm": _lib_matmul, "linalg.matmul": _lib_matmul,
    "kokkos.gemv": _lib_matvec, "linalg.matvec": _lib_matvec,
    "linalg.batch_matmul": _lib_batch_matmul,
    "sparse.spmv_csr": _lib_spmv, "kokkos.spmv_csr": _lib_spmv,
    "linalg.reduce": _lib_reduce,
}

_NESTS = {
    "kokkos.thread_parallel": (_match_spmv_nest, _match_spmm_nest, _match_rowdot_nest),
    "kokkos.team_parallel": (_match_matmul_nest,),
    "kokkos.range_parallel": (_match_relu_nest,),
}


def match(m, op, env):
    """A callable that runs ``op`` on a hand-written kernel, or None."""
    f = _LIBRARY.get(op.name)
    if f is not None:
        return f(m, op, env)
    for matcher in _NESTS.get(op.name, ()):
        call = matcher(m, op, env)
        if call is not None:
            return call
    return None
