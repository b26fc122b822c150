"""Small invocations of every kernel that uses mbarriers / TMA / cp.async /
tcgen05, for compute-sanitizer (memcheck, racecheck, synccheck):

    compute-sanitizer --tool memcheck  python scripts/sanitize.py
    compute-sanitizer --tool racecheck python scripts/sanitize.py
    compute-sanitizer --tool synccheck python scripts/sanitize.py

Each call is checked against the oracle as well, so a run also shows the
kernels still compute the right thing under the tool's serialisation.
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import paper_2509_25605_b200 as lb  # noqa: E402
import synth_inputs as S  # noqa: E402
from matrices import ragged_csr  # noqa: E402
from oracle import oracle as O  # noqa: E402

rng = np.random.default_rng(0)
cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
only = set(sys.argv[1:])


def case(name):
    def deco(f):
        if not only or name in only:
            f()
            torch.cuda.synchronize()
            print("ok", name, flush=True)
        return f
    return deco


@case("spmv_tile")
def _():
    rp, ci, v = ragged_csr(rng, 3000, 2000, max_len=40, long_rows={7: 1999, 100: 900})
    x = rng.uniform(-1, 1, 2000)
    os.environ["LAPIS_B200_SPMV_KERNEL"] = "tile"
    plan = lb.CsrPlan(cu(rp))
    y = plan.spmv(cu(ci), cu(v), cu(x)).cpu().numpy()
    del os.environ["LAPIS_B200_SPMV_KERNEL"]
    assert O.diff_outputs([y], [O.spmv_csr(rp, ci, v, x)], 1e-12)[0]


@case("spmv_vector_warpblock_noplan")
def _():
    rp, ci, v = ragged_csr(rng, 2500, 2000, max_len=30, long_rows={3: 1500})
    x = rng.uniform(-1, 1, 2000)
    y = lb.spmv_csr(cu(rp), cu(ci), cu(v), cu(x)).cpu().numpy()
    assert O.diff_outputs([y], [O.spmv_csr(rp, ci, v, x)], 1e-12)[0]
    rs, cs, vs = S.stencil_rows(27, 9, 0, 729)
    xs = rng.uniform(-1, 1, 729)
    y = lb.CsrPlan(cu(rs), exact=True).spmv(cu(cs.astype(np.int32)), cu(vs), cu(xs)).cpu().numpy()
    assert np.array_equal(y, O.spmv_csr(rs, cs, vs, xs))


@case("spmv_rowstream")
def _():
    # TMA-staged tiles (27-point rows), the global-load fallback (ragged rows
    # forced onto the kernel) and an unaligned operand (no bulk copies)
    rs, cs, vs = S.stencil_rows(27, 11, 0, 1331)
    xs = rng.uniform(-1, 1, 1331)
    want = O.spmv_csr(rs, cs, vs, xs)
    plan = lb.CsrPlan(cu(rs), exact=True)
    assert plan.info()["rowstream"]
    assert np.array_equal(plan.spmv(cu(cs.astype(np.int32)), cu(vs), cu(xs)).cpu().numpy(), want)
    va = torch.cat([torch.zeros(1, dtype=torch.float64), torch.from_numpy(vs)]).cuda()[1:]
    assert np.array_equal(plan.spmv(cu(cs.astype(np.int32)), va, cu(xs)).cpu().numpy(), want)
    rp, ci, v = ragged_csr(rng, 700, 3000, max_len=60, long_rows={3: 2900})
    x = rng.uniform(-1, 1, 3000)
    os.environ["LAPIS_B200_SPMV_KERNEL"] = "rs"
    y = lb.CsrPlan(cu(rp), exact=True).spmv(cu(ci), cu(v), cu(x)).cpu().numpy()
    del os.environ["LAPIS_B200_SPMV_KERNEL"]
    assert np.array_equal(y, O.spmv_csr(rp, ci, v, x))
    # counter tiles (half, then all of them)
    for dyn in ("50", "100"):
        os.environ["LAPIS_B200_RS_DYN"] = dyn
        assert np.array_equal(plan.spmv(cu(cs.astype(np.int32)), cu(vs), cu(xs)).cpu().numpy(), want)
    del os.environ["LAPIS_B200_RS_DYN"]


@case("spmm_plan_hints")
def _():
    # SpMM plan with hot rows and far-reuse hints (policy loads)
    rp, ci = S.powerlaw_structure_host(S.PowerLawSpec(4000, mean=8.0, seed=3))
    v = rng.uniform(-1, 1, int(rp[-1]))
    X = rng.uniform(-1, 1, (4000, 64))
    os.environ["LAPIS_B200_SPMM_HINT"] = "1"   # opt-in reuse hints
    plan = lb.SpmmPlan(cu(rp), cu(ci), 4000, 64, torch.float64, hot_bytes=64 << 10)
    del os.environ["LAPIS_B200_SPMM_HINT"]
    assert plan.info()["far_reuse_entries"] >= 0
    Y = plan.spmm(cu(v), cu(X)).cpu().numpy()
    assert O.diff_outputs([Y], [O.spmm_csr(rp, ci, v, X)], 1e-12)[0]


@case("row_fold_pipe")
def _():
    A = rng.uniform(-1, 1, (300, 1030))
    x = rng.uniform(-1, 1, 1030)
    assert np.array_equal(lb.gemv(cu(A), cu(x)).cpu().numpy(), O.matvec(A, x))
    r = lb.reduce2d(cu(A), 1, "add").cpu().numpy()
    assert np.array_equal(r, O.reduce2d(A, 1, "add"))


@case("spmm_long_rows")
def _():
    for dt in (np.float32, np.float64):
        rp, ci, v = ragged_csr(rng, 600, 5000, max_len=20, long_rows={5: 4999, 300: 2500}, dtype=dt)
        X = rng.uniform(-1, 1, (5000, 64)).astype(dt)
        Y = lb.spmm_csr(cu(rp), cu(ci), cu(v), cu(X)).cpu().numpy()
        assert O.diff_outputs([Y], [O.spmm_csr(rp, ci, v, X)], 1e-5 if dt == np.float32 else 1e-12)[0]


@case("gemm_tcgen05")
def _():
    for dt, mode, tol in ((np.float32, "auto", 1e-5), (np.float64, "auto", 1e-12),
                          (np.float32, "ozaki", 1e-5), (np.float64, "dmma", 1e-12)):
        A = rng.uniform(0, 1, (200, 300)).astype(dt)
        B = rng.uniform(0, 1, (300, 260)).astype(dt)
        C = lb.gemm(cu(A), cu(B), mode=mode).cpu().numpy()
        assert O.diff_outputs([C], [O.matmul(A, B)], tol)[0], (dt, mode)


@case("gcn_dense_tcgen05")
def _():
    rp, ci = S.powerlaw_structure_host(S.PowerLawSpec(700, mean=6.0, seed=2))
    v = S.gcn_values_host(rp, ci)
    X, W = S.gcn_features(700, 64, 4)
    H = lb.gcn_layer(cu(rp), cu(ci), cu(v), cu(X), cu(W)).cpu().numpy()
    assert O.diff_outputs([H], [O.gcn(rp, ci, v, X, W)], 1e-5)[0]

print("sanitize.py: all cases ran")
