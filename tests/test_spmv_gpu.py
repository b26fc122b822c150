"""Parity of the sm_100a CSR SpMV kernels with the reference.

* every reference-generated fixture (tests/golden/spmv*.npz): bit-exact for the
  default row-stream kernel, within diff_outputs tolerance (interp.py:1050) for
  the emitted-mapping vector kernels (VL = 1 is sequential, hence bit-exact);
* larger seeded ragged / power-law / stencil matrices against the C oracle:
  rows of <= 512 entries bit-exact, longer rows within tolerance;
* the 1M-row 5-point Laplacian (config 1) against the reference's OWN emitted
  C++ on its serial stub (oracle/_ref), bit-exact.
"""
import numpy as np
import pytest
import torch

import paper_2509_25605_b200 as lb
from conftest import bits_equal, golden_names, load_golden
from matrices import powerlaw_csr, ragged_csr, stencil_csr
from oracle import oracle as O
from oracle import ref as R

pytestmark = pytest.mark.gpu
TOL = {np.dtype(np.float64): 1e-12, np.dtype(np.float32): 1e-5}
LONG_ROW = 512


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


def assert_close(got, want, rowptr=None):
    """Ints exact; floats within diff_outputs tolerance; rows <= LONG_ROW bit-exact."""
    got, want = np.asarray(got), np.asarray(want)
    if want.dtype.kind in "iu":
        assert np.array_equal(got, want)
        return
    ok, msg = O.diff_outputs([got], [want], TOL[want.dtype])
    assert ok, msg
    if rowptr is not None:
        short = np.diff(rowptr) <= LONG_ROW
        assert bits_equal(got[short], want[short])


@pytest.mark.parametrize("name", golden_names("spmv"))
def test_golden_tile_kernel_bitexact(cuda_device, name):
    g = load_golden(name)
    rowptr, colind, values, x, _ = g["inputs"]
    y = lb.spmv_csr(cu(rowptr), cu(colind), cu(values), cu(x))
    assert bits_equal(host(y), g["outputs"][0]), name


@pytest.mark.parametrize("name", golden_names("spmv"))
@pytest.mark.parametrize("vl", [1, 2, 4, 8, 16, 32])
def test_golden_vector_kernel(cuda_device, name, vl):
    g = load_golden(name)
    rowptr, colind, values, x, _ = g["inputs"]
    y = host(lb.spmv_csr(cu(rowptr), cu(colind), cu(values), cu(x), vector_length=vl))
    if vl == 1:
        assert bits_equal(y, g["outputs"][0])
    else:
        assert_close(y, g["outputs"][0])


def test_golden_hint_drives_vector_kernel(cuda_device):
    # the emitted code computes VL from rowptr (golden/cpp/spmv.hpp:17-33)
    for name in golden_names("spmv"):
        g = load_golden(name)
        rowptr = g["inputs"][0]
        n = rowptr.shape[0] - 1
        assert lb.csr_vector_length(n, int(rowptr[-1])) == g["hints"][0]


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("idx", ["i64/i32", "i64/i64", "i32/i32"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32, np.int64, np.int32])
def test_ragged_with_long_rows(cuda_device, seed, idx, dtype):
    rng = np.random.default_rng(seed)
    rowptr, colind, values = ragged_csr(rng, 5000, 3000, max_len=60, empty_every=13,
                                        long_rows={7: 2999, 4000: 700, 4001: 513, 4999: 1500},
                                        dtype=dtype)
    x = (rng.integers(-9, 9, 3000) if np.issubdtype(dtype, np.integer)
         else rng.uniform(-1, 1, 3000)).astype(dtype)
    rp_t, ci_t = idx.split("/")
    rp = rowptr.astype(np.int64 if rp_t == "i64" else np.int32)
    ci = colind.astype(np.int64 if ci_t == "i64" else np.int32)
    want = O.spmv_csr(rowptr, colind, values, x)
    got = host(lb.spmv_csr(cu(rp), cu(ci), cu(values), cu(x)))
    assert_close(got, want, rowptr)
    got8 = host(lb.spmv_csr(cu(rp), cu(ci), cu(values), cu(x), vector_length=8))
    assert_close(got8, want)


def test_plan_reuse_and_offset_rowptr(cuda_device):
    rng = np.random.default_rng(5)
    rowptr, colind, values = powerlaw_csr(rng, 20000, mean=12.0)
    x = rng.uniform(-1, 1, 20000)
    want = O.spmv_csr(rowptr, colind, values, x)
    rp = cu(rowptr)
    plan = lb.CsrPlan(rp)
    ci, v = cu(colind), cu(values)
    for _ in range(3):
        assert_close(host(plan.spmv(ci, v, cu(x))), want, rowptr)
    x2 = rng.uniform(-1, 1, 20000)
    assert_close(host(plan.spmv(ci, v, cu(x2))), O.spmv_csr(rowptr, colind, values, x2), rowptr)
    plan.close()
    # a row-block window: rowptr not starting at 0 (subview semantics)
    r0, r1 = 3000, 9000
    sub = lb.spmv_csr(cu(rowptr[r0:r1 + 1]), ci, v, cu(x))
    assert bits_equal(host(sub)[np.diff(rowptr[r0:r1 + 1]) <= LONG_ROW],
                      want[r0:r1][np.diff(rowptr[r0:r1 + 1]) <= LONG_ROW])


def test_empty_and_degenerate(cuda_device):
    y = lb.spmv_csr(cu(np.zeros(1, np.int64)), cu(np.zeros(0, np.int32)), cu(np.zeros(0)),
                    cu(np.zeros(3)))
    assert y.numel() == 0
    y = lb.spmv_csr(cu(np.zeros(6, np.int64)), cu(np.zeros(0, np.int32)), cu(np.zeros(0)),
                    cu(np.ones(5)))
    assert host(y).tolist() == [0.0] * 5
    # 100k empty rows then one row: ownership of empty rows spans many tiles
    rowptr = np.zeros(100_002, np.int64)
    rowptr[-1] = 3
    y = host(lb.spmv_csr(cu(rowptr), cu(np.array([0, 1, 2], np.int32)), cu(np.ones(3)),
                         cu(np.array([1.0, 2.0, 3.0]))))
    assert y[-1] == 6.0 and not y[:-1].any()


def test_errors_are_raised_not_aborted(cuda_device):
    rp, ci, v, x = cu(np.array([0, 1], np.int64)), cu(np.array([0], np.int32)), cu(np.ones(1)), cu(np.ones(1))
    with pytest.raises(lb.BackendError):
        lb.spmv_csr(rp, ci, v, x, torch.empty(5, dtype=torch.float64, device="cuda"))
    with pytest.raises(lb.BackendError):
        lb.spmv_csr(rp, ci, v, x, vector_length=3)
    with pytest.raises(lb.BackendError):
        lb.spmv_csr(rp, ci, v, x.float())


def test_device_stencil_matches_host_structure(cuda_device):
    for points, n in ((5, 37), (27, 11), (27, 1), (5, 2)):
        rowptr, colind, values = stencil_csr(points, n)
        drp, dci, dv = lb.synth_stencil(points, n)
        assert np.array_equal(host(drp), rowptr)
        assert np.array_equal(host(dci), colind)
        assert bits_equal(host(dv), values)
        # a row block, rebased
        N = rowptr.size - 1
        r0, r1 = N // 3, 2 * N // 3
        brp, bci, bv = lb.synth_stencil(points, n, r0, r1)
        assert np.array_equal(host(brp), rowptr[r0:r1 + 1] - rowptr[r0])
        assert np.array_equal(host(bci), colind[rowptr[r0]:rowptr[r1]])


def test_stencil27_1m_rows_bitexact_vs_oracle(cuda_device):
    n = 100
    rp, ci, v = lb.synth_stencil(27, n)
    x = np.random.default_rng(5).uniform(-1, 1, n ** 3)
    y = host(lb.spmv_csr(rp, ci, v, cu(x)))
    want = O.spmv_csr(host(rp), host(ci), host(v), x)
    assert bits_equal(y, want)
    y32 = host(lb.spmv_csr(rp, ci, v, cu(x), vector_length=32))
    assert_close(y32, want)


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
def test_config1_laplacian_bitexact_vs_reference_emitted_cpp(cuda_device):
    # config 1: 1M rows, 4,996,000 nnz, the reference's own CPU path
    rp, ci, v = lb.synth_stencil(5, 1000)
    assert int(rp[-1]) == 4_996_000
    x = np.random.default_rng(1).uniform(-1, 1, 1_000_000)
    y = host(lb.spmv_csr(rp, ci, v, cu(x)))
    yref, _ = R.spmv_csr(host(rp), host(ci).astype(np.int64), host(v), x, threads=4)
    assert bits_equal(y, yref)


@pytest.mark.parametrize("vl", [1, 2, 4, 8, 16, 32])
@pytest.mark.parametrize("dtype", [np.float64, np.float32, np.int64])
def test_exact_vector_kernel_bitexact_all_rows(cuda_device, monkeypatch, vl, dtype):
    # the plan's exact vector mode: every row (long ones included) bit-identical
    monkeypatch.setenv("LAPIS_B200_SPMV_VL", str(vl))
    rng = np.random.default_rng(vl)
    rowptr, colind, values = ragged_csr(rng, 3000, 2500, max_len=70, empty_every=9,
                                        long_rows={5: 2499, 2999: 1300}, dtype=dtype)
    x = (rng.integers(-9, 9, 2500) if np.issubdtype(dtype, np.integer)
         else rng.uniform(-1, 1, 2500)).astype(dtype)
    plan = lb.CsrPlan(cu(rowptr), exact=True)
    assert plan.info()["vector_length"] == vl and plan.info()["exact"]
    y = host(plan.spmv(cu(colind), cu(values), cu(x)))
    assert bits_equal(y, O.spmv_csr(rowptr, colind, values, x))
    # default (tree) mode: within the diff_outputs contract; fp32 stays exact
    tree = lb.CsrPlan(cu(rowptr))
    yt = host(tree.spmv(cu(colind), cu(values), cu(x)))
    if dtype == np.float32:
        assert bits_equal(yt, O.spmv_csr(rowptr, colind, values, x))
    else:
        assert_close(yt, O.spmv_csr(rowptr, colind, values, x))


def test_plan_picks_exact_vector_for_stencils(cuda_device):
    for points, n, vl in ((27, 20, 4), (5, 60, 1)):
        rp, ci, v = lb.synth_stencil(points, n)
        plan = lb.CsrPlan(rp, exact=True)
        info = plan.info()
        assert info["vector_length"] == vl, info
        x = np.random.default_rng(0).uniform(-1, 1, rp.numel() - 1)
        y = host(plan.spmv(ci, v, cu(x)))
        want = O.spmv_csr(host(rp), host(ci), host(v), x)
        assert bits_equal(y, want)
        assert_close(host(lb.CsrPlan(rp).spmv(ci, v, cu(x))), want)
    rng = np.random.default_rng(5)
    rowptr, colind, values = powerlaw_csr(rng, 20000, mean=12.0)
    assert lb.CsrPlan(cu(rowptr)).info()["vector_length"] == 0  # irregular -> tile kernel


@pytest.mark.parametrize("nrows", [1, 31, 33, 3000])
@pytest.mark.parametrize("dtype", [np.float64, np.float32, np.int64, np.int32])
def test_warpblock_kernel_bitexact(cuda_device, monkeypatch, nrows, dtype):
    # warp-block kernel forced on ragged rows (empty rows, rows far longer than
    # its 256-entry window): in exact mode every row is the reference's
    # sequential sum
    monkeypatch.setenv("LAPIS_B200_SPMV_KERNEL", "wb")
    rng = np.random.default_rng(nrows)
    longs = {0: 700, nrows - 1: 1300} if nrows > 2 else {}
    rowptr, colind, values = ragged_csr(rng, nrows, 2500, max_len=20, empty_every=7,
                                        long_rows=longs, dtype=dtype)
    x = (rng.integers(-9, 9, 2500) if np.issubdtype(dtype, np.integer)
         else rng.uniform(-1, 1, 2500)).astype(dtype)
    want = O.spmv_csr(rowptr, colind, values, x)
    plan = lb.CsrPlan(cu(rowptr), exact=True)
    assert plan.info()["warpblock"], plan.info()
    y = host(plan.spmv(cu(colind), cu(values), cu(x)))
    assert bits_equal(y, want)
    # default mode: rows <= 512 still in order; longer fp64 rows folded by the
    # warp as a fixed tree (within tolerance); fp32 and ints stay exact
    tree = lb.CsrPlan(cu(rowptr))
    yt = host(tree.spmv(cu(colind), cu(values), cu(x)))
    if dtype == np.float64:
        assert_close(yt, want, rowptr)
    else:
        assert bits_equal(yt, want)


def test_warpblock_offset_rowptr(cuda_device, monkeypatch):
    # a row slice whose rowptr does not start at 0 (a shard's view)
    monkeypatch.setenv("LAPIS_B200_SPMV_KERNEL", "wb")
    rp, ci, v = lb.synth_stencil(5, 70)
    rph, cih, vh = host(rp), host(ci), host(v)
    r0, r1 = 101, 4000
    sub = rp[r0:r1 + 1]
    plan = lb.CsrPlan(sub)
    assert plan.info()["warpblock"]
    x = np.random.default_rng(3).uniform(-1, 1, rph.size - 1)
    y = host(plan.spmv(ci, v, cu(x)))
    want = O.spmv_csr(rph, cih, vh, x)[r0:r1]
    assert bits_equal(y, want)
    # a descending rowptr entry rules the warp-block kernel out
    bad = rph[:50].copy()
    bad[10] = bad[12]
    assert not lb.CsrPlan(cu(bad)).info()["warpblock"]


@pytest.mark.parametrize("points,n", [(27, 14), (5, 90)])
def test_native_rowblock_world1(cuda_device, points, n):
    # the C-ABI row-block path with the backend's own NCCL communicator
    # (world 1 on one GPU): bit-identical to the plan multiply
    from paper_2509_25605_b200 import sharded
    rp, ci, v = lb.synth_stencil(points, n)
    N = rp.numel() - 1
    comm = sharded.NcclComm(0, 1)
    op = sharded.NativeRowBlockSpmv(rp, ci, v, [(0, N)], 0, 1, comm, exact=True)
    info = op.info()
    assert info["interior"] == (0, N)
    x = torch.from_numpy(np.random.default_rng(9).uniform(-1, 1, N)).cuda()
    y = torch.empty(N, dtype=torch.float64, device="cuda")
    op.multiply(x, y)
    want = O.spmv_csr(host(rp), host(ci), host(v), host(x))
    assert bits_equal(host(y), want)
    op.close()
    comm.close()


def test_native_rowblock_rejects_unrebased_rowptr(cuda_device):
    from paper_2509_25605_b200 import sharded
    rp, ci, v = lb.synth_stencil(5, 30)
    sub = rp[100:200 + 1]
    with pytest.raises(lb.BackendError):
        sharded.NativeRowBlockSpmv(sub, ci, v, [(100, 200)], 0, 1, None)


def test_no_plan_call_device_dispatch(cuda_device):
    # lapis_b200_spmv_csr without a plan (the emitted C++'s LAPIS::spmv_csr):
    # a regular stencil takes the exact vector kernel (VL 4: every row
    # bit-identical), a power-law matrix the warp-block kernel (rows <= 512
    # bit-identical, hub rows within tolerance)
    rp, ci, v = lb.synth_stencil(27, 24)
    x = np.random.default_rng(1).uniform(-1, 1, rp.numel() - 1)
    y = host(lb.spmv_csr(rp, ci, v, cu(x)))
    assert bits_equal(y, O.spmv_csr(host(rp), host(ci), host(v), x))
    rng = np.random.default_rng(2)
    rowptr, colind, values = powerlaw_csr(rng, 30000, mean=10.0)
    assert np.diff(rowptr).max() > 512
    x2 = rng.uniform(-1, 1, 30000)
    y2 = host(lb.spmv_csr(cu(rowptr), cu(colind), cu(values), cu(x2)))
    assert_close(y2, O.spmv_csr(rowptr, colind, values, x2), rowptr)


def decreasing_rowptr_csr(rng, nrows, ncols, dtype=np.float64):
    """A CSR whose rowptr DECREASES at some rows (interp.py:808 sums
    range(begin, max(begin, end)): such a row is empty, its neighbours may
    overlap), spanning many tiles / warp blocks, with long rows among them."""
    rowptr, colind, values = ragged_csr(rng, nrows, ncols, max_len=40,
                                        long_rows={5: 3000, nrows // 2: 2500}, dtype=dtype)
    rp = rowptr.copy()
    nnz = int(rp[-1])
    for r in rng.choice(np.arange(10, nrows - 10), size=nrows // 50, replace=False):
        rp[r] = min(nnz, rp[r] + int(rng.integers(50, 4000)))   # row r-1 grows, row r shrinks
    return rp, colind, values


@pytest.mark.parametrize("dtype", [np.float64, np.float32, np.int64])
def test_decreasing_rowptr(cuda_device, dtype):
    """a rowptr that decreases through the no-plan call and a plan."""
    rng = np.random.default_rng(21)
    rp, colind, values = decreasing_rowptr_csr(rng, 6000, 5000, dtype=dtype)
    assert (np.diff(rp) < 0).any()
    x = (rng.integers(-9, 9, 5000) if np.issubdtype(dtype, np.integer)
         else rng.uniform(-1, 1, 5000)).astype(dtype)
    want = O.spmv_csr(rp, colind, values, x)
    for rpt in (rp, rp.astype(np.int32)):
        got = host(lb.spmv_csr(cu(rpt), cu(colind), cu(values), cu(x)))
        assert_close(got, want, np.maximum(rp, 0))
        plan = lb.CsrPlan(cu(rpt), nnz=int(rp.max()))
        assert plan.info()["vector_length"] == 1
        got = host(plan.spmv(cu(colind), cu(values), cu(x)))
        assert bits_equal(got, want) if want.dtype.kind == "f" else np.array_equal(got, want)
