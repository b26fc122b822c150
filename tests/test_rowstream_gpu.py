"""The row-stream SpMV kernel (csrc/spmv.cu spmv_rowstream_kernel): the
reference-order fold of regular structures with the entry stream staged by the
TMA engine.  Every case is bit-identical to the oracle's sequential row sums
(interp.py:808-811): stencils (the plan's and the no-plan call's choice),
forced on ragged rows (tiles larger than a stage fall back to global loads),
unaligned operands (no bulk copies), an offset rowptr and every value type."""
import numpy as np
import pytest
import torch

import paper_2509_25605_b200 as lb
from conftest import bits_equal
from matrices import ragged_csr, stencil_csr
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


def _x(rng, n, dtype):
    if np.issubdtype(dtype, np.integer):
        return rng.integers(-9, 9, n).astype(dtype)
    return rng.uniform(-1, 1, n).astype(dtype)


@pytest.mark.parametrize("points,n", [(27, 5), (27, 23), (27, 41)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32, np.int64, np.int32])
def test_stencil_plan_exact(cuda_device, points, n, dtype):
    rowptr, colind, values = stencil_csr(points, n)
    values = values.astype(dtype)
    rng = np.random.default_rng(points * 1000 + n)
    x = _x(rng, rowptr.size - 1, dtype)
    plan = lb.CsrPlan(cu(rowptr), exact=True)
    info = plan.info()
    assert info["rowstream"] and "rowstream" in info["kernel"], info
    want = O.spmv_csr(rowptr, colind, values, x)
    assert bits_equal(host(plan.spmv(cu(colind), cu(values), cu(x))), want)
    # the no-plan call (the emitted C++'s LAPIS::spmv_csr) takes it too
    assert bits_equal(host(lb.spmv_csr(cu(rowptr), cu(colind), cu(values), cu(x))), want)


@pytest.mark.parametrize("nrows", [1, 255, 257, 5000])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_forced_on_ragged_rows(cuda_device, monkeypatch, nrows, dtype):
    # long rows push a tile past its stage (global-load fallback for that tile)
    monkeypatch.setenv("LAPIS_B200_SPMV_KERNEL", "rs")
    rng = np.random.default_rng(nrows)
    longs = {0: 2400, nrows - 1: 9000} if nrows > 2 else {}
    rowptr, colind, values = ragged_csr(rng, nrows, 12000, max_len=60, empty_every=7,
                                        long_rows=longs, dtype=dtype)
    x = _x(rng, 12000, dtype)
    plan = lb.CsrPlan(cu(rowptr), exact=True)
    assert plan.info()["rowstream"], plan.info()
    want = O.spmv_csr(rowptr, colind, values, x)
    assert bits_equal(host(plan.spmv(cu(colind), cu(values), cu(x))), want)
    # forced in tree mode too: still the sequential sum
    assert bits_equal(host(lb.CsrPlan(cu(rowptr)).spmv(cu(colind), cu(values), cu(x))), want)


def test_unaligned_operands_and_offset_rowptr(cuda_device):
    rowptr, colind, values = stencil_csr(27, 13)
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, rowptr.size - 1)
    want = O.spmv_csr(rowptr, colind, values, x)
    # colind / values one element into their allocations: no 16-byte alignment
    ci = torch.cat([torch.zeros(1, dtype=torch.int32), torch.from_numpy(colind)]).cuda()[1:]
    va = torch.cat([torch.zeros(1, dtype=torch.float64), torch.from_numpy(values)]).cuda()[1:]
    plan = lb.CsrPlan(cu(rowptr), exact=True)
    assert bits_equal(host(plan.spmv(ci, va, cu(x))), want)
    # rowptr starting at 7: the entry stream begins 7 entries into the arrays
    off = 7
    rp7 = rowptr + off
    ci7 = np.concatenate([np.full(off, -1, np.int32), colind])
    va7 = np.concatenate([np.full(off, np.nan), values])
    plan7 = lb.CsrPlan(cu(rp7), exact=True)
    assert bits_equal(host(plan7.spmv(cu(ci7), cu(va7), cu(x))), want)


def test_large_stencil_matches_oracle(cuda_device):
    # a multi-tile, multi-wave 27-point case (1.7M rows) on the device generator
    n = 120
    rp, ci, v = lb.synth_stencil(27, n)
    x = np.random.default_rng(9).uniform(-1, 1, n ** 3)
    plan = lb.CsrPlan(rp, exact=True)
    assert plan.info()["rowstream"]
    y = host(plan.spmv(ci, v, cu(x)))
    assert bits_equal(y, O.spmv_csr(host(rp), host(ci), host(v), x))


@pytest.mark.parametrize("rp_dt,ci_dt", [(np.int32, np.int32), (np.int32, np.int64), (np.int64, np.int64)])
def test_index_widths(cuda_device, rp_dt, ci_dt):
    # every rowptr / colind width the C ABI accepts goes through the kernel
    rowptr, colind, values = stencil_csr(27, 17)
    rowptr, colind = rowptr.astype(rp_dt), colind.astype(ci_dt)
    x = np.random.default_rng(2).uniform(-1, 1, rowptr.size - 1)
    plan = lb.CsrPlan(cu(rowptr), exact=True)
    assert plan.info()["rowstream"]
    want = O.spmv_csr(rowptr, colind, values, x)
    assert bits_equal(host(plan.spmv(cu(colind), cu(values), cu(x))), want)
    assert bits_equal(host(lb.spmv_csr(cu(rowptr), cu(colind), cu(values), cu(x))), want)


@pytest.mark.parametrize("dyn", ["0", "15", "60", "100"])
def test_counter_tiles(cuda_device, monkeypatch, dyn):
    # the tiles past the static share come from the atomic counter
    # (LAPIS_B200_RS_DYN percent of them; large problems only): same bits
    monkeypatch.setenv("LAPIS_B200_RS_DYN", dyn)
    n = 100
    rp, ci, v = lb.synth_stencil(27, n)
    x = np.random.default_rng(int(dyn)).uniform(-1, 1, n ** 3)
    plan = lb.CsrPlan(rp, exact=True)
    y = host(plan.spmv(ci, v, cu(x)))
    want = O.spmv_csr(host(rp), host(ci), host(v), x)
    assert bits_equal(y, want)
    assert bits_equal(host(lb.spmv_csr(rp, ci, v, cu(x))), want)


@pytest.mark.parametrize("dyn", ["15", "100"])
def test_counter_tiles_ragged(cuda_device, monkeypatch, dyn):
    # forced on a ragged matrix large enough for the counter split: tiles
    # staged, tiles past a stage (global loads) and empty rows interleave
    monkeypatch.setenv("LAPIS_B200_SPMV_KERNEL", "rs")
    monkeypatch.setenv("LAPIS_B200_RS_DYN", dyn)
    rng = np.random.default_rng(77)
    nrows, ncols = 800_000, 50_000   # 12500 tiles of 64 rows: past 16 per CTA
    counts = rng.integers(0, 40, nrows)
    counts[::5] = 0
    counts[123], counts[nrows - 1] = 5000, 3000
    rowptr = np.zeros(nrows + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum(counts)
    colind = rng.integers(0, ncols, int(rowptr[-1])).astype(np.int32)
    values = rng.uniform(-1, 1, int(rowptr[-1]))
    x = rng.uniform(-1, 1, ncols)
    plan = lb.CsrPlan(cu(rowptr), exact=True)
    assert plan.info()["rowstream"], plan.info()
    assert bits_equal(host(plan.spmv(cu(colind), cu(values), cu(x))),
                      O.spmv_csr(rowptr, colind, values, x))
