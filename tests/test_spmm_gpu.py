"""Parity of the sm_100a CSR x dense SpMM with the reference loop nest
(oracle/ir/spmm.mlir lowered by the reference; golden fixture spmm_k8) and with
the C oracle on power-law matrices whose hub rows exceed the 2048-entry split."""
import numpy as np
import pytest
import torch

import paper_2509_25605_b200 as lb
from conftest import bits_equal, load_golden
from matrices import powerlaw_csr, ragged_csr
from oracle import oracle as O

pytestmark = pytest.mark.gpu
SPLIT = 2048


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_golden_spmm_bitexact(cuda_device):
    g = load_golden("spmm_k8")
    rowptr, colind, values, X, _ = g["inputs"]
    Y = lb.spmm_csr(cu(rowptr), cu(colind), cu(values), cu(X)).cpu().numpy()
    assert bits_equal(Y, g["outputs"][0])


@pytest.mark.parametrize("k", [64, 7, 1, 96])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_powerlaw_with_hub_rows(cuda_device, k, dtype):
    rng = np.random.default_rng(k)
    rowptr, colind, values = ragged_csr(rng, 3000, 9000, max_len=30, empty_every=11,
                                        long_rows={0: 8999, 1500: 2049, 1501: 5000, 2999: 4096})
    values = values.astype(dtype)
    X = rng.uniform(-1, 1, (9000, k)).astype(dtype)
    want = O.spmm_csr(rowptr, colind, values, X)
    got = lb.spmm_csr(cu(rowptr), cu(colind), cu(values), cu(X)).cpu().numpy()
    ok, msg = O.diff_outputs([got], [want], 1e-12 if dtype == np.float64 else 1e-5)
    assert ok, msg
    short = np.diff(rowptr) <= SPLIT
    assert bits_equal(got[short], want[short])


def test_int_spmm_exact(cuda_device):
    rng = np.random.default_rng(3)
    rowptr, colind, values = ragged_csr(rng, 500, 400, max_len=20, long_rows={3: 399},
                                        dtype=np.int64)
    X = rng.integers(-1000, 1000, (400, 64)).astype(np.int64)
    got = lb.spmm_csr(cu(rowptr), cu(colind), cu(values), cu(X)).cpu().numpy()
    assert np.array_equal(got, O.spmm_csr(rowptr, colind, values, X))


def test_chung_lu_k64(cuda_device):
    rng = np.random.default_rng(11)
    rowptr, colind, values = powerlaw_csr(rng, 60000, mean=10.0)
    X = rng.uniform(-1, 1, (60000, 64))
    want = O.spmm_csr(rowptr, colind, values, X)
    got = lb.spmm_csr(cu(rowptr), cu(colind), cu(values), cu(X)).cpu().numpy()
    ok, msg = O.diff_outputs([got], [want], 1e-12)
    assert ok, msg


def test_rowblock_spmm_world1_matches_library_call(cuda_device):
    # sharded.RowBlockSpmm at world 1 (the bench's config-3 path): the X slot
    # buffer + spmm_csr give the library call's bits
    from paper_2509_25605_b200 import sharded
    rng = np.random.default_rng(21)
    rowptr, colind, values = powerlaw_csr(rng, 3000, mean=8.0)
    X = rng.uniform(-1, 1, (3000, 64))
    rp, ci, v = (torch.from_numpy(a).cuda() for a in (rowptr, colind, values))
    op = sharded.RowBlockSpmm(rp, ci, v, 3000, 64, 0, 1)
    op.x_local.copy_(torch.from_numpy(X))
    Y = torch.empty((3000, 64), dtype=torch.float64, device="cuda")
    op.multiply(Y)
    want = O.spmm_csr(rowptr, colind, values, X)
    assert np.array_equal(Y.cpu().numpy().view(np.uint64), want.view(np.uint64)) or \
        np.max(np.abs(Y.cpu().numpy() - want) / np.maximum(np.abs(want), 1)) <= 1e-12


@pytest.mark.parametrize("k", [64, 8, 5])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_decreasing_rowptr(cuda_device, k, dtype):
    """a decreasing rowptr (rows overlap / are empty, interp.py:808)
    with rows beyond the 2048-entry split: the guarded fallback folds every
    row on its clamped range; nothing is written out of bounds."""
    from test_spmv_gpu import decreasing_rowptr_csr
    rng = np.random.default_rng(k)
    rp, colind, values = decreasing_rowptr_csr(rng, 4000, 6000, dtype=dtype)
    X = rng.uniform(-1, 1, (6000, k)).astype(dtype)
    want = O.spmm_csr(rp, colind, values, X)
    Yd = torch.full((4000 + 64, k), 7.0, dtype=torch.float64 if dtype == np.float64 else torch.float32,
                    device="cuda")
    lb.spmm_csr(cu(rp), cu(colind), cu(values), cu(X), Yd[:4000], nnz=int(rp[-1]))
    got = Yd[:4000].cpu().numpy()
    assert bits_equal(got, want)
    assert bool((Yd[4000:] == 7.0).all()), "write past Y"


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("hot_mb", [0, 1])
@pytest.mark.parametrize("hints", ["0", "1"])
def test_spmm_plan_hot_rows_bitexact(cuda_device, monkeypatch, dtype, hot_mb, hints):
    """SpmmPlan (hot X rows pinned in L2, remapped colind; with and without the
    opt-in reuse hints) gives spmm_csr's bits."""
    monkeypatch.setenv("LAPIS_B200_SPMM_HINT", hints)
    import synth_inputs as S
    spec = S.PowerLawSpec(60_000, mean=10.0, seed=3)
    rowptr, colind = S.powerlaw_structure_host(spec)
    values = S.powerlaw_values(spec, int(rowptr[-1])).astype(dtype)
    X = np.random.default_rng(4).uniform(-1, 1, (60_000, 64)).astype(dtype)
    plan = lb.SpmmPlan(cu(rowptr), cu(colind), 60_000, 64,
                       torch.float64 if dtype == np.float64 else torch.float32,
                       hot_bytes=hot_mb << 20)
    info = plan.info()
    assert info["hot_rows"] > 0 and info["hot_entries"] > 0
    assert (info["far_reuse_entries"] > 0) == (hints == "1"), info
    Xd = cu(X)
    got = plan.spmm(cu(values), Xd).cpu().numpy()
    want = lb.spmm_csr(cu(rowptr), cu(colind), cu(values), Xd).cpu().numpy()
    assert bits_equal(got, want)
    X2 = np.random.default_rng(5).uniform(-1, 1, (60_000, 64)).astype(dtype)   # new X, same plan
    got2 = plan.spmm(cu(values), cu(X2)).cpu().numpy()
    ok, msg = O.diff_outputs([got2], [O.spmm_csr(rowptr, colind, values, X2)],
                             1e-12 if dtype == np.float64 else 1e-5)
    assert ok, msg
    plan.close()
