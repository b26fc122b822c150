"""Parity at the BASELINE configs' own sizes, on the inputs the
bench measures (synth_inputs.py), against the C oracle (interp.py restated):

* config 2: dense matmul 4096^3 in AUTO mode — f32 (3xTF32, U(0,1) seed 3) and
  f64 (certified Ozaki, U(-1,1) seed 2) — on 8192 sampled entries
  (interp.py:711-722, 1e-5 / 1e-12 under diff_outputs);
* config 3: the power-law matrix's 117,683-entry hub row at K = 64, fp64 and
  fp32 (within tolerance: the hub is folded in fixed chunks for fp64, in the
  reference order for fp32), and a sample of short rows (<= 2048 entries)
  bit-exact;
* config 5: the full 200M-row 27-point stencil in tree mode on three row
  windows — the first plane, the middle and the last plane — within 1e-12
  (interp.py:798-812).
"""
import numpy as np
import pytest
import torch

import paper_2509_25605_b200 as lb
import synth_inputs as S
from conftest import bits_equal
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dt,seed,tol", [(np.float32, 3, 1e-5), (np.float64, 2, 1e-12)])
def test_config2_matmul_4096_auto(cuda_device, dt, seed, tol):
    n = 4096
    A, B = S.dense_operands(n, dt, seed)
    C = lb.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), mode="auto")
    rng = np.random.default_rng(0)
    ii = rng.integers(0, n, 8192)
    jj = rng.integers(0, n, 8192)
    ii[:64], jj[:64] = np.arange(64), n - 1 - np.arange(64)       # corners of the tiles too
    want = O.matmul_entries(A, B, ii, jj)
    got = C[torch.from_numpy(ii).cuda(), torch.from_numpy(jj).cuda()].cpu().numpy()
    ok, msg = O.diff_outputs([got], [want], tol)
    assert ok, msg


@pytest.fixture(scope="module")
def config3_matrix(cuda_device):
    spec = S.PowerLawSpec(10_000_000, seed=1)
    rowptr, colind = S.powerlaw_structure_device(spec)
    nnz = int(rowptr[-1].item())
    values = S.powerlaw_values(spec, nnz)
    X = S.spmm_dense(10_000_000, 64, 1)
    return spec, rowptr, colind, values, X


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_config3_hub_row_k64(config3_matrix, dt):
    spec, rowptr, colind, values, X = config3_matrix
    tdt = torch.float64 if dt == np.float64 else torch.float32
    Xd = torch.from_numpy(X.astype(dt)).cuda()
    vd = torch.from_numpy(values.astype(dt)).cuda()
    Y = lb.spmm_csr(rowptr, colind, vd, Xd)
    rp = rowptr.cpu().numpy()
    L = np.diff(rp)
    hub = int(L.argmax())
    assert L[hub] == 117_683
    rng = np.random.default_rng(1)
    short = rng.choice(np.flatnonzero(L <= 2048), 2000, replace=False)
    long_rows = np.flatnonzero(L > 2048)
    rows = np.unique(np.concatenate([[hub], short, long_rows[:50]]))
    # the sampled rows as their own CSR (same entries, same order)
    ci = colind.cpu().numpy()
    sub_rp = np.zeros(rows.size + 1, dtype=np.int64)
    sub_rp[1:] = np.cumsum(L[rows])
    idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
    want = O.spmm_csr(sub_rp, ci[idx], values.astype(dt)[idx], X.astype(dt))
    got = Y[torch.from_numpy(rows).cuda()].cpu().numpy()
    ok, msg = O.diff_outputs([got], [want], 1e-12 if dt == np.float64 else 1e-5)
    assert ok, msg
    is_short = L[rows] <= 2048
    assert bits_equal(got[is_short], want[is_short])
    if dt == np.float32:    # fp32 hub rows are folded in the reference order
        assert bits_equal(got, want)
    del Y, Xd, vd
    torch.cuda.empty_cache()


def test_config5_full_size_windows(cuda_device):
    n = 585
    N = n ** 3
    rowptr, colind, values = lb.synth_stencil(27, n)
    x = S.stencil_x(27, n, 5)
    y = lb.CsrPlan(rowptr).spmv(colind, values, torch.from_numpy(x).cuda())
    plane = n * n
    for a, b in ((0, plane), (N // 2 - plane // 2, N // 2 + plane // 2), (N - plane, N)):
        rp, ci, v = S.stencil_rows(27, n, a, b)
        want = O.spmv_csr(rp, ci, v, x)
        got = y[a:b].cpu().numpy()
        ok, msg = O.diff_outputs([got], [want], 1e-12)
        assert ok, (a, b, msg)
        # the device-built structure is the host formula's, bit for bit
        assert np.array_equal(rowptr[a:b + 1].cpu().numpy() - int(rowptr[a].item()), rp)
    del rowptr, colind, values, y
    torch.cuda.empty_cache()
