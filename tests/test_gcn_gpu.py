"""Config 4: the GCN layer relu((A_hat X) W) against the reference interpreter
(fixture gcn_small from oracle/ir/gcn_f32.mlir) and the oracle on power-law
graphs with hub rows.  EXACT mode: bit-identical (both stages follow the
reference order).  AUTO mode (the default): the SpMM stage is still the
reference's order, the dense stage + ReLU runs on the tcgen05 tensor cores
(3xTF32, csrc/gcn_dense.cu) — within the fp32 contract, 1e-5 under
diff_outputs (interp.py:1050-1071)."""
import numpy as np
import pytest
import torch

import paper_2509_25605_b200 as lb
from conftest import bits_equal, load_golden
from matrices import ragged_csr
from oracle import oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-5


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_golden_gcn(cuda_device):
    g = load_golden("gcn_small")
    rowptr, colind, values, X, W, _ = g["inputs"]
    H = lb.gcn_layer(cu(rowptr), cu(colind), cu(values), cu(X), cu(W), exact=True).cpu().numpy()
    assert bits_equal(H, g["outputs"][0])
    H = lb.gcn_layer(cu(rowptr), cu(colind), cu(values), cu(X), cu(W)).cpu().numpy()
    ok, msg = O.diff_outputs([H], [g["outputs"][0]], TOL)
    assert ok, msg


@pytest.mark.parametrize("fin,fout", [(64, 64), (64, 32), (16, 40), (3, 8)])
def test_gcn_hub_rows(cuda_device, fin, fout):
    rng = np.random.default_rng(fin * fout)
    rowptr, colind, values = ragged_csr(rng, 3000, 5000, max_len=20, empty_every=17,
                                        long_rows={4: 4999, 2000: 2600, 2999: 3000},
                                        dtype=np.float32)
    values = np.abs(values)
    X = rng.uniform(0, 1, (5000, fin)).astype(np.float32)
    W = rng.uniform(-1 / 8, 1 / 8, (fin, fout)).astype(np.float32)
    want = O.gcn(rowptr, colind, values, X, W)
    H = lb.gcn_layer(cu(rowptr), cu(colind), cu(values), cu(X), cu(W), exact=True).cpu().numpy()
    assert bits_equal(H, want)
    H = lb.gcn_layer(cu(rowptr), cu(colind), cu(values), cu(X), cu(W)).cpu().numpy()
    ok, msg = O.diff_outputs([H], [want], TOL)
    assert ok, msg
    assert ((H == 0) == (want == 0)).mean() > 0.999   # the ReLU zeros land where the reference's do


@pytest.mark.parametrize("nrows", [1, 127, 128, 129, 1000, 70001])
def test_gcn_tensor_core_stage_tails(cuda_device, nrows):
    """M tails of the 128-row tiles, a single row, negative inputs (ReLU)."""
    rng = np.random.default_rng(nrows)
    rowptr, colind, values = ragged_csr(rng, nrows, 300, max_len=12, dtype=np.float32)
    X = rng.uniform(-1, 1, (300, 64)).astype(np.float32)
    W = rng.uniform(-1 / 8, 1 / 8, (64, 64)).astype(np.float32)
    want = O.gcn(rowptr, colind, values, X, W)
    H = torch.full((nrows + 5, 64), 3.0, device="cuda")
    lb.gcn_layer(cu(rowptr), cu(colind), cu(values), cu(X), cu(W), H[:nrows])
    got = H[:nrows].cpu().numpy()
    ok, msg = O.diff_outputs([got], [want], TOL)
    assert ok, msg
    assert bool((H[nrows:] == 3.0).all()), "tensor-core stage wrote past H"


@pytest.mark.parametrize("fused", ["0", "1"])
def test_gcn_fused_and_two_stage_exact(cuda_device, monkeypatch, fused):
    # fin = fout = 64 fp32 in EXACT mode: the fused single-pass kernel (opt-in)
    # and the two-stage default give the reference's bits, hub rows included
    monkeypatch.setenv("LAPIS_B200_GCN_FUSED", fused)
    rng = np.random.default_rng(11)
    rowptr, colind, values = ragged_csr(rng, 4100, 6000, max_len=30, empty_every=13,
                                        long_rows={0: 5999, 77: 2049, 4099: 4000},
                                        dtype=np.float32)
    values = np.abs(values)
    X = rng.uniform(0, 1, (6000, 64)).astype(np.float32)
    W = rng.uniform(-1 / 8, 1 / 8, (64, 64)).astype(np.float32)
    H = lb.gcn_layer(cu(rowptr), cu(colind), cu(values), cu(X), cu(W), exact=True).cpu().numpy()
    assert bits_equal(H, O.gcn(rowptr, colind, values, X, W))
