"""Config 4: the GCN layer relu((A_hat X) W) against the reference interpreter
(fixture gcn_small from oracle/ir/gcn_f32.mlir) and the oracle on a power-law
graph with hub rows: bit-identical (both stages follow the reference order)."""
import numpy as np
import pytest
import torch

import paper_2509_25605_b200 as lb
from conftest import bits_equal, load_golden
from matrices import ragged_csr
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_golden_gcn_bitexact(cuda_device):
    g = load_golden("gcn_small")
    rowptr, colind, values, X, W, _ = g["inputs"]
    H = lb.gcn_layer(cu(rowptr), cu(colind), cu(values), cu(X), cu(W)).cpu().numpy()
    assert bits_equal(H, g["outputs"][0])


@pytest.mark.parametrize("fin,fout", [(64, 64), (16, 40), (3, 8)])
def test_gcn_hub_rows_bitexact(cuda_device, fin, fout):
    rng = np.random.default_rng(fin * fout)
    rowptr, colind, values = ragged_csr(rng, 3000, 5000, max_len=20, empty_every=17,
                                        long_rows={4: 4999, 2000: 2600, 2999: 3000},
                                        dtype=np.float32)
    values = np.abs(values)
    X = rng.uniform(0, 1, (5000, fin)).astype(np.float32)
    W = rng.uniform(-1 / 8, 1 / 8, (fin, fout)).astype(np.float32)
    H = lb.gcn_layer(cu(rowptr), cu(colind), cu(values), cu(X), cu(W)).cpu().numpy()
    assert bits_equal(H, O.gcn(rowptr, colind, values, X, W))


@pytest.mark.parametrize("fused", ["0", "1"])
def test_gcn_fused_and_two_stage_bitexact(cuda_device, monkeypatch, fused):
    # fin = fout = 64 fp32: the fused single-pass kernel (opt-in) and the
    # two-stage default give the reference's bits, hub rows included
    monkeypatch.setenv("LAPIS_B200_GCN_FUSED", fused)
    rng = np.random.default_rng(11)
    rowptr, colind, values = ragged_csr(rng, 4100, 6000, max_len=30, empty_every=13,
                                        long_rows={0: 5999, 77: 2049, 4099: 4000},
                                        dtype=np.float32)
    values = np.abs(values)
    X = rng.uniform(0, 1, (6000, 64)).astype(np.float32)
    W = rng.uniform(-1 / 8, 1 / 8, (64, 64)).astype(np.float32)
    H = lb.gcn_layer(cu(rowptr), cu(colind), cu(values), cu(X), cu(W)).cpu().numpy()
    assert bits_equal(H, O.gcn(rowptr, colind, values, X, W))
