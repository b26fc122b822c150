"""PyTorch / DLPack interop of the C-ABI wrappers (SURVEY 8(b) "Python
zero-copy"): a CUDA torch.sparse_csr_tensor goes straight
into spmv_csr / spmm_csr / gcn_layer / CsrPlan (crow / col / values used in
place), and any DLPack producer is accepted for every operand — including
outputs, which are written in place."""
import numpy as np
import pytest
import torch

import paper_2509_25605_b200 as lb
from conftest import bits_equal
from matrices import powerlaw_csr
from oracle import oracle as O

pytestmark = pytest.mark.gpu


class Capsule:
    """A foreign DLPack producer (what CuPy / JAX arrays look like to us)."""

    def __init__(self, t):
        self.t = t

    def __dlpack__(self, stream=None, **kw):
        return self.t.__dlpack__(stream=stream) if stream is not None else self.t.__dlpack__()

    def __dlpack_device__(self):
        return self.t.__dlpack_device__()


def _csr(seed=3, n=4000):
    rng = np.random.default_rng(seed)
    rowptr, colind, values = powerlaw_csr(rng, n, mean=9.0)
    return rng, rowptr, colind, values


def test_sparse_csr_tensor_spmv_spmm(cuda_device):
    rng, rowptr, colind, values = _csr()
    n = rowptr.size - 1
    A = torch.sparse_csr_tensor(torch.from_numpy(rowptr), torch.from_numpy(colind.astype(np.int64)),
                                torch.from_numpy(values), size=(n, n)).cuda()
    x = rng.uniform(-1, 1, n)
    y = lb.spmv_csr(A, torch.from_numpy(x).cuda()).cpu().numpy()
    ok, msg = O.diff_outputs([y], [O.spmv_csr(rowptr, colind, values, x)], 1e-12)
    assert ok, msg
    plan = lb.CsrPlan(A, exact=True)
    y2 = plan.spmv(A.col_indices(), A.values(), torch.from_numpy(x).cuda()).cpu().numpy()
    assert bits_equal(y2, O.spmv_csr(rowptr, colind, values, x))
    X = rng.uniform(-1, 1, (n, 16))
    Y = torch.empty((n, 16), dtype=torch.float64, device="cuda")
    out = lb.spmm_csr(A, torch.from_numpy(X).cuda(), Y)
    assert out.data_ptr() == Y.data_ptr()
    ok, msg = O.diff_outputs([Y.cpu().numpy()], [O.spmm_csr(rowptr, colind, values, X)], 1e-12)
    assert ok, msg


def test_dlpack_producers_in_and_out(cuda_device):
    rng, rowptr, colind, values = _csr(5, 3000)
    n = rowptr.size - 1
    x = rng.uniform(-1, 1, n)
    args = [Capsule(torch.from_numpy(a).cuda()) for a in (rowptr, colind, values, x)]
    ybuf = torch.zeros(n, dtype=torch.float64, device="cuda")
    lb.spmv_csr(*args, Capsule(ybuf))
    ok, msg = O.diff_outputs([ybuf.cpu().numpy()], [O.spmv_csr(rowptr, colind, values, x)], 1e-12)
    assert ok, msg   # the kernel wrote into the producer's memory
    A = rng.uniform(-1, 1, (70, 50))
    B = rng.uniform(-1, 1, (50, 30))
    C = torch.empty((70, 30), dtype=torch.float64, device="cuda")
    lb.gemm(Capsule(torch.from_numpy(A).cuda()), Capsule(torch.from_numpy(B).cuda()), Capsule(C),
            mode="exact")
    assert bits_equal(C.cpu().numpy(), O.matmul(A, B))


def test_gcn_layer_from_sparse_tensor(cuda_device):
    rng, rowptr, colind, values = _csr(7, 2000)
    n = rowptr.size - 1
    vf = np.abs(values).astype(np.float32)
    A = torch.sparse_csr_tensor(torch.from_numpy(rowptr), torch.from_numpy(colind.astype(np.int64)),
                                torch.from_numpy(vf), size=(n, n)).cuda()
    X = rng.uniform(0, 1, (n, 64)).astype(np.float32)
    W = rng.uniform(-1 / 8, 1 / 8, (64, 64)).astype(np.float32)
    H = lb.gcn_layer(A, None, None, torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda(),
                     exact=True).cpu().numpy()
    assert bits_equal(H, O.gcn(rowptr, colind, vf, X, W))
