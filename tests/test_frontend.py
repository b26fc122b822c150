"""The torch.fx frontend (paper_2509_25605_b200/frontend.py): small sparse
models — the config-4 GCN layer (torch.sparse.mm -> nn.Linear -> relu), an
SpMV (torch.mv on a CSR tensor), a two-layer GCN, a dense chain — lowered to
LAPIS IR, parsed and lowered by the reference's own pipeline, and run by the
reference interpreter: equal to the eager PyTorch module (fp32 1e-5, fp64
1e-12 under diff_outputs), and the lowered program equal to the unlowered one
bit for bit (the reference's preservation property, test_acceptance.py:38-79).
On the GPU the same programs run through runtime.run (the B200 drop-in)."""
import numpy as np
import pytest
import torch

pytest.importorskip("lapis.parser")
from lapis.interp import diff_outputs, run as interp_run  # noqa: E402
from lapis.parser import parse  # noqa: E402

from paper_2509_25605_b200 import frontend as F  # noqa: E402


class GCN(torch.nn.Module):
    def __init__(self, fin, fout):
        super().__init__()
        self.lin = torch.nn.Linear(fin, fout, bias=False)

    def forward(self, A, X):
        return torch.relu(self.lin(torch.sparse.mm(A, X)))


class GCN2(torch.nn.Module):
    def __init__(self, f):
        super().__init__()
        self.l1 = torch.nn.Linear(f, f, bias=False)
        self.l2 = torch.nn.Linear(f, 4, bias=False)
        self.act = torch.nn.ReLU()

    def forward(self, A, X):
        h = self.act(self.l1(torch.sparse.mm(A, X)))
        return torch.nn.functional.relu(self.l2(A @ h))


class SpMV(torch.nn.Module):
    def forward(self, A, x):
        return torch.mv(A, x)


class DenseChain(torch.nn.Module):
    def __init__(self):
        super().__init__()
        self.w = torch.nn.Parameter(torch.randn(6, 5, dtype=torch.float64))

    def forward(self, X):
        return torch.relu(torch.mm(X, self.w))


def _graph(n, dtype, seed=0, p=0.15):
    g = torch.Generator().manual_seed(seed)
    mask = torch.rand(n, n, generator=g) < p
    A = torch.where(mask, torch.rand(n, n, generator=g, dtype=dtype), torch.zeros((), dtype=dtype))
    return A.to_sparse_csr()


MODELS = [
    ("gcn", lambda: GCN(8, 5), lambda: (_graph(40, torch.float32), torch.rand(40, 8)), 1e-5),
    ("gcn2", lambda: GCN2(6), lambda: (_graph(33, torch.float32, 1), torch.rand(33, 6)), 1e-5),
    ("spmv", SpMV, lambda: (_graph(50, torch.float64, 2), torch.rand(50, dtype=torch.float64)),
     1e-12),
    ("dense", DenseChain, lambda: (torch.randn(7, 6, dtype=torch.float64),), 1e-12),
]


@pytest.mark.parametrize("name,make,data,tol", MODELS, ids=[m[0] for m in MODELS])
def test_frontend_matches_eager_and_preserves(name, make, data, tol):
    torch.manual_seed(0)
    m = make()
    args = data()
    low = F.lower_module(m, *args)
    inputs = low.inputs(*args)
    want = m(*args).detach().numpy()
    raw = interp_run(parse(low.text), low.entry, [a.copy() for a in inputs])
    rep = diff_outputs([np.asarray(raw.outputs[0])], [want], rel_tol=tol)
    assert rep.match, str(rep)
    got, _ = F.run_module(m, *args, backend="interp")
    assert np.array_equal(np.asarray(got), np.asarray(raw.outputs[0]))   # lowering preserves bits


def test_frontend_rejects_unsupported_ops():
    class Bad(torch.nn.Module):
        def forward(self, A, X):
            return torch.sigmoid(torch.sparse.mm(A, X))
    with pytest.raises(F.FrontendError):
        F.lower_module(Bad(), _graph(10, torch.float32), torch.rand(10, 3))
    with pytest.raises(F.FrontendError):
        F.lower_module(torch.nn.Linear(3, 3, bias=True), torch.rand(4, 3))


@pytest.mark.gpu
@pytest.mark.parametrize("name,make,data,tol", MODELS, ids=[m[0] for m in MODELS])
def test_frontend_on_b200_matches_interpreter(name, make, data, tol, cuda_device):
    torch.manual_seed(0)
    m = make()
    args = data()
    ref, rres = F.run_module(m, *args, backend="interp")
    got, gres = F.run_module(m, *args, backend="b200")
    rep = diff_outputs([got], [ref], rel_tol=tol)
    assert rep.match, str(rep)
    from lapis.interp import format_trace
    assert format_trace(gres.trace) == format_trace(rres.trace)
