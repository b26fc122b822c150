"""StreamedSpmv: the overlapped host-vector SpMV gives the exact-mode plan
result bit for bit (chunk plans may pick other kernels in the default mode:
within the fp64 tolerance) and keeps the DualView transfer semantics."""
import numpy as np
import pytest
import torch

from matrices import powerlaw_csr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("banded", [True, False])
@pytest.mark.parametrize("chunks", [1, 5, 16])
def test_streamed_matches_plan(banded, chunks, exact, cuda_device):
    import paper_2509_25605_b200 as lb
    from paper_2509_25605_b200.dualview import DualView, reset_transfer_stats, transfer_stats
    from paper_2509_25605_b200.streamed import StreamedSpmv
    if banded:
        rowptr, colind, values = lb.synth_stencil(27, 14)
        n = 14 ** 3
    else:
        rp, ci, v = powerlaw_csr(np.random.default_rng(3), 3000)
        rowptr, colind, values = (torch.from_numpy(a).to(cuda_device) for a in (rp, ci, v))
        n = 3000
    x = np.random.default_rng(1).uniform(-1, 1, n)
    want = lb.CsrPlan(rowptr, exact=True).spmv(colind, values,
                                               torch.from_numpy(x).to(cuda_device)).cpu()
    op = StreamedSpmv(rowptr, colind, values, n, chunks=chunks, exact=exact or None)
    xs = DualView.from_host(x, "x")
    ys = DualView.allocate((rowptr.numel() - 1,), torch.float64, "y")
    reset_transfer_stats()
    for _ in range(2):
        xs.modify_host()
        op.multiply(xs, ys)
        got = ys.host_view()
        if exact:
            assert torch.equal(got, want)
        else:
            err = ((got - want).abs() / torch.clamp(torch.maximum(got.abs(), want.abs()), min=1.0))
            assert float(err.max()) <= 1e-12
    st = transfer_stats()
    assert (st.h2d_count, st.d2h_count) == (2, 2)
    assert not xs.host_modified() and not ys.device_modified()
