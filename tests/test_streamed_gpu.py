"""StreamedSpmv: the overlapped host-vector SpMV gives the plan kernels'
result bit for bit and keeps the DualView transfer semantics."""
import numpy as np
import pytest
import torch

from matrices import powerlaw_csr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("banded", [True, False])
@pytest.mark.parametrize("chunks", [1, 5, 16])
def test_streamed_matches_plan(banded, chunks, cuda_device):
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
    want = lb.CsrPlan(rowptr).spmv(colind, values, torch.from_numpy(x).to(cuda_device)).cpu()
    op = StreamedSpmv(rowptr, colind, values, n, chunks=chunks)
    xs = DualView.from_host(x, "x")
    ys = DualView.allocate((rowptr.numel() - 1,), torch.float64, "y")
    reset_transfer_stats()
    for _ in range(2):
        xs.modify_host()
        op.multiply(xs, ys)
        assert torch.equal(ys.host_view(), want)
    st = transfer_stats()
    assert (st.h2d_count, st.d2h_count) == (2, 2)
    assert not xs.host_modified() and not ys.device_modified()
