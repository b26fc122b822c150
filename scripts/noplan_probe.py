"""The no-plan C-ABI SpMV (lapis_b200_spmv_csr, vector_length 0: the emitted
C++'s LAPIS::spmv_csr path) vs a plan, on the config-5 stencil and the
config-3 power-law matrix."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2509_25605_b200 as lb  # noqa: E402


def timeit(f, reps=10):
    for _ in range(3):
        f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


for name, (rp, ci, v) in (("c5 stencil", lb.synth_stencil(27, 585)),
                          ("c3 power-law", bench.powerlaw_csr_device(10_000_000, 10.0, 2.5, 1))):
    n = rp.numel() - 1
    nnz = int(rp[-1].item())
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y1 = torch.empty(n, dtype=torch.float64, device="cuda")
    y2 = torch.empty_like(y1)
    work = nnz * 12 + (n + 1) * 8 + 2 * n * 8
    t0 = timeit(lambda: lb.spmv_csr(rp, ci, v, x, y1, nnz=nnz))
    plan = lb.CsrPlan(rp)
    t1 = timeit(lambda: plan.spmv(ci, v, x, y2))
    print(f"{name}: no-plan {t0 * 1e3:.3f} ms ({work / t0 / 1e9:.0f} GB/s), plan "
          f"{t1 * 1e3:.3f} ms ({work / t1 / 1e9:.0f} GB/s) [{plan.info()['kernel']}], "
          f"max|diff| {float((y1 - y2).abs().max()):.3g}", flush=True)
    del rp, ci, v, x, y1, y2, plan
    torch.cuda.empty_cache()
