"""SpMV on the config-3 power-law matrix (10M rows, ~100M nnz): the plan's
default kernel vs the forced warp-block kernel (A/B for the irregular path)."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2509_25605_b200 as lb  # noqa: E402

rp, ci, v = bench.powerlaw_csr_device(10_000_000, 10.0, 2.5, 1)
n = rp.numel() - 1
nnz = int(rp[-1].item())
x = torch.rand(n, dtype=torch.float64, device="cuda")
work = nnz * 12 + (n + 1) * 8 + 2 * n * 8
res = {}
for mode in ["default", "wb"]:
    if mode == "wb":
        os.environ["LAPIS_B200_SPMV_KERNEL"] = "wb"
    plan = lb.CsrPlan(rp)
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        plan.spmv(ci, v, x, y)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(20):
        plan.spmv(ci, v, x, y)
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 20 / 1e3
    res[mode] = y.clone()
    print(mode, plan.info()["kernel"], f"{t * 1e3:.3f} ms  {work / t / 1e9:.0f} GB/s", flush=True)
d = (res["default"] - res["wb"]).abs().max().item()
print("max |diff|", d)
