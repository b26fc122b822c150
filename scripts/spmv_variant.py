"""Run one SpMV variant on a 27-point (or 5-point) stencil for ncu captures and
quick timing.  usage: python scripts/spmv_variant.py MODE [n] [points]
MODE: tree | exact   (kernel variants via the LAPIS_B200_* environment)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_25605_b200 as lb  # noqa: E402

mode = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 300
points = int(sys.argv[3]) if len(sys.argv) > 3 else 27
rp, ci, v = lb.synth_stencil(points, n)
N = rp.numel() - 1
x = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, N)).cuda()
plan = lb.CsrPlan(rp, exact=(mode == "exact"))
y = torch.empty(N, dtype=torch.float64, device="cuda")
for _ in range(3):
    plan.spmv(ci, v, x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    plan.spmv(ci, v, x, y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
nnz = int(rp[-1].item())
byts = nnz * 12 + (N + 1) * 8 + 2 * N * 8
print(f"{mode} {plan.info()['kernel']}: {ms:.3f} ms {byts / ms / 1e6:.1f} GB/s")
