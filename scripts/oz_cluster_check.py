"""fp64 AUTO GEMM (certified Ozaki, two-pass kernel) with and without the
2-CTA cluster B multicast: max |C - C_ref| / max(|C_ref|, 1) on a few shapes
and the 4096^3 time."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2509_25605_b200 as lb  # noqa: E402

for (m, n, k) in ((256, 128, 64), (256, 256, 256), (512, 384, 640), (384, 256, 100), (1024, 1024, 1024)):
    rng = np.random.default_rng(m + n + k)
    A = torch.from_numpy(rng.uniform(-1, 1, (m, k))).cuda()
    B = torch.from_numpy(rng.uniform(-1, 1, (k, n))).cuda()
    C = lb.gemm(A, B)
    ref = A @ B
    err = ((C - ref).abs() / ref.abs().clamp_min(1.0)).max().item()
    print(f"{m}x{n}x{k}: max rel err {err:.2e}", flush=True)
n = 4096
A = torch.rand(n, n, dtype=torch.float64, device="cuda") * 2 - 1
B = torch.rand(n, n, dtype=torch.float64, device="cuda") * 2 - 1
C = lb.gemm(A, B)
for _ in range(3):
    lb.gemm(A, B, C)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    lb.gemm(A, B, C)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
ref = A @ B
err = ((C - ref).abs() / ref.abs().clamp_min(1.0)).max().item()
print(f"4096^3: {ms:.3f} ms {2 * n ** 3 / ms / 1e9:.1f} TF/s max rel err {err:.2e}")
