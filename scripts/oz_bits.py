"""Dump Ozaki GEMM outputs for a few seeded shapes (bitwise A/B of builds)."""
import sys
import numpy as np
import torch
from paper_2509_25605_b200 import kernels

out = {}
for (m, n, k, dt) in [(4096, 4096, 4096, torch.float64), (1000, 777, 1500, torch.float64),
                      (513, 300, 700, torch.float32), (2048, 2048, 2048, torch.float32)]:
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    A = (torch.rand(m, k, generator=g, device="cuda", dtype=torch.float64) * 2 - 1).to(dt)
    B = (torch.rand(k, n, generator=g, device="cuda", dtype=torch.float64)).to(dt)
    C = kernels.gemm(A, B, mode="ozaki")
    out[f"{m}x{n}x{k}_{dt}"] = C.cpu().numpy()
np.savez(sys.argv[1], **out)
