"""Accuracy of the 3xTF32 GEMM with the rounded head (default) or the raw fp32
head (LAPIS_B200_TF32_RAWHI=1: the tensor core reads the TF32 bits, the tail
is a - trunc(a)): max |C - C64| / max(|C64|, 1) over full matrices."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_25605_b200 as lb  # noqa: E402

for n, lo in ((1024, 0.0), (4096, 0.0), (4096, -1.0), (2048, -1.0)):
    rng = np.random.default_rng(n)
    A = rng.uniform(lo, 1, (n, n)).astype(np.float32)
    B = rng.uniform(lo, 1, (n, n)).astype(np.float32)
    ref = torch.from_numpy(A).double().cuda() @ torch.from_numpy(B).double().cuda()
    C = lb.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), mode="tf32x3").double()
    err = ((C - ref).abs() / ref.abs().clamp_min(1.0)).max().item()
    print(f"n={n} U({lo},1): max rel err {err:.3e}")
