"""AUTO f32 GEMM at 4096^3: U(0,1) operands (config 2, the sign-gated Ozaki
path) and U(-1,1) operands (the gate sends them to 3xTF32): time per call and
max |C - C64| / max(|C64|, 1)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2509_25605_b200 as lb  # noqa: E402

n = 4096
for lo in (0.0, -1.0):
    rng = np.random.default_rng(3)
    A = torch.from_numpy(rng.uniform(lo, 1, (n, n)).astype(np.float32)).cuda()
    B = torch.from_numpy(rng.uniform(lo, 1, (n, n)).astype(np.float32)).cuda()
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
    ref = A.double() @ B.double()
    err = ((C.double() - ref).abs() / ref.abs().clamp_min(1.0)).max().item()
    print(f"U({lo},1): {ms:.3f} ms  {2 * n ** 3 / ms / 1e9:.1f} TF/s  max rel err {err:.2e}")
