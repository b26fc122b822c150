"""Ozaki GEMM with the m-pairs on cta_group::2 MMAs (LAPIS_B200_OZAKI_PAIR=1)
against the per-CTA kernel: errors on a few shapes (fp64 and fp32 AUTO) and
the 4096^3 times.  One process per setting: python scripts/oz_pair_check.py"""
import os
import subprocess
import sys

if len(sys.argv) > 1:
    import torch
    sys.path.insert(0, ".")
    import paper_2509_25605_b200 as lb  # noqa: E402
    import numpy as np
    tag = sys.argv[1]
    for dt in (torch.float64, torch.float32):
        for (m, n, k) in ((256, 128, 64), (256, 256, 256), (512, 384, 640), (384, 256, 100),
                          (1024, 1024, 1024), (2048, 1024, 4096)):
            rng = np.random.default_rng(m + n + k)
            A = torch.from_numpy(rng.uniform(-1, 1, (m, k))).to(dt).cuda()
            B = torch.from_numpy(rng.uniform(-1, 1, (k, n))).to(dt).cuda()
            C = lb.gemm(A, B)
            ref = A.double() @ B.double()
            err = ((C.double() - ref).abs() / ref.abs().clamp_min(1.0)).max().item()
            print(f"{tag} {dt} {m}x{n}x{k}: max rel err {err:.2e}", flush=True)
        N = 4096
        A = (torch.rand(N, N, dtype=torch.float64, device="cuda") * 2 - 1).to(dt)
        B = (torch.rand(N, N, dtype=torch.float64, device="cuda") * 2 - 1).to(dt)
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
        print(f"{tag} {dt} 4096^3: {ms:.3f} ms {2 * N ** 3 / ms / 1e9:.1f} TF/s max rel err {err:.2e}",
              flush=True)
else:
    for pair in ("0", "1"):
        r = subprocess.run(["timeout", "180", sys.executable, __file__, f"pair={pair}"],
                           env={**os.environ, "LAPIS_B200_OZAKI_PAIR": pair})
        print(f"pair={pair} rc={r.returncode}", flush=True)
