"""matvec (LAPIS::gemv) and axis-1 reduce throughput at 16384 x 16384 (f64, f32)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2509_25605_b200 as lb  # noqa: E402

for dt in (torch.float64, torch.float32):
    m = n = 16384
    A = torch.rand((m, n), dtype=dt, device="cuda")
    x = torch.rand(n, dtype=dt, device="cuda")
    y = torch.empty(m, dtype=dt, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name, f in (("gemv", lambda: lb.gemv(A, x, y)), ("reduce_add", lambda: lb.reduce2d(A, 1, "add", y))):
        for _ in range(3):
            f()
        ts = []
        for _ in range(10):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); f(); b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        t = sum(a.elapsed_time(b) for a, b in ts) / len(ts) / 1e3
        byts = A.numel() * A.element_size() + (n + m) * A.element_size()
        print(f"{name} {dt} {m}x{n}: {t * 1e3:.3f} ms {byts / t / 1e9:.0f} GB/s", flush=True)
    ref = (A.double() @ x.double())
    print("  max rel err vs fp64 torch:", float(((lb.gemv(A, x) .double() - ref).abs() / ref.abs()).max()))
