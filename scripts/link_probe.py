"""Host link probe: pinned H2D, D2H and both directions at once (1.6 GB each)."""
import time
import torch

n = 200_000_000
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(f, reps=3):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps
gb = n * 8 / 1e9
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
t = run(h2d); print(f"H2D {gb / t:.1f} GB/s")
t = run(d2h); print(f"D2H {gb / t:.1f} GB/s")
t = run(both); print(f"both: {2 * gb / t:.1f} GB/s aggregate, {t*1e3:.1f} ms for {gb:.2f} GB each way")
