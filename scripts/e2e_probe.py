"""C5-sized host<->device traffic: (a) one 1.6 GB H2D and one 1.6 GB D2H
concurrently, (b) the same in 16 / 64 pieces on two streams, (c) the pieces
with the row-chunk SpMVs of StreamedSpmv in between (the e2e path)."""
import sys
import time
import torch
sys.path.insert(0, ".")
import paper_2509_25605_b200 as lb  # noqa: E402
from paper_2509_25605_b200.dualview import DualView  # noqa: E402
from paper_2509_25605_b200.streamed import StreamedSpmv  # noqa: E402

n = 585
rp, ci, v = lb.synth_stencil(27, n)
N = rp.numel() - 1
xh = torch.rand(N, dtype=torch.float64).pin_memory()
yh = torch.empty(N, dtype=torch.float64).pin_memory()
xd = torch.empty(N, dtype=torch.float64, device="cuda")
yd = torch.rand(N, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(f, reps=3):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


def whole():
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(yd, non_blocking=True)


def pieces(p):
    def f():
        step = (N + p - 1) // p
        for i in range(0, N, step):
            with torch.cuda.stream(s1):
                xd[i:i + step].copy_(xh[i:i + step], non_blocking=True)
            with torch.cuda.stream(s2):
                yh[i:i + step].copy_(yd[i:i + step], non_blocking=True)
    return f


print(f"whole, both directions: {timed(whole):.1f} ms")
for p in (16, 64):
    print(f"{p} pieces, both directions: {timed(pieces(p)):.1f} ms")
x = DualView.from_host(xh, "x", device_buffer=xd)
y = DualView.allocate((N,), torch.float64, "y")
for c in (16, 64):
    op = StreamedSpmv(rp, ci, v, N, chunks=c)

    def e2e():
        x.modify_host()
        op.multiply(x, y)
    print(f"StreamedSpmv {c} chunks: {timed(e2e):.1f} ms")
