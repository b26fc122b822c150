"""e2e of the streamed config-5 SpMV at several chunk counts (A/B for streamed.py)."""
import argparse
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2509_25605_b200.dualview import DualView  # noqa: E402
from paper_2509_25605_b200.streamed import StreamedSpmv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--chunks", default="16,32,64")
a = ap.parse_args()
args = bench.argparse.Namespace(vl=0, steps=3, warmup=3, e2e_steps=5, no_cpu=True)
wl = bench.StencilSpmv(args, 0, 1)
xs = DualView.from_host(wl.x_host, "x", device_buffer=wl.x)
ys = DualView.allocate((wl.N,), torch.float64, "y")
for c in [int(v) for v in a.chunks.split(",")]:
    op = StreamedSpmv(wl.rowptr, wl.colind, wl.values, wl.N, chunks=c)

    def one():
        xs.modify_host()
        op.multiply(xs, ys, stream=wl.stream)

    for _ in range(2):
        one()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        one()
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / 5
    print(f"chunks {c}: {t * 1e3:.2f} ms/step, e2e {wl.work_global() / t / 1e9:.1f} GB/s", flush=True)
    del op
