"""C5 per-launch timing: back-to-back launches vs launches separated by idle
gaps, with SM clock / power samples, for the tree and exact plans.
usage: python scripts/c5_launch_probe.py [n]"""
import subprocess
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_25605_b200 as lb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 585
rp, ci, v = lb.synth_stencil(27, n)
N = rp.numel() - 1
nnz = int(rp[-1].item())
byts = nnz * 12 + (N + 1) * 8 + 2 * N * 8
x = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, N)).cuda()
y = torch.empty(N, dtype=torch.float64, device="cuda")


def smi():
    q = "clocks.sm,power.draw,clocks_throttle_reasons.active"
    return subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                          capture_output=True, text=True).stdout.strip()


for mode in ("tree", "exact", "tree", "exact"):
    plan = lb.CsrPlan(rp, exact=(mode == "exact"))
    for _ in range(3):
        plan.spmv(ci, v, x, y)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    samples = []
    stop = threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append(smi())
            time.sleep(0.05)
    th = threading.Thread(target=sampler)
    th.start()
    for a, b in ev:
        a.record()
        plan.spmv(ci, v, x, y)
        b.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    b2b = [a.elapsed_time(b) for a, b in ev]
    gap = []
    for _ in range(8):
        time.sleep(0.3)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.spmv(ci, v, x, y)
        b.record()
        torch.cuda.synchronize()
        gap.append(a.elapsed_time(b))
    print(f"{mode} {plan.info()['kernel']}")
    print("  back-to-back ms:", " ".join(f"{t:.2f}" for t in b2b),
          f"| median {np.median(b2b):.2f} = {byts / np.median(b2b) / 1e6:.0f} GB/s")
    print("  after 300 ms idle:", " ".join(f"{t:.2f}" for t in gap),
          f"| median {np.median(gap):.2f} = {byts / np.median(gap) / 1e6:.0f} GB/s")
    print("  smi (sm MHz, W, reasons):", " | ".join(samples[:12]))
