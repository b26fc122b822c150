#!/usr/bin/env python
"""Benchmark of the LAPIS hot path on B200 (contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5|c1|c3|c2f32|c2f64]
                    [--impl ours|reference]

Default workload (BASELINE.json config 5, the largest single-GPU config and
the one the metric's multi-GPU scaling is quoted on): CSR SpMV fp64 on the
3-D 27-point stencil, n = 585 -> 200,201,625 rows, 5,386,984,777 nonzeros,
int64 rowptr / int32 colind, row-block sharded over the ranks with the halo
exchange of x (paper_2509_25605_b200/sharded.py).  A step is one SpMV over the
whole matrix.  Inputs (69 GB) exceed L2 (126 MB) many times, so no flush is
needed between steps.

`value` is device-resident throughput (algorithmic bytes / step time, max over
ranks); `e2e` repeats the step through the public DualView + C-ABI path with
the x slice copied host->device and y device->host every step (pinned host
buffers).  `cpu_baseline` runs the reference's own emitted Kokkos C++ on its
serial stub (oracle/_ref) on a bounded row block of the same matrix with all
host threads, and doubles as the parity check of that row block (bit-exact).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SpMV/SpMM HBM GB/s (% of peak), matmul TFLOP/s, at 1/2/4/8 B200 vs CPU ref"


# --------------------------------------------------------------------- utilities
def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = Path(f"/tmp/lapis_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.impl != "reference":
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif world > 1:
        dist.init_process_group("gloo")
    return rank, world, local


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        dist.barrier()


# ------------------------------------------------------------------- workloads
class Stencil27Spmv:
    """Config 5 (default) / config 1: CSR SpMV fp64 on a stencil matrix."""

    def __init__(self, args, rank, world, points=27, n=585, x_seed=5):
        import paper_2509_25605_b200 as lb
        from paper_2509_25605_b200 import sharded
        self.lb, self.args, self.rank, self.world = lb, args, rank, world
        self.points, self.n = points, n
        self.N = n ** 3 if points == 27 else n * n
        self.ranges = sharded.balanced_row_ranges(self.N, world)
        self.r0, self.r1 = self.ranges[rank]
        self.stream = torch.cuda.current_stream()
        self.rowptr, self.colind, self.values = lb.synth_stencil(points, n, self.r0, self.r1)
        self.nnz_local = int(self.rowptr[-1].item())
        rng = np.random.default_rng(x_seed)
        x_host = rng.uniform(-1.0, 1.0, self.N)
        self.x_host = x_host
        self.x = torch.from_numpy(x_host).cuda()          # indexed by global column
        self.y = torch.empty(self.r1 - self.r0, dtype=torch.float64, device="cuda")
        self.op = sharded.RowBlockSpmv(self.rowptr, self.colind, self.values, self.r0, self.r1,
                                       self.N, self.ranges, rank, world)
        self.halo_bytes = 8 * self.op.plan.recv_elems
        # config 1 (80 MB) fits in L2: flush it between timed steps
        self.flush = (torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
                      if self.bytes_per_step_local() < (512 << 20) else None)
        torch.cuda.synchronize()

    @property
    def name(self):
        return (f"config5: CSR SpMV fp64, 3-D 27-point stencil n={self.n}" if self.points == 27
                else f"config1: CSR SpMV fp64, 2-D 5-point Laplacian n={self.n}")

    def config(self):
        return {"workload": self.name, "rows": self.N, "nnz": self.total_nnz(),
                "index_layout": "rowptr int64, colind int32", "x": f"U(-1,1) seed 5",
                "sharding": f"row blocks x{self.world}, halo exchange of x (NCCL P2P)",
                "l2": "inputs >> L2 (126 MB), no flush needed" if self.points == 27 else
                      "L2 flushed between steps (256 MB write)",
                "parallelism": f"rowblock{self.world}"}

    def total_nnz(self):
        return self._global_nnz()

    def _global_nnz(self):
        n = self.n
        return (3 * n - 2) ** 3 if self.points == 27 else 5 * n * n - 4 * n

    def bytes_per_step_global(self) -> int:
        # nnz*(s_v+s_i) + (N+1)*s_p + Ncols*s_v + N*s_v, int32 colind layout
        return self._global_nnz() * 12 + (self.N + 1) * 8 + self.N * 8 + self.N * 8

    def bytes_per_step_local(self) -> int:
        rows = self.r1 - self.r0
        return self.nnz_local * 12 + (rows + 1) * 8 + rows * 8 * 2 + self.halo_bytes

    def launches_per_step(self):
        return self.op.launches_per_multiply

    def kernel_name(self):
        if self.args.vl:
            return f"spmv_vector_kernel<VL={self.args.vl}> (emitted mapping, tree reduce)"
        infos = [p.info() for p in self.op.plans.values()]
        return "; ".join(sorted({i["kernel"] for i in infos})) + " <double,int64,int32>"

    def step(self):
        if self.args.vl:
            # emitted TeamPolicy mapping with an explicit vector length (no plan)
            self.lb.spmv_csr(self.rowptr, self.colind, self.values, self.x, self.y,
                             vector_length=self.args.vl, nnz=self.nnz_local)
            return
        self.op.multiply(self.x, self.y, stream=self.stream)

    # e2e through the public API with host buffers: DualView lazy sync of x's
    # owned slice (host modified every step), kernels, y read back on the host
    def e2e(self, steps, warmup):
        from paper_2509_25605_b200.dualview import DualView
        # the DualView's device side IS the owned slice of the global-indexed x
        xs = DualView.from_host(self.x_host[self.r0:self.r1], "x",
                                device_buffer=self.x[self.r0:self.r1])
        ys = DualView.allocate((self.r1 - self.r0,), torch.float64, "y")

        def one():
            xs.modify_host()
            xs.sync_device(self.stream)
            self.op.multiply(self.x, ys.device_view(), stream=self.stream)
            ys.modify_device()
            ys.sync_host(self.stream)

        for _ in range(warmup):
            one()
        barrier(self.world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / steps
        return dt, xs.nbytes, ys.nbytes

    # reference's own CPU path on a row block of the same matrix (rank 0, N=1)
    def cpu_sample(self, rows_sample):
        mid = self.N // 2
        a, b = max(0, mid - rows_sample // 2), min(self.N, mid + rows_sample // 2)
        rp, ci, v = self.lb.synth_stencil(self.points, self.n, a, b)
        return a, b, rp.cpu().numpy(), ci.cpu().numpy().astype(np.int64), v.cpu().numpy()

    def sample_bytes(self, a, b, nnz):
        rows = b - a
        return nnz * 12 + (rows + 1) * 8 + rows * 8 * 2

    def gpu_rows(self, a, b):
        return self.y[a - self.r0:b - self.r0].cpu().numpy()


WORKLOADS = {
    "c5": lambda args, r, w: Stencil27Spmv(args, r, w, 27, args.n or 585),
    "c1": lambda args, r, w: Stencil27Spmv(args, r, w, 5, args.n or 1000, x_seed=1),
}


def cpu_baseline(wl, args, threads):
    """The reference's emitted C++ on its serial stub (oracle/_ref), all host
    threads, on a bounded row block; also the bit-exact parity check of it."""
    from oracle import ref as R
    if not R.available():
        return {"unavailable": "oracle/_ref not built"}, None
    a, b, rp, ci, v = wl.cpu_sample(args.cpu_rows)
    nnz = int(rp[-1])
    yref, times = R.spmv_csr(rp, ci, v, wl.x_host, reps=args.cpu_reps, threads=threads)
    t = float(np.median(times))
    value = wl.sample_bytes(a, b, nnz) / t / 1e9
    got = wl.gpu_rows(a, b)
    bitexact = bool(np.array_equal(got.view(np.uint64), yref.view(np.uint64)))
    maxrel = float(np.max(np.abs(got - yref) / np.maximum(np.abs(yref), 1.0))) if got.size else 0.0
    base = {"value": round(value, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
            "sample": (f"rows [{a}, {b}) of the same matrix ({nnz} nnz), reference emitted "
                       f"Kokkos C++ (tests/fixtures/spmv.mlir, index colind) on its serial stub, "
                       f"{threads} row blocks on std::threads, median of {args.cpu_reps} reps"),
            "seconds_per_rep": t}
    parity = {"rows_checked": b - a, "bitexact_vs_reference": bitexact, "max_rel_err": maxrel}
    return base, parity


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    from oracle import ref as R
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    torch.cuda.set_device(0)
    wl = WORKLOADS[args.workload](args, 0, 1) if torch.cuda.is_available() else None
    a, b, rp, ci, v = wl.cpu_sample(args.cpu_rows)
    nnz = int(rp[-1])
    _, times = R.spmv_csr(rp, ci, v, wl.x_host, reps=args.warmup + args.steps, threads=threads)
    times = times[args.warmup:]
    t = float(np.mean(times))
    value = wl.sample_bytes(a, b, nnz) / t / 1e9
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(t * 1e3, 4), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": wl.config(),
           "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads,
                            "kind": "reference",
                            "sample": f"rows [{a}, {b}) ({nnz} nnz) of the workload matrix"},
           "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=0, help="grid size override")
    ap.add_argument("--cpu-rows", type=int, default=4_000_000)
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--vl", type=int, default=0,
                    help="time the emitted-mapping vector kernel with this vector length")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local = dist_setup(args)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        if world > 1:
            dist.destroy_process_group()
        return
    torch.cuda.set_device(local)
    wl = WORKLOADS[args.workload](args, rank, world)
    stream = wl.stream
    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per_step = []
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            if wl.flush is not None:
                wl.flush.fill_(1)
            s0.record(stream)
            wl.step()
            s1.record(stream)
            per_step.append((s0, s1))
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    kern = [a.elapsed_time(b) / 1e3 for a, b in per_step]
    # with an L2 flush between steps, the step time excludes the flush
    t_local = (ev0.elapsed_time(ev1) / 1e3 / args.steps if wl.flush is None
               else float(np.mean(kern)))
    t = max_over_ranks(t_local, world)
    kern_avg = max_over_ranks(float(np.mean(kern)), world)
    total_bytes = wl.bytes_per_step_global()
    value = total_bytes / t / 1e9
    pk = peaks()
    # roofline of the dominant kernel (the tile SpMV): this rank's algorithmic bytes
    local_bytes = wl.bytes_per_step_local()
    achieved = local_bytes / kern_avg / 1e9
    traffic = None
    tfile = ROOT / "profiles" / f"traffic_{args.workload}.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get("dram_bytes_per_launch")
    e2e_dt, hb, db = wl.e2e(args.e2e_steps, 2)
    e2e_dt = max_over_ranks(e2e_dt, world)
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (device-generated stencil, numpy-seeded x)",
        "config": wl.config(),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"],
                     "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4),
                     "traffic": traffic, "peak_source": pk["source"],
                     "kernel": wl.kernel_name(),
                     "algorithmic_bytes_per_launch": local_bytes},
        "e2e": {"value": round(total_bytes / e2e_dt / 1e9, 2), "unit": "GB/s",
                "h2d_bytes_per_step": hb, "d2h_bytes_per_step": db,
                "ms_per_step": round(e2e_dt * 1e3, 3),
                "path": "DualView lazy sync (x host-modified each step) + C-ABI plan SpMV + y read"},
        "gpu_launches": args.steps * wl.launches_per_step(),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        base, parity = cpu_baseline(wl, args, os.cpu_count() or 1)
        out["cpu_baseline"] = base
        if parity is not None:
            out["parity"] = parity
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
