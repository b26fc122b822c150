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
needed between steps.  Other workloads (--workload) are config 1 (SpMV, 5-point
Laplacian, 84 MB < L2: steps rotate over input copies), config 3 (SpMM, K = 64, power-law
matrix) and config 2 (dense matmul 4096^3, f32 or f64).

`value` is device-resident throughput (algorithmic bytes or flops / step time,
max over ranks); `e2e` repeats the step through the public DualView + C-ABI
path with the step's inputs copied host->device and the result device->host
every step (pinned host buffers).  `cpu_baseline` runs the reference's own
emitted Kokkos C++ on its serial stub (oracle/_ref) on a bounded sample of the
same workload with the host's threads, and doubles as the parity check of that
sample against the GPU result.
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
L2_BYTES = 126 << 20   # B200 L2


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
    if os.environ.get("LAPIS_BENCH_SHARE_GPU") == "1":
        # correctness runs of the N > 1 path on a one-GPU box: every rank on
        # cuda:0, gloo for the process group (NCCL refuses two ranks per GPU);
        # the timings of such a run mean nothing
        local = 0
    if world > 1 and args.impl != "reference":
        torch.cuda.set_device(local)
        if os.environ.get("LAPIS_BENCH_SHARE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif world > 1:
        dist.init_process_group("gloo")
    return rank, world, local


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64,
                     device="cpu" if dist.get_backend() == "gloo" else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        dist.barrier()


def timed_e2e(one, steps, warmup, world):
    for _ in range(warmup):
        one()
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / steps


def parity_report(got, want, tol):
    got, want = np.asarray(got), np.asarray(want)
    if want.dtype.kind == "f":
        iv = np.uint64 if want.dtype.itemsize == 8 else np.uint32
        bitexact = bool(np.array_equal(got.view(iv), want.view(iv)))
        denom = np.maximum(np.maximum(np.abs(got), np.abs(want)), 1.0)
        maxrel = float(np.max(np.abs(got - want) / denom)) if got.size else 0.0
    else:
        bitexact = bool(np.array_equal(got, want))
        maxrel = 0.0 if bitexact else float("inf")
    return {"bitexact_vs_reference": bitexact, "max_rel_err": maxrel, "tolerance": tol,
            "within_tolerance": bool(bitexact or maxrel <= tol)}


# ------------------------------------------------------------------- workloads
class Workload:
    unit = "GB/s"
    bound = "hbm"
    dtype = "f64"
    flush = None
    scaling = "strong"

    def launches_per_step(self) -> int:
        return 1


class StencilSpmv(Workload):
    """Config 5 (default) / config 1: CSR SpMV fp64 on a stencil matrix."""

    def __init__(self, args, rank, world, points=27, n=585, x_seed=5):
        import paper_2509_25605_b200 as lb
        from paper_2509_25605_b200 import sharded
        self.lb, self.args, self.rank, self.world = lb, args, rank, world
        self.points, self.n, self.x_seed = points, n, x_seed
        self.N = n ** 3 if points == 27 else n * n
        self.ranges = sharded.balanced_row_ranges(self.N, world)
        self.r0, self.r1 = self.ranges[rank]
        self.stream = torch.cuda.current_stream()
        self.rowptr, self.colind, self.values = lb.synth_stencil(points, n, self.r0, self.r1)
        self.nnz_local = int(self.rowptr[-1].item())
        self.x_host = np.random.default_rng(x_seed).uniform(-1.0, 1.0, self.N)
        self.x = torch.from_numpy(self.x_host).cuda()          # indexed by global column
        self.y = torch.empty(self.r1 - self.r0, dtype=torch.float64, device="cuda")
        self.op = sharded.RowBlockSpmv(self.rowptr, self.colind, self.values, self.r0, self.r1,
                                       self.N, self.ranges, rank, world)
        self.halo_bytes = 8 * self.op.plan.recv_elems
        # config 1 (84 MB) fits in L2 (126 MB): the timed steps rotate over R
        # device copies of the whole input (matrix, x, y; R * work >= 3 x L2), so
        # every step reads its operands cold from HBM without a flush kernel
        # between steps (a 256 MB write flush leaves L2 full of dirty lines whose
        # write-back would be timed inside the next SpMV)
        self.rot = [(self.rowptr, self.colind, self.values, self.x, self.y, self.op)]
        self.rot_i = 0
        self.last_y = self.y
        if self.work_local() < (512 << 20) and not args.vl:
            ncopy = -(-(3 * L2_BYTES) // int(self.work_local()))
            for _ in range(1, ncopy):
                rp, ci, v = self.rowptr.clone(), self.colind.clone(), self.values.clone()
                self.rot.append((rp, ci, v, self.x.clone(), torch.empty_like(self.y),
                                 sharded.RowBlockSpmv(rp, ci, v, self.r0, self.r1, self.N,
                                                      self.ranges, rank, world)))
        torch.cuda.synchronize()

    @property
    def name(self):
        return (f"config5: CSR SpMV fp64, 3-D 27-point stencil n={self.n}" if self.points == 27
                else f"config1: CSR SpMV fp64, 2-D 5-point Laplacian n={self.n}")

    def nnz_global(self):
        n = self.n
        return (3 * n - 2) ** 3 if self.points == 27 else 5 * n * n - 4 * n

    def config(self):
        return {"workload": self.name, "rows": self.N, "nnz": self.nnz_global(),
                "index_layout": "rowptr int64, colind int32", "x": f"U(-1,1) seed {self.x_seed}",
                "sharding": f"row blocks x{self.world}, halo exchange of x (NCCL P2P)",
                **({"launch": self.graph_note} if self.graphs else {}),
                "l2": ("inputs >> L2 (126 MB), no flush needed" if len(self.rot) == 1 else
                       f"inputs < L2: steps rotate over {len(self.rot)} device copies of the "
                       f"whole input ({len(self.rot) * self.work_local() / 1e6:.0f} MB > 3 x L2), "
                       "no flush"),
                "parallelism": f"rowblock{self.world}"}

    def work_global(self) -> float:
        # nnz*(s_v+s_i) + (N+1)*s_p + Ncols*s_v + N*s_v, int32 colind layout
        return self.nnz_global() * 12 + (self.N + 1) * 8 + self.N * 8 + self.N * 8

    def work_local(self) -> float:
        rows = self.r1 - self.r0
        return self.nnz_local * 12 + (rows + 1) * 8 + rows * 8 * 2 + self.halo_bytes

    def launches_per_step(self):
        return 1 if self.args.vl else self.op.launches_per_multiply

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
            self.last_y = self.y
            return
        rp, ci, v, x, y, op = self.rot[self.rot_i]
        g = self.graphs[self.rot_i] if self.graphs else None
        self.rot_i = (self.rot_i + 1) % len(self.rot)
        if g is not None:
            g.replay()
        else:
            op.multiply(x, y, stream=self.stream)
        self.last_y = y

    graphs = None

    def capture_graphs(self):
        """Config 1's SpMV (~15-20 us) is shorter than the host cost of one
        Python-level multiply, so on one GPU each rotation copy's multiply is
        captured once in a CUDA graph and a step replays it (same kernel, same
        arguments; the graph only removes the host launch overhead)."""
        if self.world > 1 or len(self.rot) == 1 or self.args.vl:
            return
        graphs = []
        side = torch.cuda.Stream()
        side.wait_stream(self.stream)
        for rp, ci, v, x, y, op in self.rot:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                op.multiply(x, y, stream=side)
            graphs.append(g)
        self.stream.wait_stream(side)
        torch.cuda.synchronize()
        self.graphs = graphs
        self.graph_note = f"each step replays a captured CUDA graph of the multiply ({len(graphs)} graphs, one per input copy)"

    def sharded_parity(self):
        if self.N > 50_000_000:
            return None
        rp, ci, v = self.lb.synth_stencil(self.points, self.n)
        plan = self.lb.CsrPlan(rp)
        y = plan.spmv(ci, v, self.x)
        return bool(torch.equal(y[self.r0:self.r1], self.last_y))

    def exact_variant(self, steps):
        """The same multiply with every row folded in the reference order (plan
        exact mode, bit-identical); device-resident throughput."""
        from paper_2509_25605_b200 import sharded
        ops = [(sharded.RowBlockSpmv(rp, ci, v, self.r0, self.r1, self.N, self.ranges, self.rank,
                                     self.world, exact=True), x, y)
               for rp, ci, v, x, y, _ in self.rot]
        for i in range(3):
            op, x, y = ops[i % len(ops)]
            op.multiply(x, y, stream=self.stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(self.stream)
        for i in range(steps):
            op, x, y = ops[i % len(ops)]
            op.multiply(x, y, stream=self.stream)
        b.record(self.stream)
        torch.cuda.synchronize()
        t = max_over_ranks(a.elapsed_time(b) / 1e3 / steps, self.world)
        names = sorted({p.info()["kernel"] for p in ops[0][0].plans.values()})
        return {"value": round(self.work_global() / t / 1e9, 3), "unit": "GB/s",
                "frac": round(self.work_local() / t / 1e9 / peaks()["hbm_gbs"], 4),
                "kernel": "; ".join(names), "note": "bit-identical to the reference"}

    def e2e(self, steps, warmup):
        """DualView lazy sync of this rank's x slice (host-modified every step),
        the sharded multiply, y read back on the host.  One GPU: the streamed
        multiply (paper_2509_25605_b200/streamed.py) overlaps the H2D of x, the
        row-chunk kernels and the D2H of y."""
        from paper_2509_25605_b200.dualview import DualView
        if self.world == 1 and not self.args.vl:
            from paper_2509_25605_b200.streamed import StreamedSpmv
            xs = DualView.from_host(self.x_host, "x", device_buffer=self.x)
            ys = DualView.allocate((self.N,), torch.float64, "y")
            op = StreamedSpmv(self.rowptr, self.colind, self.values, self.N)

            def one_streamed():
                xs.modify_host()
                op.multiply(xs, ys, stream=self.stream)

            t = timed_e2e(one_streamed, steps, warmup, self.world)
            # the streamed result is the device multiply's (same plan kernels)
            self.e2e_parity = bool(torch.equal(ys.host_view(), self.y.cpu()))
            self.e2e_path = (f"StreamedSpmv: H2D of x in column pieces, {len(op.plans)} row-chunk "
                             "plan SpMVs and the D2H of y overlapped on 3 streams (DualView "
                             "semantics kept)")
            return t, xs.nbytes, ys.nbytes
        xs = DualView.from_host(self.x_host[self.r0:self.r1], "x",
                                device_buffer=self.x[self.r0:self.r1])
        ys = DualView.allocate((self.r1 - self.r0,), torch.float64, "y")

        def one():
            xs.modify_host()
            xs.sync_device(self.stream)
            self.op.multiply(self.x, ys.device_view(), stream=self.stream)
            ys.modify_device()
            ys.sync_host(self.stream)

        return timed_e2e(one, steps, warmup, self.world), xs.nbytes, ys.nbytes

    def cpu_reference(self, rows_sample, threads, reps):
        """Reference emitted spmv on rows [a, b) of the same matrix."""
        from oracle import ref as R
        mid = self.N // 2
        a, b = max(0, mid - rows_sample // 2), min(self.N, mid + rows_sample // 2)
        rp, ci, v = self.lb.synth_stencil(self.points, self.n, a, b)
        rp, ci, v = rp.cpu().numpy(), ci.cpu().numpy().astype(np.int64), v.cpu().numpy()
        nnz = int(rp[-1])
        yref, times = R.spmv_csr(rp, ci, v, self.x_host, reps=reps, threads=threads)
        work = nnz * 12 + (b - a + 1) * 8 + (b - a) * 8 * 2
        desc = (f"rows [{a}, {b}) of the same matrix ({nnz} nnz): reference emitted Kokkos C++ "
                f"(tests/fixtures/spmv.mlir, index colind) on its serial stub, {threads} row "
                f"blocks on std::threads")
        got = self.last_y[a - self.r0:b - self.r0].cpu().numpy()
        return yref, got, times, work, desc, 1e-12


class MtxSpmv(Workload):
    """CSR SpMV fp64 on a Matrix Market file (--mtx; the paper's SuiteSparse
    runs): read natively (paper_2509_25605_b200/mmio.py),
    planned once, x U(-1,1) seed 7.  N > 1: independent replicas."""

    scaling = "weak"

    data = "matrix market file (--mtx), x seeded"

    def __init__(self, args, rank, world):
        import paper_2509_25605_b200 as lb
        from paper_2509_25605_b200 import mmio
        if not args.mtx:
            raise SystemExit("--workload mtx needs --mtx <file.mtx>")
        self.lb, self.args, self.world, self.path = lb, args, world, args.mtx
        rp, ci, v, (self.N, self.ncols) = mmio.read_matrix_market(args.mtx)
        self.rowptr, self.colind, self.values = mmio.to_device(rp, ci, v)
        self.nnz = int(rp[-1])
        self.stream = torch.cuda.current_stream()
        self.x_host = np.random.default_rng(7).uniform(-1.0, 1.0, self.ncols)
        self.x = torch.from_numpy(self.x_host).cuda()
        self.y = torch.empty(self.N, dtype=torch.float64, device="cuda")
        self.plan = lb.CsrPlan(self.rowptr, nnz=self.nnz)
        if self.work_local() < (512 << 20):
            self.flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()

    @property
    def name(self):
        return f"matrix market SpMV fp64: {Path(self.path).name}"

    def config(self):
        return {"workload": self.name, "rows": self.N, "cols": self.ncols, "nnz": self.nnz,
                "index_layout": "rowptr int64, colind int32", "parallelism": "replica",
                "l2": "L2 flushed between steps" if self.flush is not None else "inputs > L2"}

    def work_local(self):
        return self.nnz * 12 + (self.N + 1) * 8 + self.ncols * 8 + self.N * 8

    def work_global(self):
        return self.work_local() * self.world

    def kernel_name(self):
        return self.plan.info()["kernel"] + " <double,int64,int32>"

    def step(self):
        self.plan.spmv(self.colind, self.values, self.x, self.y, stream=self.stream)

    def e2e(self, steps, warmup):
        from paper_2509_25605_b200.dualview import DualView
        from paper_2509_25605_b200.streamed import StreamedSpmv
        xs = DualView.from_host(self.x_host, "x", device_buffer=self.x)
        ys = DualView.allocate((self.N,), torch.float64, "y")
        op = StreamedSpmv(self.rowptr, self.colind, self.values, self.ncols)

        def one():
            xs.modify_host()
            op.multiply(xs, ys, stream=self.stream)

        return timed_e2e(one, steps, warmup, self.world), xs.nbytes, ys.nbytes

    def cpu_reference(self, rows_sample, threads, reps):
        from oracle import ref as R
        rp = self.rowptr.cpu().numpy()
        b = min(self.N, rows_sample)
        e0, e1 = int(rp[0]), int(rp[b])
        ci = self.colind[e0:e1].cpu().numpy().astype(np.int64)
        v = self.values[e0:e1].cpu().numpy()
        yref, times = R.spmv_csr(rp[:b + 1] - e0, ci, v, self.x_host, reps=reps, threads=threads)
        work = (e1 - e0) * 12 + (b + 1) * 8 + b * 8 * 2
        desc = (f"rows [0, {b}) ({e1 - e0} nnz): reference emitted Kokkos C++ on its serial "
                f"stub, {threads} row blocks")
        return yref, self.y[:b].cpu().numpy(), times, work, desc, 1e-12


class PowerLawSpmm(Workload):
    """Config 3: CSR x dense SpMM fp64, K = 64, Chung-Lu power-law matrix.

    N > 1: the SAME global matrix, row-block sharded
    (sharded.RowBlockSpmm: rank r owns rows [r*c, r*c + c), c = ceil(N / world),
    and the matching rows of X and Y); a step is the NCCL all-gather of X
    followed by the local SpMM (strong scaling, total work fixed).  The
    "x_replicated" variant times the local SpMM alone (features resident on
    every GPU, the GCN case)."""

    name = "config3: CSR x dense SpMM fp64, K=64, power-law (Chung-Lu, Pareto 2.5) 10M rows"
    scaling = "strong"
    variant_key = "variants"

    def __init__(self, args, rank, world, n=10_000_000, k=64, mean=10.0, seed=1):
        import paper_2509_25605_b200 as lb
        from paper_2509_25605_b200 import sharded
        self.lb, self.args, self.world, self.rank = lb, args, world, rank
        self.N, self.k, self.seed = n, k, seed
        self.stream = torch.cuda.current_stream()
        rowptr, colind, values = powerlaw_csr_device(n, mean, 2.5, seed)
        self.nnz_global_ = int(rowptr[-1].item())
        g = torch.Generator(device="cuda").manual_seed(seed + 100)
        X = torch.rand((n, k), generator=g, dtype=torch.float64, device="cuda") * 2 - 1
        lens = (rowptr[1:] - rowptr[:-1])
        self.max_len = int(lens.max().item())
        self.median_len = float(lens.double().median().item())
        self.r0, self.r1 = sharded.equal_row_ranges(n, world)[rank]
        self.full = ((rowptr, colind, values, X.clone())
                     if world > 1 and n * k * 8 < (2 << 30) else None)
        if world > 1:
            a, b = int(rowptr[self.r0].item()), int(rowptr[self.r1].item())
            self.rowptr = (rowptr[self.r0:self.r1 + 1] - a).contiguous()
            self.colind, self.values = colind[a:b].contiguous(), values[a:b].contiguous()
            del rowptr, colind, values
        else:
            self.rowptr, self.colind, self.values = rowptr, colind, values
        self.nnz = int(self.rowptr[-1].item())
        self.op = sharded.RowBlockSpmm(self.rowptr, self.colind, self.values, n, k, rank, world)
        self.op.x_local.copy_(X[self.r0:self.r1])
        del X
        self.op.gather()
        self.X = self.op.X_full[:n]
        self.Y = torch.empty((self.r1 - self.r0, k), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()

    def config(self):
        return {"workload": self.name, "rows": self.N, "nnz": self.nnz_global_, "k": self.k,
                "max_row": self.max_len, "median_row": self.median_len,
                "index_layout": "rowptr int64, colind int32",
                "generator": f"torch CUDA generator seed {self.seed} (device)",
                "l2": "inputs >> L2",
                "sharding": (f"row blocks x{self.world}, NCCL all-gather of X "
                             f"({self.op.gather_bytes / 1e9:.2f} GB received per rank per step) "
                             "then the local SpMM" if self.world > 1 else "none"),
                "parallelism": f"rowblock{self.world}"}

    def _work(self, nnz, rows):
        # nnz*(s_v+s_i) + (N+1)*s_p + Ncols*K*s_v + N*K*s_v
        return nnz * 12 + (rows + 1) * 8 + self.N * self.k * 8 + rows * self.k * 8

    def work_global(self):
        return self._work(self.nnz_global_, self.N)

    def work_local(self):
        # the local SpMM's algorithmic bytes (its X gathers can touch every row of X)
        return self._work(self.nnz, self.r1 - self.r0)

    def launches_per_step(self):
        return 4 if self.max_len > 2048 else 1

    def kernel_name(self):
        return ("spmm_batch_kernel<double> (32 rows per warp) + long rows: "
                "long_rows_list/work, spmm_long_chunk/combine")

    def step(self):
        self.op.multiply(self.Y, stream=self.stream)

    def sharded_parity(self):
        if self.full is None:
            return None
        rp, ci, v, X = self.full
        Y = self.lb.spmm_csr(rp, ci, v, X)
        return bool(torch.equal(Y[self.r0:self.r1], self.Y))

    def exact_variant(self, steps):
        """N > 1: the X-replicated time (local SpMM only, no all-gather)."""
        if self.world == 1:
            return None
        for _ in range(3):
            self.op.multiply(self.Y, stream=self.stream, replicated=True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(self.world)
        torch.cuda.synchronize()
        a.record(self.stream)
        for _ in range(steps):
            self.op.multiply(self.Y, stream=self.stream, replicated=True)
        b.record(self.stream)
        torch.cuda.synchronize()
        t = max_over_ranks(a.elapsed_time(b) / 1e3 / steps, self.world)
        return {"x_replicated": {"value": round(self.work_global() / t / 1e9, 3), "unit": "GB/s",
                                 "ms_per_step": round(t * 1e3, 4),
                                 "note": "X resident on every GPU: local SpMM only"}}

    def e2e(self, steps, warmup):
        """This rank's rows of X host-modified every step (DualView sync of the
        slot, then the all-gather when N > 1), Y read back."""
        from paper_2509_25605_b200.dualview import DualView
        xs = DualView.from_host(self.op.x_local.cpu(), "X", device_buffer=self.op.x_local)
        ys = DualView.allocate(tuple(self.Y.shape), torch.float64, "Y")

        def one():
            xs.modify_host()
            xs.sync_device(self.stream)
            self.op.multiply(ys.device_view(), stream=self.stream)
            ys.modify_device()
            ys.sync_host(self.stream)

        return timed_e2e(one, steps, warmup, self.world), xs.nbytes, ys.nbytes

    def cpu_reference(self, rows_sample, threads, reps):
        from oracle import ref as R
        a, b = 0, min(self.N, max(1, rows_sample // 40))
        rp = self.rowptr[a:b + 1].cpu().numpy()
        ci = self.colind[rp[0]:rp[-1]].cpu().numpy()
        v = self.values[rp[0]:rp[-1]].cpu().numpy()
        rp = rp - rp[0]
        X = self.X.cpu().numpy()
        threads = min(threads, 2)   # each thread block replicates X (5 GB) on the stub
        self.cpu_threads_used = threads
        Yref, times = R.spmm_csr(rp, ci, v, X, reps=reps, threads=threads)
        nnz = int(rp[-1])
        work = nnz * 12 + (b - a + 1) * 8 + (b - a) * self.k * 8 * 2
        desc = (f"rows [{a}, {b}) ({nnz} nnz) of the same matrix: reference emitted Kokkos C++ "
                f"of oracle/ir/spmm.mlir on its serial stub, {threads} row blocks")
        got = self.Y[a:b].cpu().numpy()
        return Yref, got, times, work, desc, 1e-12


class DenseMatmul(Workload):
    """Config 2: dense linalg.matmul 4096^3 (f32: 3xTF32 / exact; f64: DMMA / exact)."""

    unit = "TFLOP/s"
    bound = "tensor"
    scaling = "weak"

    def __init__(self, args, rank, world, dt=torch.float32, n=4096):
        import paper_2509_25605_b200 as lb
        self.lb, self.args, self.world, self.n, self.dt = lb, args, world, n, dt
        self.dtype = "f32" if dt == torch.float32 else "f64"
        self.stream = torch.cuda.current_stream()
        g = torch.Generator(device="cuda").manual_seed(3 if dt == torch.float32 else 2)
        lo = 0.0 if dt == torch.float32 else -1.0   # f32 U(0,1), f64 U(-1,1)
        self.A = (torch.rand((n, n), generator=g, dtype=dt, device="cuda") * (1 - lo) + lo)
        self.B = (torch.rand((n, n), generator=g, dtype=dt, device="cuda") * (1 - lo) + lo)
        self.C = torch.empty((n, n), dtype=dt, device="cuda")
        self.mode = args.gemm_mode
        if 3 * n * n * (4 if dt == torch.float32 else 8) < (256 << 20):
            self.flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()

    @property
    def name(self):
        return f"config2: dense linalg.matmul {self.n}^3 {self.dtype} (mode {self.mode})"

    def config(self):
        return {"workload": self.name, "m": self.n, "n": self.n, "k": self.n,
                "inputs": "U(0,1)" if self.dt == torch.float32 else "U(-1,1)",
                "l2": "L2 flushed between steps" if self.flush is not None else "working set > L2",
                "parallelism": "replica"}

    def work_global(self):
        return 2.0 * self.n ** 3 * self.world

    def work_local(self):
        return 2.0 * self.n ** 3

    def effective_mode(self):
        if self.mode != "auto":
            return self.mode
        if self.dt == torch.float32:
            return "tf32x3"
        return "ozaki" if self.n * 9.0 * 2.0 ** -56 <= 0.75e-12 else "dmma"

    def kernel_name(self):
        m = self.effective_mode()
        names = {"tf32x3": "gemm_tf32x3_kernel (tcgen05 kind::tf32, 3xTF32)",
                 "dmma": "gemm_dmma_kernel (DMMA m8n8k4)",
                 "exact": "gemm_exact_kernel (reference order)",
                 "ozaki": ("gemm_ozaki_2p_kernel (tcgen05 kind::i8, two-pass Ozaki, certified)"
                           if self.dt == torch.float64 and self.n * 9.0 * 2.0 ** -56 <= 0.75e-12
                           else "gemm_ozaki_kernel (tcgen05 kind::i8, Ozaki digits, certified)")}
        return f"gemm<{self.dtype}> mode={self.mode} -> {names[m]}"

    def roofline_override(self, kern_avg):
        """The Ozaki kernel runs int8 MMAs: its roofline is the int8 tensor
        peak (2x the measured dense bf16 rate), counted in int8 ops."""
        if self.effective_mode() != "ozaki":
            return None
        S = (8 if self.n * 9.0 * 2.0 ** -56 <= 0.75e-12 else 9) if self.dt == torch.float64 else 3
        products = S * (S + 1) // 2
        ops = products * 2.0 * self.n ** 3
        pk = peaks()
        peak = 2.0 * pk["bf16_tflops"]
        achieved = ops / kern_avg / 1e12
        return {"bound": "tensor", "achieved": round(achieved, 2), "peak": round(peak, 1),
                "unit": "TOPS (int8)", "frac": round(achieved / peak, 4),
                "peak_source": f"2 x {pk['source']} bf16_tflops (dense int8 = 2x bf16 on B200)",
                "int8_products": products, "ops_per_launch": ops}

    def step(self):
        self.lb.gemm(self.A, self.B, self.C, mode=self.mode)

    def e2e(self, steps, warmup):
        from paper_2509_25605_b200.dualview import DualView
        a = DualView.from_host(self.A.cpu(), "A", device_buffer=self.A)
        b = DualView.from_host(self.B.cpu(), "B", device_buffer=self.B)
        c = DualView.allocate(tuple(self.C.shape), self.dt, "C")

        def one():
            a.modify_host()
            b.modify_host()
            a.sync_device(self.stream)
            b.sync_device(self.stream)
            self.lb.gemm(a.device_view(), b.device_view(), c.device_view(), mode=self.mode)
            c.modify_device()
            c.sync_host(self.stream)

        return timed_e2e(one, steps, warmup, self.world), a.nbytes + b.nbytes, c.nbytes

    def cpu_reference(self, rows_sample, threads, reps):
        from oracle import ref as R
        rows = max(threads, min(self.n, rows_sample // 250_000))
        A = self.A[:rows].cpu().numpy()
        B = self.B.cpu().numpy()
        Cref, times = R.matmul(A, B, reps=reps, threads=threads)
        desc = (f"rows [0, {rows}) of C: reference emitted Kokkos C++ of oracle/ir/matmul_"
                f"{self.dtype}.mlir (TeamPolicy nest) on its serial stub, {threads} row blocks")
        got = self.C[:rows].cpu().numpy()
        tol = 1e-5 if self.dt == torch.float32 else 1e-12
        return Cref, got, times, 2.0 * rows * self.n * self.n, desc, tol


class GcnLayer(Workload):
    """Config 4: GCN layer H = relu((A_hat X) W), fp32, A_hat = D^-1/2 A D^-1/2 of the
    config-3 power-law generator at 1M rows, X [N, 64] U(0,1), W [64, 64]
    U(-1/8, 1/8) (torch Linear default bound for fan-in 64), seed 4."""

    name = "config4: GCN layer relu((A_hat X) W) fp32, power-law A_hat 1M rows, 64->64"
    dtype = "f32"
    scaling = "weak"

    def __init__(self, args, rank, world, n=1_000_000, f=64, seed=4):
        import paper_2509_25605_b200 as lb
        self.lb, self.args, self.world, self.N, self.f = lb, args, world, n, f
        self.stream = torch.cuda.current_stream()
        rowptr, colind, _ = powerlaw_csr_device(n, 10.0, 2.5, seed)
        deg = (rowptr[1:] - rowptr[:-1]).clamp(min=1).to(torch.float64)
        rows = torch.repeat_interleave(torch.arange(n, device="cuda"), rowptr[1:] - rowptr[:-1])
        vals = (deg[rows] * deg[colind.long()]).rsqrt().to(torch.float32)
        self.rowptr, self.colind, self.values = rowptr, colind, vals.contiguous()
        self.nnz = int(rowptr[-1].item())
        g = torch.Generator(device="cuda").manual_seed(seed)
        self.X = torch.rand((n, f), generator=g, dtype=torch.float32, device="cuda")
        self.W = (torch.rand((f, f), generator=g, dtype=torch.float32, device="cuda") * 2 - 1) / 8
        self.H = torch.empty((n, f), dtype=torch.float32, device="cuda")
        self.max_len = int((rowptr[1:] - rowptr[:-1]).max().item())
        torch.cuda.synchronize()

    def config(self):
        return {"workload": self.name, "rows": self.N, "nnz": self.nnz, "features": self.f,
                "max_row": self.max_len, "parallelism": "replica",
                "bytes": "compulsory: A_hat + X + W + H (no A_hat X intermediate)",
                "l2": "inputs > L2 (X 256 MB)"}

    def work_local(self):
        # compulsory bytes of the layer: A_hat (int32 colind + f32 values, int64
        # rowptr), X, W read once, H written once.  The A_hat X intermediate is
        # not counted (the fused kernel never materialises it)
        f, n = self.f, self.N
        return self.nnz * 8 + (n + 1) * 8 + n * f * 4 + f * f * 4 + n * f * 4

    def work_global(self):
        return self.work_local() * self.world

    def launches_per_step(self):
        return 4 if self.max_len > 2048 else 2

    def kernel_name(self):
        return ("spmm_batch_kernel<float> + spmm_seq_long_pipe_kernel (exact-order hub rows, "
                "16-column groups) + gemm_exact_narrow_kernel<relu> (reference order)")

    def step(self):
        self.lb.gcn_layer(self.rowptr, self.colind, self.values, self.X, self.W, self.H,
                          nnz=self.nnz)

    def e2e(self, steps, warmup):
        """X (node features) host-modified every step, H read back."""
        from paper_2509_25605_b200.dualview import DualView
        xs = DualView.from_host(self.X.cpu(), "X", device_buffer=self.X)
        hs = DualView.allocate(tuple(self.H.shape), torch.float32, "H")

        def one():
            xs.modify_host()
            xs.sync_device(self.stream)
            self.lb.gcn_layer(self.rowptr, self.colind, self.values, xs.device_view(), self.W,
                              hs.device_view(), nnz=self.nnz)
            hs.modify_device()
            hs.sync_host(self.stream)

        return timed_e2e(one, steps, warmup, self.world), xs.nbytes, hs.nbytes

    def cpu_reference(self, rows_sample, threads, reps):
        from oracle import ref as R
        a, b = 0, min(self.N, max(1, rows_sample // 80))
        rp = self.rowptr[a:b + 1].cpu().numpy()
        ci = self.colind[rp[0]:rp[-1]].cpu().numpy()
        v = self.values[rp[0]:rp[-1]].cpu().numpy()
        rp = rp - rp[0]
        threads = min(threads, 4)   # each block replicates X (256 MB) on the stub
        self.cpu_threads_used = threads
        Href, times = R.gcn(rp, ci, v, self.X.cpu().numpy(), self.W.cpu().numpy(), reps=reps,
                            threads=threads)
        nnz = int(rp[-1])
        f = self.f
        work = nnz * 8 + (b - a + 1) * 8 + (b - a) * f * 4 * 3 + f * f * 4
        desc = (f"rows [{a}, {b}) ({nnz} nnz): reference emitted Kokkos C++ of "
                f"oracle/ir/gcn_f32.mlir on its serial stub, {threads} row blocks")
        return Href, self.H[a:b].cpu().numpy(), times, work, desc, 1e-5


def powerlaw_csr_device(n, mean, alpha, seed):
    """Chung-Lu power-law CSR built on the device: Pareto(alpha) row
    weights, rows and columns drawn in proportion to the weights, hubs scattered
    by a permutation, sorted and deduplicated; int64 rowptr, int32 colind,
    values U(-1, 1)."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    dev = "cuda"
    w = (1.0 - torch.rand(n, generator=g, dtype=torch.float64, device=dev)) ** (-1.0 / (alpha - 1.0))
    cdf = torch.cumsum(w, 0)
    total = int(mean * n)
    perm = torch.randperm(n, generator=g, device=dev)
    keys = []
    chunk = 25_000_000
    for c0 in range(0, total, chunk):
        m = min(chunk, total - c0)
        r = torch.searchsorted(cdf, torch.rand(m, generator=g, dtype=torch.float64, device=dev) * cdf[-1])
        c = torch.searchsorted(cdf, torch.rand(m, generator=g, dtype=torch.float64, device=dev) * cdf[-1])
        r = perm[r.clamp_(max=n - 1)]
        c = perm[c.clamp_(max=n - 1)]
        keys.append(r.to(torch.int64) * n + c.to(torch.int64))
        del r, c
    key = torch.unique(torch.cat(keys))
    del keys
    rows = torch.div(key, n, rounding_mode="floor")
    cols = (key - rows * n).to(torch.int32)
    counts = torch.bincount(rows, minlength=n)
    rowptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    rowptr[1:] = torch.cumsum(counts, 0)
    values = torch.rand(key.numel(), generator=g, dtype=torch.float64, device=dev) * 2 - 1
    return rowptr, cols.contiguous(), values


class DenseMatvec(Workload):
    """linalg.matvec / LAPIS::gemv (fixture tests/fixtures/matvec_f64.mlir
    scaled up): y = A x, A 16384 x 16384 f64 U(-1,1) seed 6 (2.1 GB > L2, no
    flush needed), folded in the reference order (bit-identical).  N > 1:
    independent replicas."""

    name = "matvec: linalg.matvec f64 16384 x 16384 (row_fold_pipe_kernel, reference order)"
    scaling = "weak"

    def __init__(self, args, rank, world, n=16384):
        import paper_2509_25605_b200 as lb
        self.lb, self.args, self.world, self.n = lb, args, world, n
        self.stream = torch.cuda.current_stream()
        g = torch.Generator(device="cuda").manual_seed(6)
        self.A = torch.rand((n, n), generator=g, dtype=torch.float64, device="cuda") * 2 - 1
        self.x = torch.rand(n, generator=g, dtype=torch.float64, device="cuda") * 2 - 1
        self.y = torch.empty(n, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()

    def config(self):
        return {"workload": self.name, "rows": self.n, "cols": self.n, "l2": "A 2.1 GB >> L2",
                "parallelism": "replica"}

    def work_local(self):
        return (self.n * self.n + 2 * self.n) * 8

    def work_global(self):
        return self.work_local() * self.world

    def kernel_name(self):
        return "row_fold_pipe_kernel<double, DOT, 16-byte> (32 rows per CTA, 6-stage cp.async ring)"

    def step(self):
        self.lb.gemv(self.A, self.x, self.y, stream=self.stream)

    def e2e(self, steps, warmup):
        """x host-modified every step, y read back (A resident)."""
        from paper_2509_25605_b200.dualview import DualView
        xs = DualView.from_host(self.x.cpu(), "x", device_buffer=self.x)
        ys = DualView.allocate((self.n,), torch.float64, "y")

        def one():
            xs.modify_host()
            xs.sync_device(self.stream)
            self.lb.gemv(self.A, xs.device_view(), ys.device_view(), stream=self.stream)
            ys.modify_device()
            ys.sync_host(self.stream)

        return timed_e2e(one, steps, warmup, self.world), xs.nbytes, ys.nbytes

    def cpu_reference(self, rows_sample, threads, reps):
        from oracle import ref as R
        rows = min(self.n, max(1, rows_sample // 4000))   # 1000 rows = 131 MB
        self.cpu_threads_used = 1
        A = self.A[:rows].cpu().numpy()
        yref, times = R.matvec(A, self.x.cpu().numpy(), reps=reps)
        work = (rows * self.n + self.n + rows) * 8
        desc = (f"rows [0, {rows}) of the same A: reference emitted Kokkos C++ of "
                "oracle/ir/matvec_f64.mlir on its serial stub, 1 thread")
        return yref, self.y[:rows].cpu().numpy(), times, work, desc, 1e-12


WORKLOADS = {
    "c5": lambda args, r, w: StencilSpmv(args, r, w, 27, args.n or 585, x_seed=5),
    "c1": lambda args, r, w: StencilSpmv(args, r, w, 5, args.n or 1000, x_seed=1),
    "c3": lambda args, r, w: PowerLawSpmm(args, r, w, args.n or 10_000_000),
    "c2f32": lambda args, r, w: DenseMatmul(args, r, w, torch.float32, args.n or 4096),
    "c2f64": lambda args, r, w: DenseMatmul(args, r, w, torch.float64, args.n or 4096),
    "c4": lambda args, r, w: GcnLayer(args, r, w, args.n or 1_000_000),
    "mtx": lambda args, r, w: MtxSpmv(args, r, w),
    "gemv": lambda args, r, w: DenseMatvec(args, r, w, args.n or 16384),
}


def cpu_baseline(wl, args, threads):
    """The reference's emitted C++ on its serial stub (oracle/_ref) on a bounded
    sample of the workload; also the parity check of that sample."""
    from oracle import ref as R
    if not R.available():
        return {"unavailable": "oracle/_ref not built"}, None
    want, got, times, work, desc, tol = wl.cpu_reference(args.cpu_rows, threads, args.cpu_reps)
    t = float(np.median(times))
    # about 10 s of CPU work in total (bounded sample, repeated)
    reps = int(min(2000, max(args.cpu_reps, np.ceil(args.cpu_seconds / max(t, 1e-6)))))
    if reps > args.cpu_reps:
        want, got, times, work, desc, tol = wl.cpu_reference(args.cpu_rows, threads, reps)
        t = float(np.median(times))
    scale = 1e9 if wl.unit == "GB/s" else 1e12
    base = {"value": round(work / t / scale, 4), "unit": wl.unit,
            "cores": getattr(wl, "cpu_threads_used", threads),
            "kind": "reference", "sample": desc + f", median of {len(times)} reps",
            "seconds_per_rep": t}
    parity = {"sample_elements": int(np.asarray(want).size), **parity_report(got, want, tol)}
    return base, parity


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    from oracle import ref as R
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    threads = os.cpu_count() or 1
    torch.cuda.set_device(0)
    wl = WORKLOADS[args.workload](args, 0, 1)
    wl.step()
    torch.cuda.synchronize()
    _, _, times, work, desc, _ = wl.cpu_reference(args.cpu_rows, threads,
                                                  args.warmup + args.steps)
    times = times[args.warmup:]
    t = float(np.mean(times))
    scale = 1e9 if wl.unit == "GB/s" else 1e12
    value = work / t / scale
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": wl.unit,
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(t * 1e3, 4), "higher_is_better": True, "scaling": wl.scaling,
           "vs_baseline": None, "dtype": wl.dtype, "data": "synthetic", "config": wl.config(),
           "cpu_baseline": {"value": round(value, 4), "unit": wl.unit, "cores": getattr(wl, "cpu_threads_used", threads),
                            "kind": "reference", "sample": desc},
           "e2e": {"value": round(value, 4), "unit": wl.unit, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def launch_census(wl):
    """Kernels one step launches, counted by the CUDA activity tracer (CUPTI via
    torch.profiler) on an untimed step after the timed region: how many of
    OUR kernels (namespace lapis_b200 / NVRTC-generated lapis_*) run per step
    and each one's share of the step's device time.  None when the tracer is
    unavailable."""
    try:
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            wl.step()
            torch.cuda.synchronize()
        per = {}
        for e in prof.events():
            if getattr(e, "device_type", None) is None or "cuda" not in str(e.device_type).lower():
                continue
            name = e.name
            if "lapis" not in name:
                continue
            short = name.split("(")[0].replace("void ", "").replace("lapis_b200::", "")
            c, t = per.get(short, (0, 0.0))
            per[short] = (c + 1, t + float(getattr(e, "device_time", 0.0) or
                                          getattr(e, "cuda_time", 0.0) or 0.0))
        if not per:
            return None
        total = sum(t for _, t in per.values()) or 1.0
        return {k: {"launches_per_step": c, "share": round(t / total, 4)}
                for k, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1])}
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--problem-size", dest="n", type=int, default=0,
                    help="problem size override")
    ap.add_argument("--cpu-rows", type=int, default=4_000_000)
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU time of the cpu_baseline sample (reps are added to reach it)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--vl", type=int, default=0,
                    help="SpMV: time the emitted-mapping vector kernel with this vector length")
    ap.add_argument("--mtx", default="", help="Matrix Market file for --workload mtx")
    ap.add_argument("--gemm-mode", default="auto", choices=["auto", "tf32x3", "dmma", "exact", "ozaki"])
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
    if hasattr(wl, "capture_graphs"):
        wl.capture_graphs()
        for _ in range(args.warmup):
            wl.step()
        torch.cuda.synchronize()
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_events = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
    per_step = []
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        ev0.record(stream)
        for s0, s1 in step_events:
            if wl.flush is None:
                # back-to-back steps bracketed by ev0 / ev1 only: an event pair
                # per step would add its own gaps to a ~20 us step (config 1)
                wl.step()
                continue
            wl.flush.fill_(1)
            s0.record(stream)
            wl.step()
            s1.record(stream)
            per_step.append((s0, s1))
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    # with an L2 flush between steps, the step time excludes the flush
    total = ev0.elapsed_time(ev1) / 1e3 / args.steps
    kern = [a.elapsed_time(b) / 1e3 for a, b in per_step] if per_step else [total]
    t_local = total if wl.flush is None else float(np.mean(kern))
    t = max_over_ranks(t_local, world)
    kern_avg = max_over_ranks(float(np.mean(kern)), world)
    scale = 1e9 if wl.unit == "GB/s" else 1e12
    value = wl.work_global() / t / scale
    pk = peaks()
    if wl.bound == "hbm":
        peak, punit, psrc = pk["hbm_gbs"], "GB/s", pk["source"] + " hbm_gbs (copy)"
    else:
        # tensor-bound: nominal B200 dense peaks (MEASURED_PEAKS has bf16 only)
        if wl.dtype == "f32":
            # dense TF32 runs at half the bf16 rate on B200; 3xTF32 issues 3
            peak = pk["bf16_tflops"] / 2.0 / 3.0
            psrc = f"{pk['source']} bf16_tflops / 2 (dense TF32 = bf16 / 2) / 3 (3xTF32 products)"
        else:
            peak, psrc = 40.0, "nominal FP64 tensor 40 TF"
        punit = "TFLOP/s"
    achieved = wl.work_local() / kern_avg / scale
    override = wl.roofline_override(kern_avg) if hasattr(wl, "roofline_override") else None
    traffic = None
    tfile = ROOT / "profiles" / f"traffic_{args.workload}.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get("dram_bytes_per_launch")
    exact_variant = (wl.exact_variant(max(3, args.steps // 2))
                     if hasattr(wl, "exact_variant") and not args.vl else None)
    census = launch_census(wl)
    wl.step()   # the parity sample below checks the headline kernel's output
    torch.cuda.synchronize()
    sharded_parity = None
    if world > 1 and hasattr(wl, "sharded_parity"):
        # this rank's rows of the sharded result against the unsharded
        # multiply of the whole matrix on the same device (small runs only)
        ok = wl.sharded_parity()
        if ok is not None:
            bad = torch.tensor([0.0 if ok else 1.0], dtype=torch.float64,
                               device="cpu" if dist.get_backend() == "gloo" else "cuda")
            dist.all_reduce(bad, op=dist.ReduceOp.MAX)
            sharded_parity = {"bitexact_vs_unsharded_all_ranks": bool(bad.item() == 0.0)}
    e2e_dt, hb, db = wl.e2e(args.e2e_steps, 2)
    e2e_dt = max_over_ranks(e2e_dt, world)
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": wl.unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 4),
        "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None, "dtype": wl.dtype,
        "data": getattr(wl, "data", "synthetic (device-generated inputs, seeded)"),
        "config": wl.config(),
        "roofline": ({**override, "traffic": traffic, "kernel": wl.kernel_name(),
                      "algorithmic_work_per_launch": wl.work_local()} if override else
                     {"bound": wl.bound, "achieved": round(achieved, 2), "peak": peak,
                      "unit": punit, "frac": round(achieved / peak, 4), "traffic": traffic,
                      "peak_source": psrc, "kernel": wl.kernel_name(),
                      "algorithmic_work_per_launch": wl.work_local()}),
        "e2e": {"value": round(wl.work_global() / e2e_dt / scale, 3), "unit": wl.unit,
                "h2d_bytes_per_step": hb, "d2h_bytes_per_step": db,
                "ms_per_step": round(e2e_dt * 1e3, 3),
                "path": getattr(wl, "e2e_path", "DualView lazy sync (inputs host-modified each "
                                "step) + C-ABI kernels + result read on the host"),
                **({"matches_device_result": wl.e2e_parity} if hasattr(wl, "e2e_parity") else {})},
        "gpu_launches": args.steps * (sum(v["launches_per_step"] for v in census.values())
                                      if census else wl.launches_per_step()),
        "gpu_launches_source": ("CUDA activity trace of one untimed step x steps" if census
                                else "static count per step x steps"),
        **({"kernels": census} if census else {}),
        **({getattr(wl, "variant_key", "exact_mode"): exact_variant} if exact_variant else {}),
        "clocks": clk.summary(),
        **({"sharded_parity": sharded_parity} if sharded_parity else {}),
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
