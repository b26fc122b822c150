#!/usr/bin/env python
"""Benchmark of the LAPIS hot path on B200 (contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W]
                    [--workload c5|c1|c3|c4|c2f32|c2f64|gemv|mtx] [--impl ours|reference]
                    [--extra c1,c2f32,...|none]

Default workload (BASELINE.json config 5, the largest single-GPU config and
the one the metric's multi-GPU scaling is quoted on): CSR SpMV fp64 on the
3-D 27-point stencil, n = 585 -> 200,201,625 rows, 5,386,984,777 nonzeros,
int64 rowptr / int32 colind, row-block sharded over the ranks with the halo
exchange of x (paper_2509_25605_b200/sharded.py).  A step is one SpMV over the
whole matrix.  Inputs (69 GB) exceed L2 (126 MB) many times, so no flush is
needed between steps.  At N = 1 the same line carries a `workloads` object with
the other configs measured in the same run (config 1 SpMV, config 2 matmul
f32 / f64, config 3 SpMM, config 4 GCN layer), each with its roofline, e2e,
CPU baseline and parity sample.

`value` is device-resident throughput (algorithmic bytes or flops / step time,
max over ranks); `e2e` repeats the step through the public DualView + C-ABI
path with the step's inputs copied host->device and the result device->host
every step (pinned host buffers).  `cpu_baseline` runs the reference's own
emitted Kokkos C++ on its serial stub (oracle/_ref) on a bounded sample of the
same workload — on all host cores (row blocks, bitwise identical) and on one
core — and doubles as the parity check of that sample against the GPU result.

Inputs: every random number comes from numpy generators defined in
synth_inputs.py (SURVEY 8(d) seeds), so the reference arm (`--impl
reference`) builds the very same sample on the host without importing this
backend; the stencil matrices are generated on the device by the backend and
on the host by the reference arm (same formula), so the parity sample also
pins the device generator at full scale.
"""
from __future__ import annotations

import argparse
import gc
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

import synth_inputs as S  # noqa: E402  (numpy only: shared by both arms)

METRIC = "SpMV/SpMM HBM GB/s (% of peak), matmul TFLOP/s, at 1/2/4/8 B200 vs CPU ref"
EXTRA_DEFAULT = "c1,c2f32,c2f64,c3,c4"


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
        self.path = Path(f"/tmp/lapis_clocks_{os.getpid()}_{time.monotonic_ns()}.csv")

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


# ------------------------------------------------- host inputs (both arms)
_MEMO: dict = {}


def memo(key, make):
    if key not in _MEMO:
        _MEMO[key] = make()
    return _MEMO[key]


def drop_memo():
    _MEMO.clear()
    gc.collect()


WORKLOAD_NAMES = {
    "c5": "config5: CSR SpMV fp64, 3-D 27-point stencil n={n}",
    "c1": "config1: CSR SpMV fp64, 2-D 5-point Laplacian n={n}",
    "c3": "config3: CSR x dense SpMM fp64, K=64, power-law (Chung-Lu, Pareto 2.5) {n} rows",
    "c4": "config4: GCN layer relu((A_hat X) W) fp32, power-law A_hat {n} rows, 64->64",
    "c2f32": "config2: dense linalg.matmul {n}^3 f32 (mode {mode})",
    "c2f64": "config2: dense linalg.matmul {n}^3 f64 (mode {mode})",
    "gemv": "matvec: linalg.matvec f64 {n} x {n} (row_fold_pipe_kernel, reference order)",
    "mtx": "matrix market SpMV fp64: {mtx}",
}
DEFAULT_N = {"c5": 585, "c1": 1000, "c3": 10_000_000, "c4": 1_000_000, "c2f32": 4096,
             "c2f64": 4096, "gemv": 16384, "mtx": 0}


class HostSample:
    """A bounded sample of a workload for the reference's CPU path: the
    emitted C++ on its serial stub (oracle/_ref), `run(reps, threads)` ->
    (output, seconds per rep); `region` tells the GPU arm which part of its
    own output the sample covers."""

    def __init__(self, run, work, desc, tol, region, max_threads=None):
        self.run, self.work, self.desc, self.tol = run, work, desc, tol
        self.region, self.max_threads = region, max_threads


def _stencil_sample(points, n, seed, rows_sample):
    from oracle import ref as R
    N = n ** 3 if points == 27 else n * n
    mid = N // 2
    a, b = (0, N) if N <= rows_sample else (mid - rows_sample // 2, mid + rows_sample // 2)
    rp, ci, v = S.stencil_rows(points, n, a, b, colind_dtype=np.int64)
    x = memo(("x", points, n, seed), lambda: S.stencil_x(points, n, seed))
    nnz = int(rp[-1])

    def run(reps, threads):
        return R.spmv_csr(rp, ci, v, x, reps=reps, threads=threads)

    work = nnz * 12 + (b - a + 1) * 8 + (b - a) * 8 * 2
    desc = (f"rows [{a}, {b}) of the same matrix ({nnz} nnz, host-generated): reference emitted "
            "Kokkos C++ (tests/fixtures/spmv.mlir, index colind) on its serial stub")
    return HostSample(run, work, desc, 1e-12, (a, b))


def powerlaw_spec(n, seed, mean=10.0):
    return memo(("spec", n, seed, mean), lambda: S.PowerLawSpec(n, mean=mean, seed=seed))


def _spmm_sample(n, k, seed, rows_sample):
    from oracle import ref as R
    spec = powerlaw_spec(n, seed)
    b = min(n, max(1, rows_sample // 40))
    rp, ci = S.powerlaw_structure_host(spec, rows=b)
    v = S.powerlaw_values(spec, 0, first=0, count=int(rp[-1]))
    X = memo(("X", n, k, seed), lambda: S.spmm_dense(n, k, seed))
    nnz = int(rp[-1])

    def run(reps, threads):
        return R.spmm_csr(rp, ci, v, X, reps=reps, threads=threads)

    work = nnz * 12 + (b + 1) * 8 + b * k * 8 * 2
    desc = (f"rows [0, {b}) of the same matrix ({nnz} nnz, host-generated): reference emitted "
            "Kokkos C++ of oracle/ir/spmm.mlir on its serial stub")
    return HostSample(run, work, desc, 1e-12, (0, b))


def gcn_host_inputs(n, f, seed):
    def make():
        spec = powerlaw_spec(n, seed)
        rp, ci = S.powerlaw_structure_host(spec)
        X, W = S.gcn_features(n, f, seed)
        return rp, ci, S.gcn_values_host(rp, ci), X, W
    return memo(("gcn", n, f, seed), make)


def _gcn_sample(n, f, seed, rows_sample, host=None):
    from oracle import ref as R
    rp_all, ci_all, v_all, X, W = host if host is not None else gcn_host_inputs(n, f, seed)
    b = min(n, max(1, rows_sample // 80))
    e = int(rp_all[b])
    rp, ci, v = rp_all[:b + 1].copy(), ci_all[:e], v_all[:e]

    def run(reps, threads):
        return R.gcn(rp, ci, v, X, W, reps=reps, threads=threads)

    work = e * 8 + (b + 1) * 8 + b * f * 4 * 3 + f * f * 4
    desc = (f"rows [0, {b}) ({e} nnz): reference emitted Kokkos C++ of oracle/ir/gcn_f32.mlir "
            "on its serial stub")
    return HostSample(run, work, desc, 1e-5, (0, b))


def _matmul_sample(n, dt, seed, rows_sample, threads_hint):
    from oracle import ref as R
    A, B = memo(("dense", n, np.dtype(dt).name, seed), lambda: S.dense_operands(n, dt, seed))
    rows = max(threads_hint, min(n, rows_sample // 250_000))
    Ar = np.ascontiguousarray(A[:rows])

    def run(reps, threads):
        return R.matmul(Ar, B, reps=reps, threads=threads)

    tag = "f32" if dt == np.float32 else "f64"
    desc = (f"rows [0, {rows}) of C: reference emitted Kokkos C++ of oracle/ir/matmul_{tag}.mlir "
            "(TeamPolicy nest) on its serial stub")
    return HostSample(run, 2.0 * rows * n * n, desc, 1e-5 if dt == np.float32 else 1e-12,
                      (0, rows))


def gemv_host(n):
    def make():
        g = np.random.default_rng(6)
        A = g.uniform(-1.0, 1.0, (n, n))
        x = g.uniform(-1.0, 1.0, n)
        return A, x
    return memo(("gemv", n), make)


def _gemv_sample(n, rows_sample):
    from oracle import ref as R
    A, x = gemv_host(n)
    rows = min(n, max(1, rows_sample // 4000))
    Ar = np.ascontiguousarray(A[:rows])

    def run(reps, threads):
        return R.matvec(Ar, x, reps=reps)

    desc = (f"rows [0, {rows}) of the same A: reference emitted Kokkos C++ of "
            "oracle/ir/matvec_f64.mlir on its serial stub")
    return HostSample(run, (rows * n + n + rows) * 8, desc, 1e-12, (0, rows), max_threads=1)


def _mtx_sample(path, rows_sample):
    from oracle import ref as R
    import scipy.io
    import scipy.sparse
    A = scipy.sparse.csr_matrix(scipy.io.mmread(path))
    A.sort_indices()
    b = min(A.shape[0], rows_sample)
    rp = A.indptr[:b + 1].astype(np.int64)
    ci = A.indices[:rp[-1]].astype(np.int64)
    v = A.data[:rp[-1]].astype(np.float64)
    x = np.random.default_rng(7).uniform(-1.0, 1.0, A.shape[1])

    def run(reps, threads):
        return R.spmv_csr(rp, ci, v, x, reps=reps, threads=threads)

    work = int(rp[-1]) * 12 + (b + 1) * 8 + b * 8 * 2
    desc = f"rows [0, {b}) ({int(rp[-1])} nnz): reference emitted Kokkos C++ on its serial stub"
    return HostSample(run, work, desc, 1e-12, (0, b))


def host_sample(key, args, n, threads) -> HostSample:
    if key == "c5":
        return _stencil_sample(27, n, 5, args.cpu_rows)
    if key == "c1":
        return _stencil_sample(5, n, 1, args.cpu_rows)
    if key == "c3":
        return _spmm_sample(n, 64, 1, args.cpu_rows)
    if key == "c4":
        return _gcn_sample(n, 64, 4, args.cpu_rows)
    if key in ("c2f32", "c2f64"):
        dt = np.float32 if key == "c2f32" else np.float64
        return _matmul_sample(n, dt, 3 if dt == np.float32 else 2, args.cpu_rows, threads)
    if key == "gemv":
        return _gemv_sample(n, args.cpu_rows)
    if key == "mtx":
        return _mtx_sample(args.mtx, args.cpu_rows)
    raise KeyError(key)


def time_cpu(sample: HostSample, threads: int, seconds: float, min_reps: int):
    """Median seconds per rep of the sample on `threads` host threads, with
    enough reps for about `seconds` of CPU work; returns (output, median, reps)."""
    out, times = sample.run(min_reps, threads)
    t = float(np.median(times))
    reps = int(min(2000, max(min_reps, np.ceil(seconds / max(t, 1e-6)))))
    if reps > min_reps:
        out, times = sample.run(reps, threads)
        t = float(np.median(times))
    return out, t, len(times)


def cpu_baseline(sample: HostSample, unit: str, threads: int, seconds: float, reps: int):
    """The reference CPU path on all host cores (row blocks on std::threads,
    bitwise identical to one thread) and on one core (the stub is
    serial by construction)."""
    from oracle import ref as R
    scale = 1e9 if unit == "GB/s" else 1e12
    cores = min(threads, sample.max_threads or threads)
    want, t, n = time_cpu(sample, cores, seconds, reps)
    base = {"value": round(sample.work / t / scale, 4), "unit": unit, "cores": cores,
            "kind": "reference", "sample": f"{sample.desc}, {cores} row blocks, median of {n} reps",
            "seconds_per_rep": t, "build": R.compile_flags()}
    if cores > 1:
        _, t1, n1 = time_cpu(sample, 1, seconds / 2, max(1, reps // 2))
        base["one_core"] = {"value": round(sample.work / t1 / scale, 4), "unit": unit,
                            "cores": 1, "seconds_per_rep": t1, "reps": n1}
    return base, want


# ------------------------------------------------------------------- workloads
class Workload:
    unit = "GB/s"
    bound = "hbm"
    dtype = "f64"
    flush = None
    scaling = "strong"
    key = ""

    def launches_per_step(self) -> int:
        return 1

    def gpu_region(self, region):
        raise NotImplementedError


class StencilSpmv(Workload):
    """Config 5 (default) / config 1: CSR SpMV fp64 on a stencil matrix."""

    def __init__(self, args, rank, world, points=27, n=585, x_seed=5):
        import paper_2509_25605_b200 as lb
        from paper_2509_25605_b200 import sharded
        self.key = "c5" if points == 27 else "c1"
        self.lb, self.args, self.rank, self.world = lb, args, rank, world
        self.points, self.n, self.x_seed = points, n, x_seed
        self.N = n ** 3 if points == 27 else n * n
        self.ranges = sharded.balanced_row_ranges(self.N, world)
        self.r0, self.r1 = self.ranges[rank]
        self.stream = torch.cuda.current_stream()
        self.rowptr, self.colind, self.values = lb.synth_stencil(points, n, self.r0, self.r1)
        self.nnz_local = int(self.rowptr[-1].item())
        self.x_host = memo(("x", points, n, x_seed), lambda: S.stencil_x(points, n, x_seed))
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
        return WORKLOAD_NAMES[self.key].format(n=self.n)

    def nnz_global(self):
        return S.stencil_nnz(self.points, self.n)

    def config(self):
        return stencil_config(self.key, self.points, self.n, self.x_seed, self.world)

    def extra_config(self):
        d = {}
        if self.graphs:
            d["launch"] = self.graph_note
        d["l2"] = ("inputs >> L2 (126 MB), no flush needed" if len(self.rot) == 1 else
                   f"inputs < L2: steps rotate over {len(self.rot)} device copies of the whole "
                   f"input ({len(self.rot) * self.work_local() / 1e6:.0f} MB > 3 x L2), no flush")
        return d

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
        if (self.group is not None and self.left is not None and self.rot_i == 0
                and self.left >= len(self.rot)):
            # the next len(rot) steps: one replay of the graph of all copies
            self.group.replay()
            self.group_left = len(self.rot)
        if self.left is not None:
            self.left -= 1
        g = self.graphs[self.rot_i] if self.graphs else None
        self.rot_i = (self.rot_i + 1) % len(self.rot)
        if self.group_left > 0:
            self.group_left -= 1          # covered by the group replay
        elif g is not None:
            g.replay()
        else:
            op.multiply(x, y, stream=self.stream)
        self.last_y = y

    graphs = None
    group = None          # graph of one multiply per rotation copy (launch-bound config 1)
    group_left = 0
    left = None           # timed steps still to run (plan_steps), None outside the timed loop

    def plan_steps(self, steps):
        """The timed loop announces its step count, so whole groups of
        len(rot) steps replay the group graph and only the rest replays
        single-step graphs: exactly `steps` multiplies run."""
        self.left = steps if self.group is not None else None

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
        group = None
        if os.environ.get("LAPIS_B200_BENCH_GROUP", "1") != "0":
            group = torch.cuda.CUDAGraph()
            with torch.cuda.graph(group, stream=side):
                for rp, ci, v, x, y, op in self.rot:
                    op.multiply(x, y, stream=side)
            for _ in range(2):    # upload + warm the group graph outside the timed steps
                group.replay()
        self.stream.wait_stream(side)
        torch.cuda.synchronize()
        self.graphs = graphs
        self.group = group
        self.graph_note = (f"each step replays a captured CUDA graph of the multiply ({len(graphs)} graphs, "
                           f"one per input copy)") if group is None else (f"the timed steps replay captured CUDA graphs: one graph of {len(graphs)} "
                           f"multiplies (one per input copy) per {len(graphs)} steps, single-multiply "
                           f"graphs for a remainder; launch_floor_us measured the same way")

    def sharded_parity(self):
        if self.N > 50_000_000:
            return None
        rp, ci, v = self.lb.synth_stencil(self.points, self.n)
        plan = self.lb.CsrPlan(rp)
        y = plan.spmv(ci, v, self.x)
        return bool(torch.equal(y[self.r0:self.r1], self.last_y))

    def launch_floor(self, steps):
        """Per-step cost of an EMPTY step with the same launch mechanism (the
        same graph grouping as the timed steps, each node one of our kernels
        on 1 element, replayed back to back): the fixed launch / ramp cost
        inside a ~20 us config-1 step.  None unless the steps replay graphs."""
        if not self.graphs:
            return None
        tiny_x = torch.zeros(1, dtype=torch.float64, device="cuda")
        tiny_y = torch.empty_like(tiny_x)
        side = torch.cuda.Stream()
        side.wait_stream(self.stream)
        nr = len(self.rot) if self.group is not None else 1
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            self.lb.relu(tiny_x, tiny_y, stream=side)
        grp = torch.cuda.CUDAGraph()   # the same grouping as the timed steps
        with torch.cuda.graph(grp, stream=side):
            for _ in range(nr):
                self.lb.relu(tiny_x, tiny_y, stream=side)
        self.stream.wait_stream(side)
        for _ in range(3):
            g.replay()
            grp.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(self.stream)
        for _ in range(steps // nr):
            grp.replay()
        for _ in range(steps % nr):
            g.replay()
        b.record(self.stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / 1e3 / steps

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
        out = {"value": round(self.work_global() / t / 1e9, 3), "unit": "GB/s",
               "frac": round(self.work_local() / t / 1e9 / peaks()["hbm_gbs"], 4),
               "ms_per_step": round(t * 1e3, 4),
               "kernel": "; ".join(names), "note": "bit-identical to the reference",
               "path": "reference-order CsrPlan: also what the emitted C++ seam LAPIS::spmv_csr "
                       "replays from its second call on (b200::CsrPlanCache, "
                       "include/lapis_b200_runtime.hpp)"}
        if self.world == 1:
            # the no-plan call the emitted C++'s LAPIS::spmv_csr makes
            # (lapis_b200_spmv_csr: structure pass + reference-order kernel)
            rp, ci, v, x, y, _ = self.rot[0]
            for _ in range(2):
                self.lb.spmv_csr(rp, ci, v, x, y, stream=self.stream)
            torch.cuda.synchronize()
            a.record(self.stream)
            for _ in range(steps):
                self.lb.spmv_csr(rp, ci, v, x, y, stream=self.stream)
            b.record(self.stream)
            torch.cuda.synchronize()
            t1 = a.elapsed_time(b) / 1e3 / steps
            out["no_plan"] = {"value": round(self.work_global() / t1 / 1e9, 3), "unit": "GB/s",
                              "ms_per_step": round(t1 * 1e3, 4),
                              "path": "lapis_b200_spmv_csr without a plan: the seam's first "
                                      "call, or a call after rowptr was modified; bit-identical"}
        return out

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

    def gpu_region(self, region):
        a, b = region
        if a < self.r0 or b > self.r1:
            return None
        return self.last_y[a - self.r0:b - self.r0].cpu().numpy()


def stencil_config(key, points, n, seed, world):
    return {"workload": WORKLOAD_NAMES[key].format(n=n),
            "rows": n ** 3 if points == 27 else n * n, "nnz": S.stencil_nnz(points, n),
            "index_layout": "rowptr int64, colind int32", "x": f"U(-1,1) numpy seed {seed}",
            "sharding": f"row blocks x{world}, halo exchange of x (NCCL P2P)",
            "parallelism": f"rowblock{world}"}


class MtxSpmv(Workload):
    """CSR SpMV fp64 on a Matrix Market file (--mtx; the paper's SuiteSparse
    runs): read natively (paper_2509_25605_b200/mmio.py),
    planned once, x U(-1,1) seed 7.  N > 1: independent replicas."""

    scaling = "weak"
    key = "mtx"
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
        return WORKLOAD_NAMES["mtx"].format(mtx=Path(self.path).name)

    def config(self):
        return {"workload": self.name, "parallelism": "replica"}

    def extra_config(self):
        return {"rows": self.N, "cols": self.ncols, "nnz": self.nnz,
                "index_layout": "rowptr int64, colind int32",
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

    def gpu_region(self, region):
        a, b = region
        return self.y[a:b].cpu().numpy()


class PowerLawSpmm(Workload):
    """Config 3: CSR x dense SpMM fp64, K = 64, Chung-Lu power-law matrix
    (synth_inputs.PowerLawSpec: n = 10M, seed 1 -> nnz 99,891,191, longest row
    117,683; structure built on the device, values and X from numpy).

    N > 1: the SAME global matrix, row-block sharded
    (sharded.RowBlockSpmm: rank r owns rows [r*c, r*c + c), c = ceil(N / world),
    and the matching rows of X and Y); a step is the NCCL all-gather of X
    followed by the local SpMM (strong scaling, total work fixed).  The
    "x_replicated" variant times the local SpMM alone (features resident on
    every GPU, the GCN case)."""

    key = "c3"
    scaling = "strong"
    variant_key = "variants"

    def __init__(self, args, rank, world, n=10_000_000, k=64, mean=10.0, seed=1):
        import paper_2509_25605_b200 as lb
        from paper_2509_25605_b200 import sharded
        self.lb, self.args, self.world, self.rank = lb, args, world, rank
        self.N, self.k, self.seed = n, k, seed
        self.stream = torch.cuda.current_stream()
        spec = powerlaw_spec(n, seed, mean)
        rowptr, colind = S.powerlaw_structure_device(spec)
        self.nnz_global_ = int(rowptr[-1].item())
        values = torch.from_numpy(S.powerlaw_values(spec, self.nnz_global_)).cuda()
        lens = rowptr[1:] - rowptr[:-1]
        self.max_len = int(lens.max().item())
        self.median_len = float(lens.double().median().item())
        del lens
        X_host = memo(("X", n, k, seed), lambda: S.spmm_dense(n, k, seed))
        self.r0, self.r1 = sharded.equal_row_ranges(n, world)[rank]
        self.full = ((rowptr, colind, values, torch.from_numpy(X_host).cuda())
                     if world > 1 and n * k * 8 < (2 << 30) else None)
        if world > 1:
            a, b = int(rowptr[self.r0].item()), int(rowptr[self.r1].item())
            self.rowptr = (rowptr[self.r0:self.r1 + 1] - a).contiguous()
            self.colind, self.values = colind[a:b].contiguous(), values[a:b].contiguous()
            del rowptr, colind, values
        else:
            self.rowptr, self.colind, self.values = rowptr, colind, values
        self.nnz = int(self.rowptr[-1].item())
        # an SpMM plan pins the most referenced X rows in L2 (LAPIS_BENCH_SPMM_PLAN=0: off)
        self.use_plan = os.environ.get("LAPIS_BENCH_SPMM_PLAN", "1") == "1"
        self.op = sharded.RowBlockSpmm(self.rowptr, self.colind, self.values, n, k, rank, world,
                                       plan=self.use_plan,
                                       hot_bytes=int(os.environ.get("LAPIS_BENCH_SPMM_HOT_MB", "0")) << 20)
        self.op.x_local.copy_(torch.from_numpy(X_host[self.r0:self.r1]))
        self.op.gather()
        self.X = self.op.X_full[:n]
        self.Y = torch.empty((self.r1 - self.r0, k), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()

    def config(self):
        return powerlaw_config("c3", self.N, self.k, self.seed, self.world)

    def extra_config(self):
        return {"nnz": self.nnz_global_, "max_row": self.max_len, "median_row": self.median_len,
                "l2": "inputs >> L2",
                "spmm_plan": self.op.plan.info() if self.op.plan is not None else None,
                **({"gather": f"NCCL all-gather of X ({self.op.gather_bytes / 1e9:.2f} GB "
                              "received per rank per step) then the local SpMM"}
                   if self.world > 1 else {})}

    def _work(self, nnz, rows):
        # nnz*(s_v+s_i) + (N+1)*s_p + Ncols*K*s_v + N*K*s_v
        return nnz * 12 + (rows + 1) * 8 + self.N * self.k * 8 + rows * self.k * 8

    def work_global(self):
        return self._work(self.nnz_global_, self.N)

    def work_local(self):
        # the local SpMM's algorithmic bytes (its X gathers can touch every row of X)
        return self._work(self.nnz, self.r1 - self.r0)

    def launches_per_step(self):
        return 4 if self.max_len > 2048 else 2

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

    def gpu_region(self, region):
        a, b = region
        if a < self.r0 or b > self.r1:
            return None
        return self.Y[a - self.r0:b - self.r0].cpu().numpy()


def powerlaw_config(key, n, k, seed, world, extra=None):
    d = {"workload": WORKLOAD_NAMES[key].format(n=n), "rows": n, "k": k,
         "index_layout": "rowptr int64, colind int32",
         "generator": f"synth_inputs.PowerLawSpec(n={n}, mean=10, seed={seed}) (numpy draws)",
         "sharding": (f"row blocks x{world}, NCCL all-gather of the dense operand" if world > 1
                      else "none"),
         "parallelism": f"rowblock{world}"}
    d.update(extra or {})
    return d


class DenseMatmul(Workload):
    """Config 2: dense linalg.matmul 4096^3 (f32: sign-gated Ozaki, 3xTF32 for
    operands with negative entries; f64: certified Ozaki on the int8 tensor cores).  N > 1: row blocks of A
    and C (sharded.RowBlockGemm), B replicated by one broadcast when the
    operator is built (not part of a step); strong scaling."""

    unit = "TFLOP/s"
    bound = "tensor"
    scaling = "strong"

    def __init__(self, args, rank, world, dt=torch.float32, n=4096):
        import paper_2509_25605_b200 as lb
        from paper_2509_25605_b200 import sharded
        self.lb, self.args, self.world, self.n, self.dt = lb, args, world, n, dt
        self.dtype = "f32" if dt == torch.float32 else "f64"
        self.key = "c2" + self.dtype
        self.stream = torch.cuda.current_stream()
        npdt = np.float32 if dt == torch.float32 else np.float64
        seed = 3 if dt == torch.float32 else 2
        A, B = memo(("dense", n, np.dtype(npdt).name, seed),
                    lambda: S.dense_operands(n, npdt, seed))
        self.r0, self.r1 = sharded.equal_row_ranges(n, world)[rank]
        self.A = torch.from_numpy(A[self.r0:self.r1]).cuda()
        Bd = (torch.from_numpy(B).cuda() if rank == 0 else
              torch.empty((n, n), dtype=dt, device="cuda"))
        self.op = sharded.RowBlockGemm(self.A, Bd, n, rank, world)
        self.B = self.op.B
        self.C = torch.empty((self.r1 - self.r0, n), dtype=dt, device="cuda")
        self.mode = args.gemm_mode
        if 3 * n * n * (4 if dt == torch.float32 else 8) < (256 << 20):
            self.flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()

    def config(self):
        return matmul_config(self.key, self.n, self.mode, self.world)

    def extra_config(self):
        return {"l2": "L2 flushed between steps" if self.flush is not None else "working set > L2"}

    def work_global(self):
        return 2.0 * self.n ** 3

    def work_local(self):
        return 2.0 * (self.r1 - self.r0) * self.n * self.n

    def effective_mode(self):
        if self.mode != "auto":
            return self.mode
        if self.dt == torch.float32:
            # AUTO f32: the sign-gated Ozaki path for non-negative operands
            # (config 2's U(0, 1) inputs) while k is in its certified range
            return "ozaki" if 3 * self.n * 65025 < 2 ** 31 else "tf32x3"
        return "ozaki" if self.n * 9.0 * 2.0 ** -56 <= 0.75e-12 else "dmma"

    def kernel_name(self):
        m = self.effective_mode()
        names = {"tf32x3": "gemm_tf32x3_kernel (tcgen05 kind::tf32, 3xTF32)",
                 "dmma": "gemm_dmma_kernel (DMMA m8n8k4)",
                 "exact": "gemm_exact_kernel (reference order)",
                 "ozaki": ("gemm_ozaki_2p_kernel (tcgen05 kind::i8, two-pass Ozaki, certified, "
                           "CTA pairs on cta_group::2 MMAs, M = 256)"
                           if self.dt == torch.float64 and self.n * 9.0 * 2.0 ** -56 <= 0.75e-12
                           else "gemm_ozaki_2p_kernel<float> (tcgen05 kind::i8, one-pass Ozaki, 3 digits, "
                           "certified, sign-gated, CTA pairs on cta_group::2 MMAs)" if self.dt == torch.float32
                           else "gemm_ozaki_kernel (tcgen05 kind::i8, Ozaki digits, certified)")}
        return f"gemm<{self.dtype}> mode={self.mode} -> {names[m]}"

    def roofline_override(self, kern_avg):
        """The Ozaki kernel runs int8 MMAs: its roofline is the int8 tensor
        peak (2x the measured dense bf16 rate), counted in int8 ops."""
        if self.effective_mode() != "ozaki":
            return None
        S_ = (8 if self.n * 9.0 * 2.0 ** -56 <= 0.75e-12 else 9) if self.dt == torch.float64 else 3
        products = S_ * (S_ + 1) // 2
        ops = products * self.work_local()
        pk = peaks()
        peak = 2.0 * pk["bf16_tflops"]
        achieved = ops / kern_avg / 1e12
        return {"bound": "tensor", "achieved": round(achieved, 2), "peak": round(peak, 1),
                "unit": "TOPS (int8)", "frac": round(achieved / peak, 4),
                "peak_source": f"2 x {pk['source']} bf16_tflops (dense int8 = 2x bf16 on B200)",
                "int8_products": products, "ops_per_launch": ops}

    def step(self):
        self.op.multiply(self.C, mode=self.mode, stream=self.stream)

    def sharded_parity(self):
        if self.world == 1:
            return None
        A, _ = _MEMO[("dense", self.n, "float32" if self.dt == torch.float32 else "float64",
                      3 if self.dt == torch.float32 else 2)]
        ref = self.lb.gemm(torch.from_numpy(A).cuda(), self.B, mode=self.mode)
        return bool(torch.equal(ref[self.r0:self.r1], self.C))

    def e2e(self, steps, warmup):
        """This rank's rows of A and the (replicated) B host-modified every
        step, C's row block read back."""
        from paper_2509_25605_b200.dualview import DualView
        a = DualView.from_host(self.A.cpu(), "A", device_buffer=self.A)
        b = DualView.from_host(self.B.cpu(), "B", device_buffer=self.B)
        c = DualView.allocate(tuple(self.C.shape), self.dt, "C")

        def one():
            a.modify_host()
            b.modify_host()
            a.sync_device(self.stream)
            b.sync_device(self.stream)
            self.lb.gemm(a.device_view(), b.device_view(), c.device_view(), mode=self.mode,
                         stream=self.stream)
            c.modify_device()
            c.sync_host(self.stream)

        return timed_e2e(one, steps, warmup, self.world), a.nbytes + b.nbytes, c.nbytes

    def gpu_region(self, region):
        a, b = region
        if a < self.r0 or b > self.r1:
            return None
        return self.C[a - self.r0:b - self.r0].cpu().numpy()


def matmul_config(key, n, mode, world):
    f32 = key.endswith("f32")
    return {"workload": WORKLOAD_NAMES[key].format(n=n, mode=mode), "m": n, "n": n, "k": n,
            "inputs": "U(0,1) numpy seed 3" if f32 else "U(-1,1) numpy seed 2",
            "sharding": (f"row blocks of A and C x{world}; B replicated by one NCCL broadcast "
                         "when the operator is built (outside the timed steps)" if world > 1
                         else "none"),
            "parallelism": f"rowblock{world}"}


class GcnLayer(Workload):
    """Config 4: GCN layer H = relu((A_hat X) W), fp32, A_hat = D^-1/2 A D^-1/2 of the
    config-3 power-law generator at 1M rows (seed 4), X [N, 64] U(0,1), W [64, 64]
    U(-1/8, 1/8) (torch Linear default bound for fan-in 64).  N > 1: row blocks of
    A_hat and H, one all-gather of X per step, W broadcast once
    (sharded.RowBlockGcn)."""

    key = "c4"
    dtype = "f32"
    scaling = "strong"

    def __init__(self, args, rank, world, n=1_000_000, f=64, seed=4):
        import paper_2509_25605_b200 as lb
        from paper_2509_25605_b200 import sharded
        self.lb, self.args, self.world, self.N, self.f, self.seed = lb, args, world, n, f, seed
        self.stream = torch.cuda.current_stream()
        spec = powerlaw_spec(n, seed)
        rowptr, colind = S.powerlaw_structure_device(spec)
        rp_h, ci_h = rowptr.cpu().numpy(), colind.cpu().numpy()
        X, W = S.gcn_features(n, f, seed)
        vals_h = S.gcn_values_host(rp_h, ci_h)
        _MEMO[("gcn", n, f, seed)] = (rp_h, ci_h, vals_h, X, W)
        values = torch.from_numpy(vals_h).cuda()
        self.nnz_global_ = int(rp_h[-1])
        self.max_len = int(np.diff(rp_h).max())
        self.r0, self.r1 = sharded.equal_row_ranges(n, world)[rank]
        if world > 1:
            a, b = int(rp_h[self.r0]), int(rp_h[self.r1])
            self.rowptr = (rowptr[self.r0:self.r1 + 1] - a).contiguous()
            self.colind, self.values = colind[a:b].contiguous(), values[a:b].contiguous()
            del rowptr, colind, values
        else:
            self.rowptr, self.colind, self.values = rowptr, colind, values
        self.nnz = int(self.rowptr[-1].item())
        Wd = torch.from_numpy(W).cuda() if rank == 0 else torch.empty((f, f), device="cuda")
        self.op = sharded.RowBlockGcn(self.rowptr, self.colind, self.values, Wd, n, rank, world)
        self.op.x_local.copy_(torch.from_numpy(X[self.r0:self.r1]))
        self.op.gather()
        self.X = self.op.spmm.X_full[:n]
        self.W = self.op.W
        self.H = torch.empty((self.r1 - self.r0, f), dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()

    def config(self):
        return powerlaw_config("c4", self.N, self.f, self.seed, self.world,
                               {"features": self.f,
                                "bytes": "compulsory: A_hat + X + W + H (no A_hat X intermediate)"})

    def extra_config(self):
        return {"nnz": self.nnz_global_, "max_row": self.max_len, "l2": "inputs > L2 (X 256 MB)"}

    def work_local(self):
        # compulsory bytes of the layer: A_hat (int32 colind + f32 values, int64
        # rowptr), X, W read once, H written once.  The A_hat X intermediate is
        # not counted
        f, rows = self.f, self.r1 - self.r0
        return self.nnz * 8 + (rows + 1) * 8 + self.N * f * 4 + f * f * 4 + rows * f * 4

    def work_global(self):
        f, n = self.f, self.N
        return self.nnz_global_ * 8 + (n + 1) * 8 + n * f * 4 + f * f * 4 + n * f * 4

    def launches_per_step(self):
        return 4 if self.max_len > 2048 else 3

    def kernel_name(self):
        return ("spmm_batch_kernel<float> + spmm_seq_long_pipe_kernel (exact-order hub rows, "
                "16-column groups) + dense stage 2 with the ReLU fused")

    def step(self):
        self.op.multiply(self.H, stream=self.stream)

    def sharded_parity(self):
        if self.world == 1:
            return None
        rp, ci, v, X, W = _MEMO[("gcn", self.N, self.f, self.seed)]
        H = self.lb.gcn_layer(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(),
                              torch.from_numpy(v).cuda(), self.X, self.W)
        return bool(torch.equal(H[self.r0:self.r1], self.H))

    def e2e(self, steps, warmup):
        """This rank's rows of X (node features) host-modified every step (then
        the all-gather when N > 1), H's row block read back."""
        from paper_2509_25605_b200.dualview import DualView
        xs = DualView.from_host(self.op.x_local.cpu(), "X", device_buffer=self.op.x_local)
        hs = DualView.allocate(tuple(self.H.shape), torch.float32, "H")

        def one():
            xs.modify_host()
            xs.sync_device(self.stream)
            self.op.multiply(hs.device_view(), stream=self.stream)
            hs.modify_device()
            hs.sync_host(self.stream)

        return timed_e2e(one, steps, warmup, self.world), xs.nbytes, hs.nbytes

    def gpu_region(self, region):
        a, b = region
        if a < self.r0 or b > self.r1:
            return None
        return self.H[a - self.r0:b - self.r0].cpu().numpy()


class DenseMatvec(Workload):
    """linalg.matvec / LAPIS::gemv (fixture tests/fixtures/matvec_f64.mlir
    scaled up): y = A x, A 16384 x 16384 f64 U(-1,1) numpy seed 6 (2.1 GB > L2, no
    flush needed), folded in the reference order (bit-identical).  N > 1:
    independent replicas."""

    key = "gemv"
    scaling = "weak"

    def __init__(self, args, rank, world, n=16384):
        import paper_2509_25605_b200 as lb
        self.lb, self.args, self.world, self.n = lb, args, world, n
        self.stream = torch.cuda.current_stream()
        A, x = gemv_host(n)
        self.A = torch.from_numpy(A).cuda()
        self.x = torch.from_numpy(x).cuda()
        self.y = torch.empty(n, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()

    def config(self):
        return {"workload": WORKLOAD_NAMES["gemv"].format(n=self.n), "rows": self.n,
                "cols": self.n, "parallelism": "replica"}

    def extra_config(self):
        return {"l2": "A 2.1 GB >> L2"}

    def work_local(self):
        return (self.n * self.n + 2 * self.n) * 8

    def work_global(self):
        return self.work_local() * self.world

    def kernel_name(self):
        return "row_fold_pipe_kernel<double, DOT, 16-byte> (32 rows per CTA, 3-stage cp.async ring)"

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

    def gpu_region(self, region):
        a, b = region
        return self.y[a:b].cpu().numpy()


WORKLOADS = {
    "c5": lambda args, r, w, n: StencilSpmv(args, r, w, 27, n, x_seed=5),
    "c1": lambda args, r, w, n: StencilSpmv(args, r, w, 5, n, x_seed=1),
    "c3": lambda args, r, w, n: PowerLawSpmm(args, r, w, n),
    "c2f32": lambda args, r, w, n: DenseMatmul(args, r, w, torch.float32, n),
    "c2f64": lambda args, r, w, n: DenseMatmul(args, r, w, torch.float64, n),
    "c4": lambda args, r, w, n: GcnLayer(args, r, w, n),
    "mtx": lambda args, r, w, n: MtxSpmv(args, r, w),
    "gemv": lambda args, r, w, n: DenseMatvec(args, r, w, n),
}
UNITS = {"c2f32": "TFLOP/s", "c2f64": "TFLOP/s"}
DTYPES = {"c2f32": "f32", "c4": "f32"}
SCALING = {"gemv": "weak", "mtx": "weak"}


def static_config(key, args, n, world):
    """The config object of a workload without building it (the reference arm
    reports the same config as the B200 arm)."""
    if key in ("c5", "c1"):
        return stencil_config(key, 27 if key == "c5" else 5, n, 5 if key == "c5" else 1, world)
    if key == "c3":
        return powerlaw_config("c3", n, 64, 1, world)
    if key == "c4":
        return powerlaw_config("c4", n, 64, 4, world,
                               {"features": 64,
                                "bytes": "compulsory: A_hat + X + W + H (no A_hat X intermediate)"})
    if key in ("c2f32", "c2f64"):
        return matmul_config(key, n, args.gemm_mode, world)
    if key == "gemv":
        return {"workload": WORKLOAD_NAMES["gemv"].format(n=n), "rows": n, "cols": n,
                "parallelism": "replica"}
    return {"workload": WORKLOAD_NAMES["mtx"].format(mtx=Path(args.mtx).name),
            "parallelism": "replica"}


def run_reference_arm(args, rank, world):
    """The reference's own CPU path (oracle/_ref: its emitted Kokkos C++ on its
    serial stub) on the host cores, over a bounded sample of the same workload
    built on the host from synth_inputs — no part of the B200 backend is
    imported or loaded.  `value` uses every host core (row blocks, bitwise
    identical to one thread); `one_core` is the stub as shipped (serial)."""
    if rank != 0:
        return
    from oracle import ref as R
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    key = args.workload
    n = args.n or DEFAULT_N[key]
    threads = os.cpu_count() or 1
    sample = host_sample(key, args, n, threads)
    cores = min(threads, sample.max_threads or threads)
    unit = UNITS.get(key, "GB/s")
    scale = 1e9 if unit == "GB/s" else 1e12
    _, times = sample.run(args.warmup + args.steps, cores)
    times = times[args.warmup:]
    t = float(np.mean(times))
    value = sample.work / t / scale
    one = None
    if cores > 1:
        reps1 = max(1, min(args.steps, int(np.ceil(20.0 / max(t * cores, 1e-6)))))
        _, t1 = sample.run(reps1 + 1, 1)
        one = float(np.mean(t1[1:])) if len(t1) > 1 else float(t1[0])
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": unit,
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(t * 1e3, 4), "higher_is_better": True,
           "scaling": SCALING.get(key, "strong"), "vs_baseline": None,
           "dtype": DTYPES.get(key, "f64"), "data": "synthetic (numpy-seeded, host-generated)",
           "config": static_config(key, args, n, world),
           "cpu_baseline": {"value": round(value, 4), "unit": unit, "cores": cores,
                            "kind": "reference", "sample": f"{sample.desc}, {cores} row blocks",
                            "build": R.compile_flags(),
                            **({"one_core": {"value": round(sample.work / one / scale, 4),
                                             "unit": unit, "cores": 1,
                                             "ms_per_step": round(one * 1e3, 4)}}
                               if one else {})},
           "e2e": {"value": round(value, 4), "unit": unit, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def _short_name(name: str) -> str:
    return name.split("(")[0].replace("void ", "").replace("lapis_b200::", "")


GRAPH_CENSUS_ERR: list = []


def graph_census(wl):
    """Kernels of one step, read from a CUDA graph capture of that step
    (lapis_b200_graph_kernels walks the captured graph's kernel nodes): exact
    launch counts per kernel, no tracer involved.  None when the step cannot
    be captured."""
    import ctypes as C
    from paper_2509_25605_b200 import _capi
    side = torch.cuda.Stream()
    old_stream, old_graphs = wl.stream, getattr(wl, "graphs", None)
    g = torch.cuda.CUDAGraph(keep_graph=True)
    try:
        torch.cuda.synchronize()
        side.wait_stream(torch.cuda.current_stream())
        wl.stream = side
        if old_graphs is not None:
            wl.graphs = None
        with torch.cuda.graph(g, stream=side):
            wl.step()
        buf = C.create_string_buffer(1 << 16)
        n = C.c_int64()
        rc = _capi.lib().lapis_b200_graph_kernels(C.c_void_p(g.raw_cuda_graph()), buf, len(buf),
                                                 C.byref(n))
        if rc != 0:
            return None
        names = [x for x in buf.value.decode().split("\n") if x]
        try:
            dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True,
                                 text=True, timeout=30).stdout.split("\n")
            names = [d or m for d, m in zip(dem, names)]
        except (OSError, subprocess.SubprocessError):
            pass
        per = {}
        for nm in names:
            k = _short_name(nm)
            per[k] = per.get(k, 0) + 1
        return per
    except Exception as e:
        GRAPH_CENSUS_ERR.append(f"{type(e).__name__}: {e}"[:200])
        return None
    finally:
        wl.stream = old_stream
        if old_graphs is not None:
            wl.graphs = old_graphs
        try:
            g.reset()
        except Exception:
            pass
        torch.cuda.synchronize()


def profiler_census(wl):
    """Launch counts and each kernel's share of one untimed step's device time
    from the CUDA activity tracer (CUPTI via torch.profiler); (None, None)
    when unavailable."""
    try:
        import warnings
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                wl.step()
                torch.cuda.synchronize()
        cnt, per = {}, {}
        for e in prof.events():
            if getattr(e, "device_type", None) is None or "cuda" not in str(e.device_type).lower():
                continue
            if "lapis" not in e.name:
                continue
            k = _short_name(e.name)
            cnt[k] = cnt.get(k, 0) + 1
            per[k] = per.get(k, 0.0) + float(getattr(e, "device_time", 0.0) or
                                             getattr(e, "cuda_time", 0.0) or 0.0)
        total = sum(per.values())
        return (cnt or None), ({k: v / total for k, v in per.items()} if total > 0 else None)
    except Exception:
        return None, None


def launch_census(wl):
    """How many of OUR kernels (namespace lapis_b200 / NVRTC lapis_*) one step
    launches — from a graph capture of the step when it can be captured, else
    from the activity tracer — and, where the tracer saw them, each one's
    share of the step's device time."""
    counts = graph_census(wl)
    pcounts, shares = profiler_census(wl)
    src = "CUDA graph capture of one untimed step (kernel nodes) x steps"
    if counts:
        counts = {k: c for k, c in counts.items() if "lapis" in k}
    if not counts:
        counts, src = pcounts, "CUDA activity trace of one untimed step x steps" + (
            f" (graph capture failed: {GRAPH_CENSUS_ERR[-1]})" if GRAPH_CENSUS_ERR else "")
    if not counts:
        return None, None
    shares = shares or {}
    return ({k: {"launches_per_step": c,
                 "share": round(shares[k], 4) if k in shares else None}
             for k, c in sorted(counts.items(), key=lambda kv: -shares.get(kv[0], 0.0))}, src)


def measure(wl, args, rank, world, local, steps, warmup, cpu_seconds, with_cpu=True):
    """Warm-up, K timed steps (CUDA events on the launching stream, max over
    ranks), roofline of the dominant kernel, e2e, launch census, the CPU
    baseline and the parity sample.  Returns the JSON object of one workload."""
    stream = wl.stream
    for _ in range(warmup):
        wl.step()
    torch.cuda.synchronize()
    if hasattr(wl, "capture_graphs"):
        wl.capture_graphs()
        for _ in range(warmup):
            wl.step()
        torch.cuda.synchronize()
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_events = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(steps)]
    if hasattr(wl, "plan_steps") and wl.flush is None:
        wl.rot_i = 0
        wl.plan_steps(steps)
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
    if hasattr(wl, "plan_steps"):
        wl.left = None
    # with an L2 flush between steps, the step time excludes the flush
    total = ev0.elapsed_time(ev1) / 1e3 / steps
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
    tfile = ROOT / "profiles" / f"traffic_{wl.key}.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get("dram_bytes_per_launch")
    floor = wl.launch_floor(steps) if hasattr(wl, "launch_floor") else None
    exact_variant = (wl.exact_variant(max(3, steps // 2))
                     if hasattr(wl, "exact_variant") and not args.vl else None)
    census, census_src = launch_census(wl)
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
        "value": round(value, 3), "unit": wl.unit, "ms_per_step": round(t * 1e3, 4),
        "steps": steps, "warmup": warmup, "scaling": wl.scaling, "dtype": wl.dtype,
        "config": wl.config(), "workload_detail": wl.extra_config(),
        "roofline": ({**override, "traffic": traffic, "kernel": wl.kernel_name(),
                      "algorithmic_work_per_launch": wl.work_local()} if override else
                     {"bound": wl.bound, "achieved": round(achieved, 2), "peak": peak,
                      "unit": punit, "frac": round(achieved / peak, 4), "traffic": traffic,
                      "peak_source": psrc, "kernel": wl.kernel_name(),
                      "algorithmic_work_per_launch": wl.work_local(),
                      **({"launch_floor_us": round(floor * 1e6, 3),
                          "frac_floor_corrected": round(wl.work_local() / max(kern_avg - floor, 1e-9)
                                                        / scale / peak, 4)}
                         if floor else {})}),
        "e2e": {"value": round(wl.work_global() / e2e_dt / scale, 3), "unit": wl.unit,
                "h2d_bytes_per_step": hb, "d2h_bytes_per_step": db,
                "ms_per_step": round(e2e_dt * 1e3, 3),
                "path": getattr(wl, "e2e_path", "DualView lazy sync (inputs host-modified each "
                                "step) + C-ABI kernels + result read on the host"),
                **({"matches_device_result": wl.e2e_parity} if hasattr(wl, "e2e_parity") else {})},
        "gpu_launches": steps * (sum(v["launches_per_step"] for v in census.values())
                                 if census else wl.launches_per_step()),
        "gpu_launches_source": census_src or "static count per step x steps",
        **({"kernels": census} if census else {}),
        **({getattr(wl, "variant_key", "exact_mode"): exact_variant} if exact_variant else {}),
        "clocks": clk.summary(),
        **({"sharded_parity": sharded_parity} if sharded_parity else {}),
    }
    if rank == 0 and world == 1 and with_cpu and not args.no_cpu:
        from oracle import ref as R
        if not R.available():
            out["cpu_baseline"] = {"unavailable": "oracle/_ref not built"}
        else:
            threads = os.cpu_count() or 1
            sample = host_sample(wl.key, args, wl.n_arg, threads)
            base, want = cpu_baseline(sample, wl.unit, threads, cpu_seconds, args.cpu_reps)
            out["cpu_baseline"] = base
            got = wl.gpu_region(sample.region)
            if got is not None:
                out["parity"] = {"sample_elements": int(np.asarray(want).size),
                                 "sample": sample.desc.split(":")[0],
                                 **parity_report(got, want, sample.tol)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--problem-size", dest="n", type=int, default=0,
                    help="problem size override")
    ap.add_argument("--extra", default=None,
                    help="comma list of workloads measured in the same run after the headline "
                         f"(N = 1 default for c5: {EXTRA_DEFAULT}; 'none' to skip)")
    ap.add_argument("--cpu-rows", type=int, default=4_000_000)
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU time of the headline cpu_baseline sample")
    ap.add_argument("--extra-cpu-seconds", type=float, default=4.0)
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
    n = args.n or DEFAULT_N[args.workload]
    wl = WORKLOADS[args.workload](args, rank, world, n)
    wl.n_arg = n
    head = measure(wl, args, rank, world, local, args.steps, args.warmup, args.cpu_seconds)
    del wl
    drop_memo()
    torch.cuda.empty_cache()
    extras = args.extra
    if extras is None:
        extras = EXTRA_DEFAULT if (args.workload == "c5" and world == 1 and not args.n
                                   and not args.vl) else "none"
    workloads = {}
    for key in [k for k in extras.split(",") if k and k != "none"]:
        try:
            sub = WORKLOADS[key](args, rank, world, DEFAULT_N[key])
            sub.n_arg = DEFAULT_N[key]
            # config 1's ~18 us steps: at least 200 of them, so the host's
            # submission of the first graph (the GPU idles behind ev0 until
            # it arrives) is not a tenth of the timed region
            wsteps = max(args.steps, 200) if key == "c1" else args.steps
            workloads[key] = measure(sub, args, rank, world, local, wsteps, args.warmup,
                                     args.extra_cpu_seconds)
            del sub
        except Exception as e:   # one failing extra must not cost the headline line
            workloads[key] = {"error": f"{type(e).__name__}: {e}"}
        drop_memo()
        torch.cuda.empty_cache()
    out = {"metric": METRIC, "value": head.pop("value"), "unit": head.pop("unit"),
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": head.pop("ms_per_step"), "higher_is_better": True,
           "scaling": head.pop("scaling"), "vs_baseline": None, "dtype": head.pop("dtype"),
           "data": "synthetic (numpy-seeded inputs, synth_inputs.py; stencils generated on the "
                   "device)",
           **{k: v for k, v in head.items() if k not in ("steps", "warmup")}}
    if workloads:
        out["workloads"] = workloads
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
