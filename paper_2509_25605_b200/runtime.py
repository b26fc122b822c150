"""B200 executor of LAPIS programs: the drop-in for ``lapis.interp.run``.

``run(program, entry, inputs, config)`` takes the same arguments as the
reference's compile-and-call API (interp.py:1037-1039) — a parsed (usually
pipeline-lowered) ``lapis.ir.Program``, the entry function name, numpy inputs
matching the signature, an optional ``ExecConfig`` — and returns the same
``RunResult(outputs, trace, counters)``, so ``diff_outputs`` and the
reference's own assertions apply unchanged.  What differs is where the work
runs:

* every device kernel — top-level ``kokkos.{range,thread,team}_parallel``
  with ``executionSpace = device``, the kernel-library ops ``kokkos.gemm`` /
  ``kokkos.gemv`` and any pre-lowering ``linalg.*`` / ``sparse.spmv_csr`` /
  ``scf.parallel`` — runs on the B200: the hot nests (CSR SpMV / SpMM, dense
  matmul / matvec / batch matmul, axis reductions) on the hand-written kernels
  of liblapis_b200.so (recognize.py), every other nest as a generated CUDA
  kernel compiled by NVRTC (cudagen.py, csrc/jit.cu);
* dual buffers are real: a pinned host array plus a device allocation with
  the reference's shared modified flags; ``kokkos.sync`` is a real
  cudaMemcpy when the other side is modified and the trace records exactly
  the interpreter's events (H2D / D2H bytes, SyncNoop, StaleAccess;
  interp.py:259-322);
* host-context code (scalar arithmetic, host loops, ``executionSpace = host``
  kernels, host loads / stores) runs on the host, as in the reference.

There is no CPU fallback for device kernels: a nest that neither a
hand-written kernel nor the generator maps raises ``InterpError`` at its op
path.  Generated kernels are bit-identical to the interpreter; hand-written
kernels are bit-identical for integers and within the reference's float
tolerance (``diff_outputs``, interp.py:1050-1071) — pass ``exact=True`` to
route floats through the reference-order variants as well.
"""
from __future__ import annotations

import ctypes as C
import itertools
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi, cudagen

try:  # the reference package is the caller: its IR, config and result types
    from lapis import interp as _li
    from lapis.dialect import (classify_combiner, parallel_hint_operands,
                               parallel_init_operands, scf_parallel_bounds)
    from lapis.ir import DYNAMIC, MemRefType, ScalarType, func_result_types, op_path, walk
    ExecConfig, RunResult, TransferEvent = _li.ExecConfig, _li.RunResult, _li.TransferEvent
    InterpError, StaleAccessError = _li.InterpError, _li.StaleAccessError
except ImportError as _e:  # pragma: no cover - exercised only without the caller package
    raise ImportError("paper_2509_25605_b200.runtime needs the reference's `lapis` package "
                      "(baseline/_ref or /root/reference/pkg/src) on sys.path") from _e

NP_DTYPES = {"f16": np.float16, "f32": np.float32, "f64": np.float64,
             "i1": np.uint8, "i32": np.int32, "i64": np.int64, "index": np.int64}
TORCH_DTYPES = {"f16": torch.float16, "f32": torch.float32, "f64": torch.float64,
                "i1": torch.uint8, "i32": torch.int32, "i64": torch.int64, "index": torch.int64}
ELEM_BYTES = {"f16": 2, "f32": 4, "f64": 8, "i1": 1, "i32": 4, "i64": 8, "index": 8}
FLOATS = ("f16", "f32", "f64")
TRIP_LIMIT = 1 << 31


# ------------------------------------------------------------ scalar semantics
# (interp.py:139-195 restated: ints wrap, floats round to their kind)
def _wrap(v: int, kind: str) -> int:
    if kind == "i1":
        return v & 1
    w = 32 if kind == "i32" else 64
    v &= (1 << w) - 1
    return v - (1 << w) if v >= 1 << (w - 1) else v


def _round(v: float, kind: str) -> float:
    if kind == "f64":
        return float(v)
    if kind == "f32":
        return float(np.float32(v))
    return float(np.float16(v))


def _coerce(v, kind: str):
    return _round(float(v), kind) if kind in FLOATS else _wrap(int(v), kind)


def _unsigned(v: int, kind: str) -> int:
    return v & ((1 << (32 if kind == "i32" else 64)) - 1)


def _combine(acc, x, comb: str, kind: str):
    if comb == "add":
        return _coerce(acc + x, kind)
    if comb == "mul":
        return _coerce(acc * x, kind)
    if comb == "min":
        return acc if acc <= x else x
    return acc if acc >= x else x


# ----------------------------------------------------------------- storage
class Root:
    """One allocation: host storage (numpy over pinned memory), the device
    storage of a separate-memory buffer, and the shared modified flags.

    Buffers the reference keeps in ONE logical storage (host / unassigned
    spaces, or no separate device memory) are executed on the device through
    a mirror of that storage; the mirror's freshness is physical bookkeeping
    and never appears in the trace."""

    __slots__ = ("name", "kind", "extents", "space", "separate", "host", "host_t", "dev",
                 "mirror", "host_fresh", "mirror_fresh", "modified_host", "modified_device",
                 "refcount", "freed", "device_only")

    def __init__(self, name, kind, extents, space, separate, device_only, data=None, device=None):
        self.name, self.kind, self.extents, self.space = name, kind, tuple(extents), space
        self.separate, self.device_only = separate, device_only
        n = int(np.prod(self.extents)) if self.extents else 1
        self.host = self.host_t = None
        if not device_only:
            self.host_t = _pinned_zeros(n, kind) if data is None else data
            self.host = self.host_t.numpy()
        self.dev = torch.zeros(n, dtype=TORCH_DTYPES[kind], device=device) \
            if (separate or device_only) else None
        self.mirror = None
        self.host_fresh, self.mirror_fresh = True, False
        self.modified_host = self.modified_device = False
        self.refcount, self.freed = 1, False

    @property
    def nbytes(self) -> int:
        return (int(np.prod(self.extents)) if self.extents else 1) * ELEM_BYTES[self.kind]

    def strides(self) -> tuple:
        out = [1] * len(self.extents)
        for i in range(len(self.extents) - 2, -1, -1):
            out[i] = out[i + 1] * self.extents[i + 1]
        return tuple(out)


def _pinned_zeros(n: int, kind: str) -> torch.Tensor:
    t = torch.zeros(n, dtype=TORCH_DTYPES[kind])
    if torch.cuda.is_available():
        t = t.pin_memory()
    return t


def _pinned_from(arr: np.ndarray, kind: str) -> torch.Tensor:
    out = _pinned_zeros(arr.size, kind)
    out.numpy()[:] = arr.reshape(-1)
    return out


@dataclass(frozen=True)
class View:
    """A memref value: a window into a root (interp.py:127-136)."""
    root: Root
    offsets: tuple
    shape: tuple

    @staticmethod
    def whole(root: Root) -> "View":
        return View(root, (0,) * len(root.extents), root.extents)

    def flat_offset(self) -> int:
        return sum(o * s for o, s in zip(self.offsets, self.root.strides()))


# ------------------------------------------------------------------ machine
class _Machine:
    def __init__(self, program, config, eager: bool, exact: bool, library: bool, stream):
        self.program, self.config, self.eager = program, config, eager
        self.exact, self.library = exact, library
        self.trace: list = []
        self.counters = {"single": {}, "barrier": {}, "store": {}, "hint": {}}
        self.ctx = "host"
        self._paths: dict = {}
        self._alloc_serial = 0
        self.funcs = {f.attrs["sym_name"]: f for f in program.funcs()}
        if not torch.cuda.is_available():
            raise _capi.BackendError("the B200 executor needs a CUDA device (no CPU fallback)",
                                     _capi.ERR_UNSUPPORTED)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        from .kernels import _device_init
        self._probe = torch.empty(1, device=self.device)
        _device_init(self._probe)
        self.err = torch.zeros(8, dtype=torch.int64, device=self.device)
        self._err_ops: list = []          # kernel error-op tables, indexed by launch
        self._pending_counts: list = []   # (counted list, device tensor)
        self.launches = 0
        self.kernel_log: list = []
        self._versions: dict = {}
        self.csr_checked: dict = {}
        self.csr_plans: dict = {}
        self.globals = {}
        for op in program.ops:
            if op.name == "memref.global":
                t = op.attrs["type"]
                data = np.array([_coerce(v, t.element.kind) for v in op.attrs["value"].elements],
                                dtype=NP_DTYPES[t.element.kind])
                root = self._new_root(f"@{op.attrs['sym_name']}", t.element.kind, t.shape, t.space,
                                      _pinned_from(data, t.element.kind))
                root.modified_host = True
                self.globals[op.attrs["sym_name"]] = root

    # -- plumbing
    def path(self, op) -> str:
        p = self._paths.get(id(op))
        if p is None:
            p = op_path(op, self.program)
            self._paths[id(op)] = p
        return p

    def fail(self, op, message: str):
        raise InterpError(message, self.path(op))

    def _new_root(self, name, kind, extents, space, data=None) -> Root:
        separate_mem = self.config.has_separate_device_memory
        if self.eager:
            separate = separate_mem
            device_only = False
        else:
            separate = separate_mem and space == "dualview"
            device_only = separate_mem and space == "device"
        return Root(name, kind, extents, space, separate, device_only, data, self.device)

    # -- physical coherence of one-storage buffers (never traced)
    def _host_array(self, root: Root) -> np.ndarray:
        if root.host is None:
            raise InterpError(f"host access to device-space buffer {root.name}")
        if not root.host_fresh:
            root.host_t.copy_(root.mirror, non_blocking=False)
            root.host_fresh = True
        return root.host

    def _host_t(self, root: Root) -> torch.Tensor:
        self._host_array(root)
        return root.host_t

    def _mirror(self, root: Root) -> torch.Tensor:
        if root.mirror is None:
            root.mirror = torch.empty(root.host.size, dtype=TORCH_DTYPES[root.kind],
                                      device=self.device)
            root.mirror_fresh = False
        if not root.mirror_fresh:
            root.mirror.copy_(root.host_t, non_blocking=True)
            root.mirror_fresh = True
            self.inflight = True
            self._versions[id(root)] = self._versions.get(id(root), 0) + 1
        return root.mirror

    def _host_written(self, root: Root) -> None:
        root.mirror_fresh = False

    def _sync_stream(self) -> None:
        self.stream.synchronize()
        self.inflight = False

    inflight = False

    # -- storage selection (interp.py:250-275)
    def _uses_device(self, root: Root) -> bool:
        if not self.config.has_separate_device_memory:
            return False
        if self.eager:
            return self.ctx == "device"
        if root.space == "dualview":
            return self.ctx == "device"
        return root.space == "device"

    def device_storage(self, root: Root, op) -> torch.Tensor:
        """The device tensor a kernel in the current context reads/writes."""
        if root.freed or root.refcount < 1:
            self.fail(op, f"access to freed buffer {root.name}")
        if self._uses_device(root):
            return root.dev
        return self._mirror(root)

    def after_device_write(self, root: Root) -> None:
        self._versions[id(root)] = self._versions.get(id(root), 0) + 1
        if not self._uses_device(root):
            root.host_fresh = False

    def version(self, root: Root) -> int:
        """Bumped whenever a kernel or a copy changes the root's device data
        (the key of cached structure checks)."""
        return self._versions.get(id(root), 0)

    def host_storage(self, root: Root, write: bool, op) -> np.ndarray:
        if root.freed or root.refcount < 1:
            self.fail(op, f"access to freed buffer {root.name}")
        if self.config.has_separate_device_memory:
            if self.eager:
                use_device = self.ctx == "device"
            elif root.space == "dualview":
                use_device = self.ctx == "device"
            elif root.space == "device":
                if self.ctx != "device":
                    self.fail(op, f"host access to device-space buffer {root.name}")
                use_device = True
            else:
                use_device = False
            if use_device:
                raise InterpError("device storage accessed from host code", self.path(op))
            if not write and root.modified_device and root.space == "dualview" and not self.eager:
                self._stale(root, "host", op)
        if self.inflight:
            self._sync_stream()   # async copies from / into pinned host memory have landed
        arr = self._host_array(root)
        if write:
            self._host_written(root)
        return arr

    def _stale(self, root: Root, space: str, op) -> None:
        self.trace.append(TransferEvent("StaleAccess", root.name, space=space, path=self.path(op)))
        if self.config.strict_stale_checking:
            raise StaleAccessError(f"stale {space} read of {root.name}", self.path(op))

    def _flat_index(self, view: View, idx, op) -> int:
        for i, (x, extent) in enumerate(zip(idx, view.shape)):
            if not (0 <= x < extent):
                self.fail(op, f"index {x} out of bounds for extent {extent} in dim {i}")
        flat = 0
        for x, off, s in zip(idx, view.offsets, view.root.strides()):
            flat += (off + x) * s
        return flat

    def load_element(self, view: View, idx, op):
        arr = self.host_storage(view.root, False, op)
        v = arr[self._flat_index(view, idx, op)]
        return float(v) if view.root.kind in FLOATS else int(v)

    def store_element(self, view: View, idx, value, op) -> None:
        arr = self.host_storage(view.root, True, op)
        arr[self._flat_index(view, idx, op)] = value
        key = self.path(op)
        self.counters["store"][key] = self.counters["store"].get(key, 0) + 1

    # -- dual-buffer sync (interp.py:294-312), real copies
    def sync(self, root: Root, space: str) -> None:
        if not self.config.has_separate_device_memory:
            self.trace.append(TransferEvent("SyncNoop", root.name, space=space))
            return
        if not root.separate:
            # host/unassigned storage is one logical buffer: flags only
            if space == "device" and root.modified_host:
                root.modified_host = False
                self.trace.append(TransferEvent("H2D", root.name, bytes=root.nbytes))
            elif space == "host" and root.modified_device:
                root.modified_device = False
                self.trace.append(TransferEvent("D2H", root.name, bytes=root.nbytes))
            else:
                self.trace.append(TransferEvent("SyncNoop", root.name, space=space))
            return
        if space == "device":
            if root.modified_host:
                root.dev.copy_(self._host_t(root), non_blocking=True)
                self.inflight = True
                self._versions[id(root)] = self._versions.get(id(root), 0) + 1
                root.modified_host = False
                self.trace.append(TransferEvent("H2D", root.name, bytes=root.nbytes))
            else:
                self.trace.append(TransferEvent("SyncNoop", root.name, space=space))
        else:
            if root.modified_device:
                self._host_t(root).copy_(root.dev, non_blocking=True)
                self.inflight = True
                self._host_written(root)
                root.modified_device = False
                self.trace.append(TransferEvent("D2H", root.name, bytes=root.nbytes))
            else:
                self.trace.append(TransferEvent("SyncNoop", root.name, space=space))

    # -- entry (interp.py:324-370)
    def run_entry(self, entry: str, inputs: list):
        func = self.funcs.get(entry)
        if func is None:
            raise InterpError(f"no function named @{entry}")
        params = func.region(0).args
        if len(inputs) != len(params):
            raise InterpError(f"@{entry} takes {len(params)} arguments, got {len(inputs)}")
        env: dict = {}
        for i, (param, value) in enumerate(zip(params, inputs)):
            t = param.type
            if isinstance(t, MemRefType):
                arr = np.asarray(value)
                if arr.ndim != t.rank:
                    raise InterpError(f"argument {i}: rank {arr.ndim} does not match {t}")
                for d, (have, want) in enumerate(zip(arr.shape, t.shape)):
                    if want != DYNAMIC and have != want:
                        raise InterpError(f"argument {i}: extent {have} in dim {d} does not match {t}")
                kind = t.element.kind
                root = self._new_root(f"arg{i}", kind, tuple(int(d) for d in arr.shape), t.space,
                                      _pinned_from(_coerce_array(arr, kind), kind))
                root.modified_host = True
                env[param] = View.whole(root)
            elif isinstance(t, ScalarType):
                env[param] = _coerce(value, t.kind)
            else:
                raise InterpError(f"argument {i}: unsupported parameter type {t}")
        returned = self.exec_region(func.region(0), env) or []
        outputs = []
        for v, t in zip(returned, func_result_types(func)):
            if isinstance(t, MemRefType):
                view: View = v
                if (self.config.has_separate_device_memory and not self.eager
                        and view.root.space == "dualview" and view.root.modified_device):
                    self.sync(view.root, "host")
                outputs.append(view)
            else:
                outputs.append(v)
        self.finish()
        outputs = [self._materialize(o) if isinstance(o, View) else o for o in outputs]
        result = RunResult(outputs, self.trace, self.counters)
        result.kernels = list(self.kernel_log)   # B200 extra: which path ran each kernel
        return result

    def _materialize(self, view: View) -> np.ndarray:
        dtype = NP_DTYPES[view.root.kind]
        root = view.root
        if root.space == "device" and root.dev is not None:
            data = root.dev.cpu().numpy()
        else:
            data = self._host_array(root)
        if not root.extents:
            return np.asarray(data[0], dtype=dtype).reshape(())
        arr = np.asarray(data, dtype=dtype).reshape(root.extents)
        window = tuple(slice(o, o + s) for o, s in zip(view.offsets, view.shape))
        return arr[window].copy()

    def finish(self) -> None:
        """Wait for the device, surface the first kernel error, merge counters."""
        self._sync_stream()
        for h in self.csr_plans.values():
            _capi.lib().lapis_b200_csr_plan_destroy(h)
        self.csr_plans.clear()
        self.check_errors()
        for counted, dev in self._pending_counts:
            vals = dev.cpu().tolist()
            for (cat, op), n in zip(counted, vals):
                if n and cat != "stale":
                    key = self.path(op)
                    self.counters[cat][key] = self.counters[cat].get(key, 0) + int(n)
        self._pending_counts.clear()

    def check_errors(self) -> None:
        rec = self.err.cpu().tolist()
        if not rec[0]:
            return
        code, opid, a, b, c = rec[0], rec[1], rec[2], rec[3], rec[4]
        launch, local = divmod(opid, 1 << 20)
        op = self._err_ops[launch][local]
        if code == cudagen.ERR_OOB:
            msg = f"index {a} out of bounds for extent {b} in dim {c}"
        elif code in (cudagen.ERR_DIVZERO, cudagen.ERR_FDIVZERO):
            msg = "division by zero"
        elif code == cudagen.ERR_SHIFT:
            msg = "negative shift amount"
        else:
            msg = f"non-positive step {a}"
        self.fail(op, msg)

    # -- region execution (host context)
    def exec_region(self, region, env):
        for op in region.ops:
            if op.name == "func.return":
                return [env[v] for v in op.operands]
            self.exec_op(op, env)
        return None

    def exec_op(self, op, env) -> None:
        h = _HOST.get(op.name)
        if h is None:
            self.fail(op, f"cannot interpret op {op.name}")
        h(self, op, env)

    def _check_trips(self, total: int, op) -> None:
        if total > TRIP_LIMIT:
            self.fail(op, f"trip count {total} exceeds the 2^31 simulation guard")

    # -- host-side loops (executionSpace = host kernels, host loops)
    def host_parallel(self, op, env, ubs, lbs, steps, inits, index_args) -> None:
        ranges, total = [], 1
        for d in range(len(ubs)):
            lo = lbs[d] if lbs else 0
            st = steps[d] if steps else 1
            if st <= 0:
                self.fail(op, f"non-positive step {st}")
            r = range(lo, ubs[d], st)
            ranges.append(r)
            total *= len(r)
        self._check_trips(total, op)
        accs = [env[v] for v in inits]
        body = op.region(0)
        term = body.ops[-1]
        kinds = [classify_combiner(r) for r in term.regions] if term.name == "scf.reduce" else []
        for idx in itertools.product(*ranges):
            for a, v in zip(index_args, idx):
                env[a] = v
            for inner in body.ops[:-1]:
                self.exec_op(inner, env)
            if term.name == "scf.reduce":
                for i, cv in enumerate(term.operands):
                    kind = inits[i].type.kind
                    if kinds[i] is not None:
                        accs[i] = _combine(accs[i], env[cv], kinds[i], kind)
                    else:
                        accs[i] = self._run_combiner(term.regions[i], accs[i], env[cv])
            elif term.name not in ("scf.yield", "kokkos.yield"):
                self.exec_op(term, env)
        for r, acc in zip(op.results, accs):
            env[r] = acc

    def _run_combiner(self, region, acc, contrib):
        env = {region.args[0]: acc, region.args[1]: contrib}
        for inner in region.ops[:-1]:
            self.exec_op(inner, env)
        return env[region.ops[-1].operands[0]]

    # -- device kernels
    def kernel_roots(self, op, env):
        """Roots a device kernel reads / writes, in walk order (interp.py:817-840)."""
        reads: dict = {}
        writes: dict = {}
        first_load: dict = {}

        def note(value, is_write, at):
            v = env.get(value)
            if isinstance(v, View):
                (writes if is_write else reads)[id(v.root)] = v.root
                if not is_write:
                    first_load.setdefault(id(v.root), at)

        for inner in walk(op):
            name = inner.name
            if name == "memref.load":
                note(inner.operands[0], False, inner)
            elif name == "memref.store":
                note(inner.operands[1], True, inner)
            elif name == "memref.copy":
                note(inner.operands[0], False, inner)
                note(inner.operands[1], True, inner)
            elif name in _LIBRARY_OPERANDS:
                rd, wr = _LIBRARY_OPERANDS[name](inner)
                for v in rd:
                    note(v, False, inner)
                for v in wr:
                    note(v, True, inner)
        return list(reads.values()), list(writes.values()), first_load

    def launch(self, op, env, space: str) -> None:
        """Run one device (or host-context, mirrored) kernel on the GPU."""
        prev = self.ctx
        self.ctx = space
        try:
            reads, writes, first_load = self.kernel_roots(op, env)
            eager_copy = self.eager and space == "device" and prev == "host"
            stale = []
            if self.config.has_separate_device_memory and not self.eager:
                for r in reads:
                    if r.space != "dualview":
                        continue
                    if space == "device" and r.modified_host:
                        stale.append((r, "device"))
                    elif space == "host" and r.modified_device:
                        stale.append((r, "host"))
            if stale and self.config.strict_stale_checking:
                r, sp = stale[0]
                self._stale(r, sp, first_load[id(r)])
            if stale:
                # relaxed checking: the kernel reads the stale copy and the
                # trace gets one StaleAccess per executed load of it
                self.generated(op, env, stale_roots=stale)
                self.kernel_log.append((self.path(op), "generated"))
                for w in writes:
                    self.after_device_write(w)
                return
            if eager_copy and self.config.has_separate_device_memory:
                touched = {id(r): r for r in reads}
                for w in writes:
                    touched[id(w)] = w
                for r in touched.values():
                    r.dev.copy_(self._host_t(r), non_blocking=True)
                    self.inflight = True
                    self._versions[id(r)] = self._versions.get(id(r), 0) + 1
                    self.trace.append(TransferEvent("H2D", r.name, bytes=r.nbytes))
            if op.name in cudagen.LIBRARY_OPS:
                _library_checks(self, op, env)
            from . import recognize
            call = recognize.match(self, op, env) if self.library else None
            if call is not None:
                call()
                self.kernel_log.append((self.path(op), "library"))
            else:
                self.generated(op, env)
                self.kernel_log.append((self.path(op), "generated"))
            for w in writes:
                self.after_device_write(w)
            if eager_copy and self.config.has_separate_device_memory:
                for w in writes:
                    self._host_t(w).copy_(w.dev, non_blocking=True)
                    self.inflight = True
                    self._host_written(w)
                    self.trace.append(TransferEvent("D2H", w.name, bytes=w.nbytes))
        finally:
            self.ctx = prev

    # -- generated kernels
    _gen_cache: dict = {}

    def generated(self, op, env, stale_roots=()) -> None:
        vl, ts = 1, None
        if op.name in ("kokkos.team_parallel", "kokkos.thread_parallel"):
            tsv, vlv = parallel_hint_operands(op)
            if vlv is not None:
                vl = int(env[vlv])
            if tsv is not None:
                ts = int(env[tsv])
        stale_ids = {id(r) for r, _ in stale_roots}
        counted = tuple(v for v in _free_memrefs(op)
                        if isinstance(env.get(v), View) and id(env[v].root) in stale_ids)
        key = (id(op), vl, ts, tuple(id(v) for v in counted))
        kern = _Machine._gen_cache.get(key)
        if kern is None or kern[0] is not op:
            try:
                name = f"lapis_gen_{len(_Machine._gen_cache)}"
                if op.name in cudagen.LIBRARY_OPS:
                    if counted:
                        raise cudagen.GenError("relaxed stale reads inside a library op", op)
                    k = cudagen.generate_library(op, name)
                else:
                    k = cudagen.generate(op, name, vl=vl, ts=ts, count_loads=counted)
            except cudagen.GenError as e:
                raise InterpError(f"no B200 kernel for this nest: {e}",
                                  self.path(e.op if e.op is not None else op)) from None
            handle = _jit_compile(k.source, k.name)
            fold = _jit_compile(k.source, k.fold_name) if k.fold_name else None
            kern = (op, k, handle, fold)
            _Machine._gen_cache[key] = kern
        _, k, handle, fold = kern
        counts = self._launch_generated(op, env, k, handle, fold)
        if counted:
            # the events must sit at this point of the trace: read the counts now
            self._sync_stream()
            vals = counts.cpu().tolist()
            space = dict((id(r), sp) for r, sp in stale_roots)
            for (cat, lop), c in zip(k.counted, vals):
                if cat == "stale" and c:
                    root = env[lop.operands[0]].root
                    self.trace.extend([TransferEvent("StaleAccess", root.name, space=space[id(root)],
                                                     path=self.path(lop))] * int(c))

    def _launch_generated(self, op, env, k, handle, fold) -> None:
        launch_id = len(self._err_ops)
        self._err_ops.append(k.error_ops)
        counts = torch.zeros(max(1, len(k.counted)), dtype=torch.int64, device=self.device)
        self._pending_counts.append((k.counted, counts))
        # extent of the launch
        if k.mapping == "team":
            n = int(env[op.operands[0]])
            grid = min(max(n, 1), cudagen.MAX_GRID)
        elif k.mapping == "thread":
            n = int(env[op.operands[0]])
            groups = cudagen.BLOCK // k.vl
            grid = min(max(-(-n // groups), 1), cudagen.MAX_GRID)
        else:
            n = _library_total(op, env) if op.name in cudagen.LIBRARY_OPS \
                else self._range_total(op, env)
            grid = min(max(-(-n // cudagen.BLOCK), 1), cudagen.MAX_GRID)
        contribs, outs = [], []
        for kind, _, _, _ in k.top_reduce:
            contribs.append(torch.empty(max(n, 1), dtype=TORCH_DTYPES[kind], device=self.device))
            outs.append(torch.empty(1, dtype=TORCH_DTYPES[kind], device=self.device))
        slots = []
        for s in k.slots:
            if s.kind == "scalar":
                slots.append(_pack_scalar(env[s.value], s.value.type.kind))
            elif s.kind == "ptr":
                view: View = env[s.value]
                t = self.device_storage(view.root, op)
                slots.append(t.data_ptr() + view.flat_offset() * ELEM_BYTES[view.root.kind])
            elif s.kind == "extent":
                slots.append(env[s.value].shape[s.dim])
            elif s.kind == "stride":
                slots.append(env[s.value].root.strides()[s.dim])
            elif s.aux == "errors":
                slots.append(self.err.data_ptr())
            elif s.aux == "errbase":
                slots.append(launch_id << 20)
            elif s.aux == "counters":
                slots.append(counts.data_ptr())
            elif s.aux.startswith("contrib"):
                slots.append(contribs[int(s.aux[7:])].data_ptr())
            elif s.aux.startswith("out"):
                slots.append(outs[int(s.aux[3:])].data_ptr())
            elif s.aux.startswith("init"):
                r = int(s.aux[4:])
                kind, _, _, init = k.top_reduce[r]
                slots.append(_pack_scalar(env[init], kind))
            elif s.aux == "fold_n":
                slots.append(n)
            else:
                raise AssertionError(s)
        blob = struct.pack(f"<{max(len(slots), 1)}Q", *[(v & (2 ** 64 - 1)) for v in slots] or [0])
        # error op ids carry the launch index in their high bits
        if n > 0:
            _capi.check(_capi.lib().lapis_b200_jit_launch(
                handle, grid, k.block, 0, blob, len(blob), C.c_void_p(self.stream.cuda_stream)),
                "generated kernel")
            self.launches += 1
        if k.top_reduce:
            if n > 0:
                _capi.check(_capi.lib().lapis_b200_jit_launch(
                    fold, 1, 32, 0, blob, len(blob), C.c_void_p(self.stream.cuda_stream)),
                    "generated fold")
                self.launches += 1
                self._sync_stream()
                self.check_errors()
                vals = [o.cpu().item() for o in outs]
            else:
                vals = [env[init] for (_, _, _, init) in k.top_reduce]
            for r, (kind, _, _, _), v in zip(op.results, k.top_reduce, vals):
                env[r] = _coerce(v, kind)
        return counts

    def _range_total(self, op, env) -> int:
        if op.name == "scf.parallel":
            lows, ups, steps, _ = scf_parallel_bounds(op)
            total = 1
            for lo, hi, st in zip(lows, ups, steps):
                lo, hi, st = env[lo], env[hi], env[st]
                if st <= 0:
                    self.fail(op, f"non-positive step {st}")
                total *= len(range(lo, hi, st))
            return total
        dims = op.attrs.get("dims", 1)
        total = 1
        for v in op.operands[:dims]:
            total *= max(int(env[v]), 0)
        return total


def _free_memrefs(op) -> list:
    """Memref values a nest reads that are defined outside it."""
    inside = set()
    for o in walk(op):
        inside.update(id(r) for r in o.results)
        for reg in o.regions:
            inside.update(id(a) for a in reg.args)
    out, seen = [], set()
    for o in walk(op):
        if o.name == "memref.load":
            v = o.operands[0]
            if id(v) not in inside and id(v) not in seen:
                seen.add(id(v))
                out.append(v)
    return out


def _library_checks(m: _Machine, op, env) -> None:
    """The interpreter's shape errors for library ops (interp.py:711-812, 949-976)."""
    name = op.name
    if name in ("linalg.matmul", "kokkos.gemm"):
        a, b, c = (env[v] for v in op.operands[:3])
        (mm, kk), (kk2, nn) = a.shape, b.shape
        if kk != kk2 or c.shape != (mm, nn):
            m.fail(op, f"matmul shape mismatch {a.shape} x {b.shape} -> {c.shape}")
    elif name in ("linalg.matvec", "kokkos.gemv"):
        a, x, y = (env[v] for v in op.operands[:3])
        mm, nn = a.shape
        if x.shape != (nn,) or y.shape != (mm,):
            m.fail(op, f"matvec shape mismatch {a.shape} x {x.shape} -> {y.shape}")
    elif name == "linalg.batch_matmul":
        a, b, c = (env[v] for v in op.operands[:3])
        if not (a.shape[0] == b.shape[0] == c.shape[0]):
            m.fail(op, "batch extents must match")
        nb, mm, kk = a.shape
        if b.shape[1] != kk or c.shape[1:] != (mm, b.shape[2]):
            m.fail(op, f"batch_matmul shape mismatch {a.shape} x {b.shape} -> {c.shape}")
    elif name in ("sparse.spmv_csr", "kokkos.spmv_csr"):
        rowptr, y = env[op.operands[0]], env[op.operands[4]]
        nrows = rowptr.shape[0] - 1
        if y.shape[0] != nrows:
            m.fail(op, f"y has extent {y.shape[0]}, rowptr implies {nrows} rows")


def _library_total(op, env) -> int:
    """Output elements of a library op's generated kernel (one thread each)."""
    name = op.name
    if name == "linalg.reduce":
        src = env[op.operands[0]]
        axes = list(op.attrs["axes"])
        return int(np.prod([e for d, e in enumerate(src.shape) if d not in axes], dtype=np.int64))
    if name in ("linalg.matvec", "kokkos.gemv"):
        return env[op.operands[2]].shape[0]
    if name in ("sparse.spmv_csr", "kokkos.spmv_csr"):
        return max(env[op.operands[0]].shape[0] - 1, 0)
    out = env[op.operands[1] if name == "linalg.fill" else
              op.operands[-1] if name == "linalg.elementwise" else op.operands[2]]
    return int(np.prod(out.shape, dtype=np.int64))


def _coerce_array(arr: np.ndarray, kind: str) -> np.ndarray:
    if kind == "i1":
        return (arr.astype(np.int64) & 1).astype(np.uint8)
    if kind in FLOATS:
        return arr.astype(NP_DTYPES[kind])
    if arr.dtype.kind == "f":
        return np.trunc(arr).astype(np.int64).astype(NP_DTYPES[kind])
    return arr.astype(np.int64).astype(NP_DTYPES[kind])


def _pack_scalar(v, kind: str) -> int:
    if kind == "f64":
        return struct.unpack("<Q", struct.pack("<d", float(v)))[0]
    if kind == "f32":
        return struct.unpack("<I", struct.pack("<f", float(v)))[0]
    return int(v) & (2 ** 64 - 1)


_JIT: dict = {}


def _jit_compile(source: str, name: str):
    key = (torch.cuda.current_device(), name, source)
    h = _JIT.get(key)
    if h is None:
        out = C.c_void_p()
        _capi.check(_capi.lib().lapis_b200_jit_compile(source.encode(), name.encode(), C.byref(out)),
                    "jit_compile")
        h = out
        _JIT[key] = h
    return h


# operands read / written by library ops (interp.py:832-838, plus the rest)
_LIBRARY_OPERANDS = {
    "kokkos.gemm": lambda op: (op.operands[:2], op.operands[2:3]),
    "kokkos.gemv": lambda op: (op.operands[:2], op.operands[2:3]),
    "linalg.matmul": lambda op: (op.operands[:2], op.operands[2:3]),
    "linalg.matvec": lambda op: (op.operands[:2], op.operands[2:3]),
    "linalg.batch_matmul": lambda op: (op.operands[:2], op.operands[2:3]),
    "linalg.fill": lambda op: ([], op.operands[1:2]),
    "linalg.elementwise": lambda op: (op.operands[:-1], op.operands[-1:]),
    "linalg.reduce": lambda op: (op.operands[:1], op.operands[1:2]),
    "sparse.spmv_csr": lambda op: (op.operands[:4], op.operands[4:5]),
    "kokkos.spmv_csr": lambda op: (op.operands[:4], op.operands[4:5]),
}


# ----------------------------------------------------------- host handlers
def _int_binop(fn):
    def h(m, op, env):
        a, b = env[op.operands[0]], env[op.operands[1]]
        env[op.results[0]] = _wrap(fn(m, op, a, b), op.results[0].type.kind)
    return h


def _float_binop(fn):
    def h(m, op, env):
        a, b = env[op.operands[0]], env[op.operands[1]]
        env[op.results[0]] = _round(fn(m, op, a, b), op.results[0].type.kind)
    return h


def _divi(m, op, a, b):
    if b == 0:
        m.fail(op, "division by zero")
    q = abs(a) // abs(b)
    return q if (a >= 0) == (b >= 0) else -q


def _ceildivsi(m, op, a, b):
    if b == 0:
        m.fail(op, "division by zero")
    return -((-a) // b)


def _shli(m, op, a, b):
    if b < 0:
        m.fail(op, "negative shift amount")
    return 0 if b >= 64 else a << b


def _divf(m, op, a, b):
    if b == 0.0:
        m.fail(op, "division by zero")
    return a / b


_CMPI = {
    "eq": lambda a, b, k: a == b, "ne": lambda a, b, k: a != b,
    "slt": lambda a, b, k: a < b, "sle": lambda a, b, k: a <= b,
    "sgt": lambda a, b, k: a > b, "sge": lambda a, b, k: a >= b,
    "ult": lambda a, b, k: _unsigned(a, k) < _unsigned(b, k),
    "ule": lambda a, b, k: _unsigned(a, k) <= _unsigned(b, k),
    "ugt": lambda a, b, k: _unsigned(a, k) > _unsigned(b, k),
    "uge": lambda a, b, k: _unsigned(a, k) >= _unsigned(b, k),
}
_CMPF = {"oeq": lambda a, b: a == b, "one": lambda a, b: a != b, "olt": lambda a, b: a < b,
         "ole": lambda a, b: a <= b, "ogt": lambda a, b: a > b, "oge": lambda a, b: a >= b}


def _h_constant(m, op, env):
    env[op.results[0]] = _coerce(op.attrs["value"], op.results[0].type.kind)


def _h_cmpi(m, op, env):
    a, b = env[op.operands[0]], env[op.operands[1]]
    env[op.results[0]] = 1 if _CMPI[op.attrs["predicate"]](a, b, op.operands[0].type.kind) else 0


def _h_cmpf(m, op, env):
    a, b = env[op.operands[0]], env[op.operands[1]]
    env[op.results[0]] = 1 if _CMPF[op.attrs["predicate"]](a, b) else 0


def _h_select(m, op, env):
    env[op.results[0]] = env[op.operands[1]] if env[op.operands[0]] else env[op.operands[2]]


def _h_index_cast(m, op, env):
    env[op.results[0]] = _wrap(env[op.operands[0]], op.results[0].type.kind)


def _h_minui(m, op, env):
    a, b = env[op.operands[0]], env[op.operands[1]]
    k = op.results[0].type.kind
    env[op.results[0]] = a if _unsigned(a, k) <= _unsigned(b, k) else b


def _h_maxsi(m, op, env):
    a, b = env[op.operands[0]], env[op.operands[1]]
    env[op.results[0]] = a if a >= b else b


def _h_alloc(m: _Machine, op, env):
    t = op.results[0].type
    extents = []
    dyn = iter(op.operands)
    for d in t.shape:
        if d == DYNAMIC:
            e = int(env[next(dyn)])
            if e < 0:
                m.fail(op, f"negative allocation extent {e}")
            extents.append(e)
        else:
            extents.append(d)
    m._alloc_serial += 1
    root = m._new_root(f"alloc{m._alloc_serial}({m.path(op)})", t.element.kind, tuple(extents),
                       t.space)
    env[op.results[0]] = View.whole(root)


def _h_dealloc(m, op, env):
    view: View = env[op.operands[0]]
    view.root.refcount -= 1
    if view.root.refcount <= 0:
        view.root.freed = True


def _h_load(m, op, env):
    view = env[op.operands[0]]
    env[op.results[0]] = m.load_element(view, tuple(env[v] for v in op.operands[1:]), op)


def _h_store(m, op, env):
    m.store_element(env[op.operands[1]], tuple(env[v] for v in op.operands[2:]),
                    env[op.operands[0]], op)


def _h_dim(m, op, env):
    env[op.results[0]] = env[op.operands[0]].shape[op.attrs["index"]]


def _h_subview(m, op, env):
    base: View = env[op.operands[0]]
    rank = len(base.shape)
    offs = tuple(env[v] for v in op.operands[1:1 + rank])
    sizes = tuple(env[v] for v in op.operands[1 + rank:])
    for d, (o, s) in enumerate(zip(offs, sizes)):
        if o < 0 or s < 0 or o + s > base.shape[d]:
            m.fail(op, f"subview [{o}, {o + s}) out of bounds for extent {base.shape[d]} in dim {d}")
    base.root.refcount += 1
    env[op.results[0]] = View(base.root, tuple(a + b for a, b in zip(base.offsets, offs)), sizes)


def _h_cast(m, op, env):
    base: View = env[op.operands[0]]
    base.root.refcount += 1
    for have, want in zip(base.shape, op.results[0].type.shape):
        if want != DYNAMIC and have != want:
            m.fail(op, f"cast extent mismatch: runtime {have} vs static {want}")
    env[op.results[0]] = base


def _h_copy(m, op, env):
    src: View = env[op.operands[0]]
    dst: View = env[op.operands[1]]
    if src.shape != dst.shape:
        m.fail(op, f"copy shape mismatch {src.shape} vs {dst.shape}")
    for idx in itertools.product(*(range(e) for e in src.shape)) if src.shape else [()]:
        m.store_element(dst, idx, m.load_element(src, idx, op), op)


def _h_get_global(m, op, env):
    root = m.globals[op.attrs["symbol"]]
    root.refcount += 1
    env[op.results[0]] = View.whole(root)


def _h_scf_parallel(m: _Machine, op, env):
    # a pre-lowering parallel loop in host context: run it on the device over
    # the host storage (interp.py:650-659 semantics) when it maps to a kernel;
    # loops that allocate per iteration stay host code
    if _device_mappable(op):
        m.launch(op, env, m.ctx)
        return
    lows, ups, steps, inits = scf_parallel_bounds(op)
    m.host_parallel(op, env, [env[v] for v in ups], [env[v] for v in lows],
                    [env[v] for v in steps], list(inits), op.region(0).args)


def _device_mappable(op) -> bool:
    return not any(o.name in ("memref.alloc", "memref.dealloc", "func.call", "memref.copy",
                              "memref.subview", "memref.cast", "memref.get_global",
                              "linalg.matmul", "linalg.matvec", "sparse.spmv_csr",
                              "kokkos.spmv_csr")
                   for o in walk(op)) and all(
        getattr(v.type, "kind", "f64") != "f16" for o in walk(op) for v in o.results)


def _h_scf_for(m, op, env):
    lo, hi, step = (env[v] for v in op.operands)
    if step <= 0:
        m.fail(op, f"non-positive step {step}")
    r = range(lo, hi, step)
    m._check_trips(len(r), op)
    body = op.region(0)
    iv = body.args[0]
    for i in r:
        env[iv] = i
        for inner in body.ops[:-1]:
            m.exec_op(inner, env)


def _h_scf_if(m, op, env):
    if env[op.operands[0]]:
        region = op.region(0)
    elif len(op.regions) > 1:
        region = op.region(1)
    else:
        return
    for inner in region.ops[:-1]:
        m.exec_op(inner, env)


def _h_call(m, op, env):
    callee = m.funcs.get(op.attrs["callee"])
    if callee is None:
        m.fail(op, f"unknown function @{op.attrs['callee']}")
    inner = {p: env[a] for p, a in zip(callee.region(0).args, op.operands)}
    returned = m.exec_region(callee.region(0), inner)
    for r, v in zip(op.results, returned or []):
        env[r] = v


def _h_library(m: _Machine, op, env):
    # linalg.* / sparse.spmv_csr run in the current context (interp.py:704-812);
    # kokkos.gemm / gemv / spmv_csr always on the device (interp.py:949-976)
    space = "device" if op.name.startswith("kokkos.") else m.ctx
    m.launch(op, env, space)


def _h_kernel(m: _Machine, op, env):
    space = op.attrs.get("executionSpace")
    if op.name in ("kokkos.team_parallel", "kokkos.thread_parallel"):
        _, vl = parallel_hint_operands(op)
        if vl is not None:
            m.counters["hint"][m.path(op)] = env[vl]
    if space == "device":
        m.launch(op, env, "device")
        return
    # host execution space (or a nested op reached from host code)
    prev = m.ctx
    if space is not None:
        m.ctx = space
    try:
        _host_kokkos(m, op, env)
    finally:
        m.ctx = prev


def _host_kokkos(m: _Machine, op, env):
    inits = parallel_init_operands(op)
    if op.name == "kokkos.range_parallel":
        dims = op.attrs.get("dims", 1)
        m.host_parallel(op, env, [env[v] for v in op.operands[:dims]], None, None, inits,
                        op.region(0).args)
    elif op.name == "kokkos.thread_parallel":
        m.host_parallel(op, env, [env[op.operands[0]]], None, None, inits, op.region(0).args)
    else:
        args = op.region(0).args
        env[args[1]] = ("team", m.path(op))
        m.host_parallel(op, env, [env[op.operands[0]]], None, None, inits, [args[0]])


def _h_single(m, op, env):
    key = m.path(op)
    m.counters["single"][key] = m.counters["single"].get(key, 0) + 1
    for inner in op.region(0).ops[:-1]:
        m.exec_op(inner, env)


def _h_team_barrier(m, op, env):
    key = m.path(op)
    m.counters["barrier"][key] = m.counters["barrier"].get(key, 0) + 1


def _h_sync(m: _Machine, op, env):
    if m.eager:
        return
    m.sync(env[op.operands[0]].root, op.attrs["space"])


def _h_modify(m: _Machine, op, env):
    if m.eager or not m.config.has_separate_device_memory:
        return
    root = env[op.operands[0]].root
    if op.attrs["space"] == "device":
        root.modified_device = True
    else:
        root.modified_host = True


def _h_noop(m, op, env):
    pass


_HOST = {
    "arith.constant": _h_constant,
    "arith.addi": _int_binop(lambda m, op, a, b: a + b),
    "arith.subi": _int_binop(lambda m, op, a, b: a - b),
    "arith.muli": _int_binop(lambda m, op, a, b: a * b),
    "arith.divi": _int_binop(_divi),
    "arith.ceildivsi": _int_binop(_ceildivsi),
    "arith.shli": _int_binop(_shli),
    "arith.addf": _float_binop(lambda m, op, a, b: a + b),
    "arith.subf": _float_binop(lambda m, op, a, b: a - b),
    "arith.mulf": _float_binop(lambda m, op, a, b: a * b),
    "arith.divf": _float_binop(_divf),
    "arith.cmpi": _h_cmpi,
    "arith.cmpf": _h_cmpf,
    "arith.select": _h_select,
    "arith.index_cast": _h_index_cast,
    "arith.minui": _h_minui,
    "arith.maxsi": _h_maxsi,
    "memref.alloc": _h_alloc,
    "memref.dealloc": _h_dealloc,
    "memref.load": _h_load,
    "memref.store": _h_store,
    "memref.dim": _h_dim,
    "memref.subview": _h_subview,
    "memref.cast": _h_cast,
    "memref.copy": _h_copy,
    "memref.get_global": _h_get_global,
    "scf.parallel": _h_scf_parallel,
    "scf.for": _h_scf_for,
    "scf.if": _h_scf_if,
    "scf.yield": _h_noop,
    "func.call": _h_call,
    "linalg.matmul": _h_library,
    "linalg.matvec": _h_library,
    "linalg.batch_matmul": _h_library,
    "linalg.fill": _h_library,
    "linalg.elementwise": _h_library,
    "linalg.reduce": _h_library,
    "sparse.spmv_csr": _h_library,
    "kokkos.spmv_csr": _h_library,   # sparse_route.py: the kernel-library route
    "kokkos.range_parallel": _h_kernel,
    "kokkos.team_parallel": _h_kernel,
    "kokkos.thread_parallel": _h_kernel,
    "kokkos.single": _h_single,
    "kokkos.team_barrier": _h_team_barrier,
    "kokkos.sync": _h_sync,
    "kokkos.modify": _h_modify,
    "kokkos.gemm": _h_library,
    "kokkos.gemv": _h_library,
    "kokkos.yield": _h_noop,
}


# ------------------------------------------------------------------ public API
def run(program, entry: str, inputs: list, config=None, *, exact: bool = False,
        library: bool = True, stream=None):
    """Execute ``entry`` on the B200 with the lazy dual-buffer policy — the
    drop-in for ``lapis.interp.run`` (interp.py:1037-1039).

    ``exact=True`` routes floating-point hot kernels through their
    reference-order variants (bit-identical to the interpreter);
    ``library=False`` disables the hand-written kernels so that every nest
    runs as a generated kernel (used by the parity tests)."""
    return _Machine(program, config or ExecConfig(), False, exact, library, stream).run_entry(
        entry, inputs)


def run_eager_baseline(program, entry: str, inputs: list, config=None, *, exact: bool = False,
                       library: bool = True, stream=None):
    """The eager policy (interp.py:1042-1047): every kernel-touched buffer is
    copied to the device before each device kernel and every written buffer
    back afterwards."""
    return _Machine(program, config or ExecConfig(), True, exact, library, stream).run_entry(
        entry, inputs)
