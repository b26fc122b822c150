"""Kokkos loop nest -> CUDA C++ for sm_100a (the generated-kernel path).

The reference emits every top-level kokkos.{range,thread,team}_parallel nest
as a Kokkos lambda (emitter.py:596-780) and runs it on a serial stub
(lapis_serial_stub.hpp:313-419).  Nests that have no hand-written kernel
(paper_2509_25605_b200/recognize.py) are emitted here as one CUDA kernel each,
compiled by NVRTC inside liblapis_b200.so (csrc/jit.cu) and launched by the
executor (runtime.py).  The mapping is the Kokkos-on-CUDA one:

    team_parallel(league, VL)   -> one CTA per league index (grid-stride),
                                   TS = 256 / VL "threads" of VL lanes each
    thread_parallel(n, VL)      -> one group of VL lanes per index (grid-stride)
    range_parallel toprange/md  -> one thread per (flattened) index
    teamthread range            -> the CTA's groups stride over the range
    threadvector range          -> the group's lanes stride over the range
    single perTeam / perThread  -> group 0 lane 0 / lane 0 of the group
    team_barrier                -> __syncthreads()

Semantics follow the reference interpreter exactly, so generated kernels are
bit-identical to it (interp.py):
  * every arithmetic op is rounded to its type (NVRTC --fmad=false, no
    contraction), ints wrap in two's complement (interp.py:145-171, 469-562);
  * reductions fold in ascending index order (interp.py:407-431): a vector
    reduce folds the VL lane contributions of each step in lane order through
    shuffles, a teamthread reduce folds the CTA's contributions of each chunk
    in order through shared memory — no padding terms, so no -0.0 drift;
  * loads/stores are bounds-checked; division by zero, negative shifts and
    non-positive steps are reported through an error record that the
    executor turns into the interpreter's InterpError (interp.py:269-276,
    485-507, 650-670);
  * "single", "barrier" and "store" executions are counted per op path, on
    the one lane that the serial reference would have run
    (interp.py:597-602, 918-928).
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field

CTYPE = {"f64": "double", "f32": "float", "i64": "long long", "index": "long long",
         "i32": "int", "i1": "int"}
STORE_CTYPE = dict(CTYPE, i1="unsigned char")
UTYPE = {"i64": "unsigned long long", "index": "unsigned long long", "i32": "unsigned int",
         "i1": "unsigned int"}
FLOAT_KINDS = ("f32", "f64")
INT_KINDS = ("i1", "i32", "i64", "index")
WIDTH = {"i1": 1, "i32": 32, "i64": 64, "index": 64}

BLOCK = 256               # threads per CTA of thread/range kernels
MAX_GRID = 148 * 16       # grid-stride cap: 16 CTAs per SM on the 148 SMs

# error codes written into the record (runtime.py formats the messages)
ERR_OOB, ERR_DIVZERO, ERR_SHIFT, ERR_STEP, ERR_FDIVZERO = 1, 2, 3, 4, 5


class GenError(Exception):
    """The nest uses a construct the generator does not map (reported by the
    executor as an InterpError at the op's path; there is no CPU fallback)."""

    def __init__(self, message: str, op=None):
        super().__init__(message)
        self.op = op


@dataclass
class Slot:
    """One 8-byte parameter slot: a free scalar, or part of a free memref."""
    kind: str            # "scalar" | "ptr" | "extent" | "stride" | "aux"
    value: object = None  # the IR Value (scalar / memref)
    dim: int = 0
    aux: str = ""


@dataclass
class Kernel:
    name: str
    source: str = ""
    slots: list = field(default_factory=list)
    mapping: str = ""            # "range" | "thread" | "team"
    vl: int = 1
    ts: int = 1
    block: int = BLOCK
    counted: list = field(default_factory=list)   # [(category, op)] in counter-slot order
    error_ops: list = field(default_factory=list)  # op per error id
    top_reduce: list = field(default_factory=list)  # [(kind, combiner, init Value)] host results
    fold_name: str = ""


def _hex_double(v: float) -> str:
    bits = struct.unpack("<q", struct.pack("<d", float(v)))[0]
    return f"__longlong_as_double({bits}LL)"


def _hex_float(v: float) -> str:
    bits = struct.unpack("<i", struct.pack("<f", float(v)))[0]
    return f"__int_as_float({bits})"


def _int_lit(v: int, kind: str) -> str:
    if kind in ("i64", "index"):
        if v == -(1 << 63):
            return "(-9223372036854775807LL - 1LL)"
        return f"{v}LL"
    if kind == "i32":
        if v == -(1 << 31):
            return "(-2147483647 - 1)"
        return f"{v}"
    return f"{v & 1}"


def literal(v, kind: str) -> str:
    if kind == "f64":
        return _hex_double(v)
    if kind == "f32":
        return _hex_float(v)
    return _int_lit(int(v), kind)


def _kind(value) -> str:
    t = value.type
    k = getattr(t, "kind", None)
    if k is None:
        raise GenError(f"value of type {t} is not a scalar")
    if k == "f16":
        raise GenError("f16 arithmetic has no generated-kernel mapping")
    return k


_PRELUDE = r"""
struct LbParams { unsigned long long s[%(nslots)d]; };
static __device__ __forceinline__ void lb_err(unsigned long long* E, int code, long long op,
                                              long long a, long long b, long long c) {
  if (atomicCAS(E, 0ull, (unsigned long long)code) == 0ull) {
    E[1] = (unsigned long long)op; E[2] = (unsigned long long)a;
    E[3] = (unsigned long long)b; E[4] = (unsigned long long)c;
  }
}
static __device__ __forceinline__ long long lb_divi64(long long a, long long b) {
  return (b == -1LL) ? (long long)(0ull - (unsigned long long)a) : a / b;
}
static __device__ __forceinline__ int lb_divi32(int a, int b) {
  return (b == -1) ? (int)(0u - (unsigned)a) : a / b;
}
static __device__ __forceinline__ long long lb_ceildiv64(long long a, long long b) {
  if (b == -1LL) return (long long)(0ull - (unsigned long long)a);
  long long q = a / b, r = a %% b;
  return (r != 0 && ((r > 0) == (b > 0))) ? q + 1 : q;
}
static __device__ __forceinline__ int lb_ceildiv32(int a, int b) {
  if (b == -1) return (int)(0u - (unsigned)a);
  int q = a / b, r = a %% b;
  return (r != 0 && ((r > 0) == (b > 0))) ? q + 1 : q;
}
"""


class _Ctx:
    """Where the code being emitted runs: the replication level decides which
    lane stands for the serial reference (counting, side effects)."""

    def __init__(self, level: str, canon: str):
        self.level = level      # "range" | "team" | "thread" | "vector"
        self.canon = canon      # C expression: this lane is the serial one


class NestGen:
    """Generates one kernel (plus an ordered-fold kernel for host results)."""

    def __init__(self, top, name: str, vl: int = 1, ts: int | None = None, path_of=None,
                 count_loads=()):
        self.top = top
        self.count_loads = set(count_loads)
        self.k = Kernel(name=name)
        self.vl = max(1, min(32, 1 << int(math.log2(max(1, vl)))))
        self.path_of = path_of or (lambda op: op.name)
        self.names: dict = {}
        self.lines: list[str] = []
        self.ind = 1
        self.tmp = 0
        self.defined: set = set()
        self.slot_of: dict = {}           # (Value, kind, dim) -> slot index
        self.counter_of: dict = {}        # (category, op) -> counter index
        self.max_team_acc = 0
        self.ts_hint = ts

    # ------------------------------------------------------------- utilities
    def emit(self, s: str) -> None:
        self.lines.append("  " * self.ind + s)

    def fresh(self, base: str = "t") -> str:
        self.tmp += 1
        return f"{base}{self.tmp}_"

    def name(self, v) -> str:
        n = self.names.get(v)
        if n is None:
            n = f"v{len(self.names)}"
            self.names[v] = n
        return n

    def slot(self, kind: str, value=None, dim: int = 0, aux: str = "") -> int:
        key = (id(value), kind, dim, aux)
        idx = self.slot_of.get(key)
        if idx is None:
            idx = len(self.k.slots)
            self.k.slots.append(Slot(kind, value, dim, aux))
            self.slot_of[key] = idx
        return idx

    def counter(self, category: str, op) -> str:
        key = (category, id(op))
        idx = self.counter_of.get(key)
        if idx is None:
            idx = len(self.k.counted)
            self.k.counted.append((category, op))
            self.counter_of[key] = idx
        return f"lb_cnt{idx}"

    def error_id(self, op) -> int:
        for i, o in enumerate(self.k.error_ops):
            if o is op:
                return i
        self.k.error_ops.append(op)
        return len(self.k.error_ops) - 1

    # ------------------------------------------------------------ free values
    def scalar(self, v) -> str:
        """C expression of a scalar value (free values become parameter slots)."""
        if v in self.defined:
            return self.name(v)
        kind = _kind(v)
        idx = self.slot("scalar", v)
        n = self.name(v)
        if n not in self._unpacked:
            self._unpacked.add(n)
            if kind == "f64":
                self._head.append(f"const double {n} = __longlong_as_double((long long)P.s[{idx}]);")
            elif kind == "f32":
                self._head.append(f"const float {n} = __int_as_float((int)(unsigned)P.s[{idx}]);")
            else:
                self._head.append(f"const {CTYPE[kind]} {n} = ({CTYPE[kind]})(long long)P.s[{idx}];")
        return n

    def memref(self, v):
        """(pointer name, [extent exprs], [stride exprs]) of a free memref."""
        t = v.type
        if not hasattr(t, "shape"):
            raise GenError(f"{v} is not a memref")
        if v in self.defined:
            raise GenError("memrefs created inside a device kernel are not supported")
        kind = t.element.kind
        if kind == "f16":
            raise GenError("f16 buffers have no generated-kernel mapping")
        base = self.name(v)
        if base not in self._unpacked:
            self._unpacked.add(base)
            p = self.slot("ptr", v)
            self._head.append(f"{STORE_CTYPE[kind]}* const {base} = ({STORE_CTYPE[kind]}*)P.s[{p}];")
            for d in range(t.rank):
                e = self.slot("extent", v, d)
                s = self.slot("stride", v, d)
                self._head.append(f"const long long {base}_e{d} = (long long)P.s[{e}];")
                self._head.append(f"const long long {base}_s{d} = (long long)P.s[{s}];")
        return base, [f"{base}_e{d}" for d in range(t.rank)], [f"{base}_s{d}" for d in range(t.rank)]

    def define(self, v, ctype: str, expr: str) -> str:
        n = self.name(v)
        self.defined.add(v)
        self.emit(f"const {ctype} {n} = {expr};")
        return n

    # ----------------------------------------------------------- arithmetic
    def wrap(self, kind: str, expr_unsigned: str) -> str:
        if kind == "i1":
            return f"((int)(({expr_unsigned}) & 1u))"
        return f"(({CTYPE[kind]})({expr_unsigned}))"

    def emit_arith(self, op) -> bool:
        name = op.name
        if name == "arith.constant":
            r = op.results[0]
            kind = _kind(r)
            self.define(r, CTYPE[kind], literal(op.attrs["value"], kind))
            return True
        if name in ("arith.addi", "arith.subi", "arith.muli"):
            r = op.results[0]
            kind = _kind(r)
            a, b = (self.scalar(v) for v in op.operands)
            sym = {"arith.addi": "+", "arith.subi": "-", "arith.muli": "*"}[name]
            u = UTYPE[kind]
            self.define(r, CTYPE[kind], self.wrap(kind, f"({u}){a} {sym} ({u}){b}"))
            return True
        if name in ("arith.divi", "arith.ceildivsi"):
            r = op.results[0]
            kind = _kind(r)
            a, b = (self.scalar(v) for v in op.operands)
            eid = self.error_id(op)
            n = self.name(r)
            self.defined.add(r)
            ct = CTYPE[kind]
            self.emit(f"{ct} {n} = 0;")
            self.emit(f"if ({b} == 0) lb_err(lb_E, {ERR_DIVZERO}, lb_eb + {eid}, 0, 0, 0); else {{")
            if kind == "i1":
                self.emit(f"  {n} = {a};")  # b is 1
            elif kind == "i32":
                fn = "lb_divi32" if name == "arith.divi" else "lb_ceildiv32"
                self.emit(f"  {n} = {fn}({a}, {b});")
            else:
                fn = "lb_divi64" if name == "arith.divi" else "lb_ceildiv64"
                self.emit(f"  {n} = {fn}({a}, {b});")
            self.emit("}")
            return True
        if name == "arith.shli":
            r = op.results[0]
            kind = _kind(r)
            a, b = (self.scalar(v) for v in op.operands)
            eid = self.error_id(op)
            n = self.name(r)
            self.defined.add(r)
            u = UTYPE[kind]
            w = WIDTH[kind]
            self.emit(f"{CTYPE[kind]} {n} = 0;")
            self.emit(f"if ({b} < 0) lb_err(lb_E, {ERR_SHIFT}, lb_eb + {eid}, (long long){b}, 0, 0);")
            self.emit(f"else if ((long long){b} < {w}) {n} = {self.wrap(kind, f'({u}){a} << (unsigned)({b})')};")
            return True
        if name in ("arith.addf", "arith.subf", "arith.mulf"):
            r = op.results[0]
            kind = _kind(r)
            a, b = (self.scalar(v) for v in op.operands)
            sym = {"arith.addf": "+", "arith.subf": "-", "arith.mulf": "*"}[name]
            self.define(r, CTYPE[kind], f"{a} {sym} {b}")
            return True
        if name == "arith.divf":
            r = op.results[0]
            kind = _kind(r)
            a, b = (self.scalar(v) for v in op.operands)
            eid = self.error_id(op)
            n = self.name(r)
            self.defined.add(r)
            self.emit(f"{CTYPE[kind]} {n} = 0;")
            self.emit(f"if ({b} == 0) lb_err(lb_E, {ERR_FDIVZERO}, lb_eb + {eid}, 0, 0, 0); else {n} = {a} / {b};")
            return True
        if name == "arith.cmpi":
            r = op.results[0]
            kind = _kind(op.operands[0])
            a, b = (self.scalar(v) for v in op.operands)
            pred = op.attrs["predicate"]
            signed = {"eq": "==", "ne": "!=", "slt": "<", "sle": "<=", "sgt": ">", "sge": ">="}
            if pred in signed:
                expr = f"({a} {signed[pred]} {b})"
            else:
                u = UTYPE[kind] if kind != "i1" else "unsigned int"
                sym = {"ult": "<", "ule": "<=", "ugt": ">", "uge": ">="}[pred]
                if kind == "i1":
                    expr = f"(((unsigned)({a}) & 1u) {sym} ((unsigned)({b}) & 1u))"
                else:
                    expr = f"(({u}){a} {sym} ({u}){b})"
            self.define(r, "int", f"{expr} ? 1 : 0")
            return True
        if name == "arith.cmpf":
            r = op.results[0]
            a, b = (self.scalar(v) for v in op.operands)
            sym = {"oeq": "==", "one": "!=", "olt": "<", "ole": "<=", "ogt": ">",
                   "oge": ">="}[op.attrs["predicate"]]
            self.define(r, "int", f"({a} {sym} {b}) ? 1 : 0")
            return True
        if name == "arith.select":
            r = op.results[0]
            kind = _kind(r)
            c, a, b = (self.scalar(v) for v in op.operands)
            self.define(r, CTYPE[kind], f"{c} ? {a} : {b}")
            return True
        if name == "arith.index_cast":
            r = op.results[0]
            kind = _kind(r)
            a = self.scalar(op.operands[0])
            if kind == "i1":
                expr = f"((int)((long long)({a}) & 1LL))"
            elif kind == "i32":
                expr = f"((int)(unsigned int)(unsigned long long)(long long)({a}))"
            else:
                expr = f"((long long)({a}))"
            self.define(r, CTYPE[kind], expr)
            return True
        if name == "arith.minui":
            r = op.results[0]
            kind = _kind(r)
            a, b = (self.scalar(v) for v in op.operands)
            u = UTYPE[kind]
            self.define(r, CTYPE[kind], f"(({u}){a} <= ({u}){b}) ? {a} : {b}")
            return True
        if name == "arith.maxsi":
            r = op.results[0]
            kind = _kind(r)
            a, b = (self.scalar(v) for v in op.operands)
            self.define(r, CTYPE[kind], f"({a} >= {b}) ? {a} : {b}")
            return True
        return False

    # ------------------------------------------------------------- memory
    def index_expr(self, op, view, idx_values) -> tuple[str, str]:
        """(ok condition, flat offset) for view[idx]; reports the first OOB index."""
        base, ext, st = self.memref(view)
        idx = [self.scalar(v) for v in idx_values]
        if len(idx) != len(ext):
            raise GenError("index rank does not match the memref", op)
        eid = self.error_id(op)
        conds = []
        for d, (i, e) in enumerate(zip(idx, ext)):
            conds.append(f"((unsigned long long)({i}) < (unsigned long long){e})")
        ok = self.fresh("ok")
        self.emit(f"bool {ok} = true;")
        for d, (i, e) in enumerate(zip(idx, ext)):
            self.emit(f"if ({ok} && !((unsigned long long)({i}) < (unsigned long long){e})) "
                      f"{{ {ok} = false; lb_err(lb_E, {ERR_OOB}, lb_eb + {eid}, (long long)({i}), {e}, {d}); }}")
        flat = " + ".join(f"(long long)({i}) * {s}" for i, s in zip(idx, st)) or "0"
        return ok, flat

    def emit_load(self, op, ctx: "_Ctx") -> None:
        view = op.operands[0]
        if view in self.count_loads:
            # a relaxed-stale read: the interpreter records one event per load
            self.emit(f"if ({ctx.canon}) {self.counter('stale', op)}++;")
        r = op.results[0]
        kind = _kind(r)
        base = self.memref(view)[0]
        ok, flat = self.index_expr(op, view, op.operands[1:])
        n = self.name(r)
        self.defined.add(r)
        self.emit(f"{CTYPE[kind]} {n} = 0;")
        self.emit(f"if ({ok}) {n} = ({CTYPE[kind]}){base}[{flat}];")

    def emit_store(self, op, ctx: _Ctx) -> None:
        val = self.scalar(op.operands[0])
        view = op.operands[1]
        kind = view.type.element.kind
        base = self.memref(view)[0]
        ok, flat = self.index_expr(op, view, op.operands[2:])
        cnt = self.counter("store", op)
        conv = f"(unsigned char)(({val}) & 1)" if kind == "i1" else val
        self.emit(f"if ({ctx.canon}) {{ if ({ok}) {base}[{flat}] = {conv}; {cnt}++; }}")

    # ------------------------------------------------------------ combiners
    def combine(self, acc: str, contrib: str, kind: str, comb, region) -> None:
        if comb == "add" or comb == "mul":
            sym = "+" if comb == "add" else "*"
            if kind in FLOAT_KINDS:
                self.emit(f"{acc} = {acc} {sym} {contrib};")
            else:
                u = UTYPE[kind]
                self.emit(f"{acc} = {self.wrap(kind, f'({u}){acc} {sym} ({u}){contrib}')};")
        elif comb == "min":
            self.emit(f"{acc} = ({acc} <= {contrib}) ? {acc} : {contrib};")
        elif comb == "max":
            self.emit(f"{acc} = ({acc} >= {contrib}) ? {acc} : {contrib};")
        else:
            # an unclassified combiner region: run its ops (interp.py:436-440)
            a, b = region.args
            self.emit("{")
            self.ind += 1
            self.define(a, CTYPE[kind], acc)
            self.define(b, CTYPE[kind], contrib)
            inner = _Ctx("vector", "true")
            for o in region.ops[:-1]:
                self.emit_op(o, inner)
            self.emit(f"{acc} = {self.scalar(region.ops[-1].operands[0])};")
            self.ind -= 1
            self.emit("}")

    def reduce_info(self, loop, inits):
        from lapis.dialect import classify_combiner
        term = loop.region(0).ops[-1]
        if term.name != "scf.reduce":
            raise GenError("reducing loop without scf.reduce terminator", loop)
        out = []
        for i, (init, contrib) in enumerate(zip(inits, term.operands)):
            out.append((_kind(init), classify_combiner(term.regions[i]), term.regions[i], contrib))
        return out

    # ------------------------------------------------------------ regions
    def emit_body(self, region, ctx: _Ctx) -> None:
        for o in region.ops:
            if o.name in ("scf.yield", "kokkos.yield", "scf.reduce"):
                continue
            self.emit_op(o, ctx)

    def emit_op(self, op, ctx: _Ctx) -> None:
        name = op.name
        if self.emit_arith(op):
            return
        if name == "memref.load":
            self.emit_load(op, ctx)
        elif name == "memref.store":
            self.emit_store(op, ctx)
        elif name == "memref.dim":
            v = op.operands[0]
            ext = self.memref(v)[1]
            self.define(op.results[0], "long long", ext[op.attrs["index"]])
        elif name == "scf.for":
            lo, hi, step = (self.scalar(v) for v in op.operands)
            iv = op.region(0).args[0]
            eid = self.error_id(op)
            n = self.name(iv)
            self.defined.add(iv)
            self.emit(f"if ({step} <= 0) lb_err(lb_E, {ERR_STEP}, lb_eb + {eid}, (long long){step}, 0, 0); else")
            self.emit(f"for (long long {n} = {lo}; {n} < {hi}; {n} += {step}) {{")
            self.ind += 1
            self.emit_body(op.region(0), ctx)
            self.ind -= 1
            self.emit("}")
        elif name == "scf.if":
            c = self.scalar(op.operands[0])
            self.emit(f"if ({c}) {{")
            self.ind += 1
            self.emit_body(op.region(0), ctx)
            self.ind -= 1
            if len(op.regions) > 1:
                self.emit("} else {")
                self.ind += 1
                self.emit_body(op.region(1), ctx)
                self.ind -= 1
            self.emit("}")
        elif name == "scf.parallel":
            self.emit_seq_parallel(op, ctx)
        elif name == "kokkos.range_parallel":
            level = op.attrs.get("parallelLevel")
            if level == "threadvector":
                self.emit_vector_loop(op, ctx)
            elif level == "teamthread":
                if ctx.level != "team":
                    raise GenError("teamthread loop outside a team", op)
                self.emit_teamthread_loop(op, ctx)
            else:
                raise GenError(f"nested {level} range", op)
        elif name == "kokkos.single":
            cnt = self.counter("single", op)
            self.emit(f"if ({ctx.canon}) {{")
            self.ind += 1
            self.emit(f"{cnt}++;")
            self.emit_body(op.region(0), _Ctx(ctx.level, "true"))
            self.ind -= 1
            self.emit("}")
        elif name == "kokkos.team_barrier":
            if ctx.level != "team":
                raise GenError("team_barrier outside team-level code", op)
            cnt = self.counter("barrier", op)
            self.emit(f"__syncthreads(); if ({ctx.canon}) {cnt}++;")
        else:
            raise GenError(f"no generated-kernel mapping for {name}", op)

    def emit_seq_parallel(self, op, ctx: _Ctx) -> None:
        """A nested scf.parallel (pre-lowering IR) runs sequentially inside the
        enclosing index, in the interpreter's row-major order."""
        from lapis.dialect import scf_parallel_bounds
        lows, ups, steps, inits = scf_parallel_bounds(op)
        args = op.region(0).args
        red = self.reduce_info(op, inits) if inits else []
        accs = []
        for r, init, (kind, _, _, _) in zip(op.results, inits, red):
            n = self.name(r)
            self.defined.add(r)
            self.emit(f"{CTYPE[kind]} {n} = {self.scalar(init)};")
            accs.append(n)
        eid = self.error_id(op)
        opened = 0
        for lo, hi, st, a in zip(lows, ups, steps, args):
            lo_, hi_, st_ = self.scalar(lo), self.scalar(hi), self.scalar(st)
            n = self.name(a)
            self.defined.add(a)
            self.emit(f"if ({st_} <= 0) lb_err(lb_E, {ERR_STEP}, lb_eb + {eid}, (long long){st_}, 0, 0); else")
            self.emit(f"for (long long {n} = {lo_}; {n} < {hi_}; {n} += {st_}) {{")
            self.ind += 1
            opened += 1
        self.emit_body(op.region(0), ctx)
        for acc, (kind, comb, region, contrib) in zip(accs, red):
            self.combine(acc, self.scalar(contrib), kind, comb, region)
        for _ in range(opened):
            self.ind -= 1
            self.emit("}")

    def emit_vector_loop(self, op, ctx: _Ctx) -> None:
        from lapis.dialect import parallel_init_operands
        n_ = self.scalar(op.operands[0])
        inits = parallel_init_operands(op)
        j = op.region(0).args[0]
        jn = self.name(j)
        self.defined.add(j)
        vctx = _Ctx("vector", "true")
        if not inits:
            self.emit(f"for (long long {jn} = lb_lane; {jn} < {n_}; {jn} += LB_VL) {{")
            self.ind += 1
            self.emit_body(op.region(0), vctx)
            self.ind -= 1
            self.emit("}")
            return
        red = self.reduce_info(op, inits)
        accs = []
        for r, init, (kind, _, _, _) in zip(op.results, inits, red):
            n = self.name(r)
            self.defined.add(r)
            self.emit(f"{CTYPE[kind]} {n} = {self.scalar(init)};")
            accs.append(n)
        b = self.fresh("b")
        self.emit(f"for (long long {b} = 0; {b} < {n_}; {b} += LB_VL) {{")
        self.ind += 1
        self.emit(f"const long long {jn} = {b} + lb_lane;")
        cs = []
        for kind, _, _, _ in red:
            c = self.fresh("c")
            self.emit(f"{CTYPE[kind]} {c} = 0;")
            cs.append(c)
        self.emit(f"if ({jn} < {n_}) {{")
        self.ind += 1
        self.emit_body(op.region(0), vctx)
        for c, (_, _, _, contrib) in zip(cs, red):
            self.emit(f"{c} = {self.scalar(contrib)};")
        self.ind -= 1
        self.emit("}")
        cnt = self.fresh("n")
        lane = self.fresh("l")
        self.emit(f"const int {cnt} = ({n_} - {b}) < LB_VL ? (int)({n_} - {b}) : LB_VL;")
        self.emit(f"for (int {lane} = 0; {lane} < {cnt}; ++{lane}) {{")
        self.ind += 1
        for acc, c, (kind, comb, region, _) in zip(accs, cs, red):
            x = self.fresh("x")
            self.emit(f"const {CTYPE[kind]} {x} = (LB_VL == 1) ? {c} : __shfl_sync(lb_gmask, {c}, {lane}, LB_VL);")
            self.combine(acc, x, kind, comb, region)
        self.ind -= 1
        self.emit("}")
        self.ind -= 1
        self.emit("}")

    def emit_teamthread_loop(self, op, ctx: _Ctx) -> None:
        from lapis.dialect import parallel_init_operands
        n_ = self.scalar(op.operands[0])
        inits = parallel_init_operands(op)
        i = op.region(0).args[0]
        iname = self.name(i)
        self.defined.add(i)
        tctx = _Ctx("thread", "(lb_lane == 0)")
        if not inits:
            self.emit(f"for (long long {iname} = lb_tt; {iname} < {n_}; {iname} += LB_TS) {{")
            self.ind += 1
            self.emit_body(op.region(0), tctx)
            self.ind -= 1
            self.emit("}")
            return
        red = self.reduce_info(op, inits)
        self.max_team_acc = max(self.max_team_acc, len(red))
        accs = []
        for r, init, (kind, _, _, _) in zip(op.results, inits, red):
            n = self.name(r)
            self.defined.add(r)
            self.emit(f"{CTYPE[kind]} {n} = {self.scalar(init)};")
            accs.append(n)
        b = self.fresh("b")
        self.emit(f"for (long long {b} = 0; {b} < {n_}; {b} += LB_TS) {{")
        self.ind += 1
        self.emit(f"const long long {iname} = {b} + lb_tt;")
        cs = []
        for kind, _, _, _ in red:
            c = self.fresh("c")
            self.emit(f"{CTYPE[kind]} {c} = 0;")
            cs.append(c)
        self.emit(f"if ({iname} < {n_}) {{")
        self.ind += 1
        self.emit_body(op.region(0), tctx)
        for c, (_, _, _, contrib) in zip(cs, red):
            self.emit(f"{c} = {self.scalar(contrib)};")
        self.ind -= 1
        self.emit("}")
        for k, (c, (kind, _, _, _)) in enumerate(zip(cs, red)):
            self.emit(f"if (lb_lane == 0) (({CTYPE[kind]}*)(lb_slots + {k} * LB_TS))[lb_tt] = {c};")
        self.emit("__syncthreads();")
        cnt = self.fresh("n")
        l_ = self.fresh("l")
        self.emit(f"const int {cnt} = ({n_} - {b}) < LB_TS ? (int)({n_} - {b}) : LB_TS;")
        self.emit(f"for (int {l_} = 0; {l_} < {cnt}; ++{l_}) {{")
        self.ind += 1
        for k, (acc, (kind, comb, region, _)) in enumerate(zip(accs, red)):
            x = self.fresh("x")
            self.emit(f"const {CTYPE[kind]} {x} = (({CTYPE[kind]}*)(lb_slots + {k} * LB_TS))[{l_}];")
            self.combine(acc, x, kind, comb, region)
        self.ind -= 1
        self.emit("}")
        self.emit("__syncthreads();")
        self.ind -= 1
        self.emit("}")

    # ------------------------------------------------------------ top level
    def generate(self) -> Kernel:
        from lapis.dialect import parallel_hint_operands, parallel_init_operands, scf_parallel_bounds
        top = self.top
        self._head: list[str] = []
        self._unpacked: set = set()
        E = self.slot("aux", aux="errors")
        Cn = self.slot("aux", aux="counters")
        EB = self.slot("aux", aux="errbase")
        body_start = len(self.lines)
        k = self.k
        if top.name == "kokkos.team_parallel":
            k.mapping = "team"
            ts_hint, _ = parallel_hint_operands(top)
            ts = self.ts_hint if self.ts_hint else max(1, BLOCK // self.vl)
            ts = max(1, min(ts, 1024 // self.vl))
            k.vl, k.ts, k.block = self.vl, ts, ts * self.vl
            inits = parallel_init_operands(top)
            league = self.scalar(top.operands[0])
            idx_arg = top.region(0).args[0]
            n = self.name(idx_arg)
            self.defined.add(idx_arg)
            self.emit(f"for (long long {n} = blockIdx.x; {n} < {league}; {n} += gridDim.x) {{")
            self.ind += 1
            ctx = _Ctx("team", "(lb_tt == 0 && lb_lane == 0)")
            self.emit_body(top.region(0), ctx)
            self.emit_top_contrib(top, inits, n, ctx)
            self.ind -= 1
            self.emit("}")
        elif top.name == "kokkos.thread_parallel":
            k.mapping = "thread"
            k.vl, k.ts, k.block = self.vl, BLOCK // self.vl, BLOCK
            inits = parallel_init_operands(top)
            nn = self.scalar(top.operands[0])
            idx_arg = top.region(0).args[0]
            n = self.name(idx_arg)
            self.defined.add(idx_arg)
            self.emit(f"for (long long {n} = lb_gid; {n} < {nn}; {n} += lb_ngroups) {{")
            self.ind += 1
            ctx = _Ctx("thread", "(lb_lane == 0)")
            self.emit_body(top.region(0), ctx)
            self.emit_top_contrib(top, inits, n, ctx)
            self.ind -= 1
            self.emit("}")
        elif top.name in ("kokkos.range_parallel", "scf.parallel"):
            k.mapping = "range"
            k.vl, k.ts, k.block = 1, BLOCK, BLOCK
            self.vl = 1
            args = top.region(0).args
            if top.name == "scf.parallel":
                lows, ups, steps, inits = scf_parallel_bounds(top)
                lows = [self.scalar(v) for v in lows]
                ups = [self.scalar(v) for v in ups]
                steps = [self.scalar(v) for v in steps]
            else:
                dims = top.attrs.get("dims", 1)
                ups = [self.scalar(v) for v in top.operands[:dims]]
                lows = ["0LL"] * dims
                steps = ["1LL"] * dims
                inits = parallel_init_operands(top)
            trips = []
            for d, (lo, hi, st) in enumerate(zip(lows, ups, steps)):
                t = f"lb_trip{d}"
                self._head.append(
                    f"const long long {t} = ({st} <= 0 || {hi} <= {lo}) ? 0LL : "
                    f"(({hi} - {lo}) + {st} - 1) / {st};")
                trips.append(t)
            eid = self.error_id(top)
            for st in steps:
                if st not in ("1LL",):
                    self._head.append(
                        f"if (blockIdx.x == 0 && threadIdx.x == 0 && {st} <= 0) "
                        f"lb_err(lb_E, {ERR_STEP}, lb_eb + {eid}, (long long){st}, 0, 0);")
            total = " * ".join(trips) or "1LL"
            self._head.append(f"const long long lb_total = {total};")
            self.emit("for (long long lb_t = (long long)blockIdx.x * blockDim.x + threadIdx.x; "
                      "lb_t < lb_total; lb_t += (long long)gridDim.x * blockDim.x) {")
            self.ind += 1
            self.emit("long long lb_r = lb_t;")
            for d in range(len(trips) - 1, -1, -1):
                a = args[d]
                an = self.name(a)
                self.defined.add(a)
                self.emit(f"const long long {an} = {lows[d]} + (lb_r % {trips[d]}) * {steps[d]};"
                          f" lb_r /= {trips[d]};")
            ctx = _Ctx("range", "true")
            self.emit_body(top.region(0), ctx)
            self.emit_top_contrib(top, inits, "lb_t", ctx)
            self.ind -= 1
            self.emit("}")
        else:
            raise GenError(f"{top.name} is not a kernel root", top)

        body = self.lines[body_start:]
        fold_src = self.fold_kernel() if k.top_reduce else ""
        nslots = len(k.slots)
        ncnt = len(k.counted)
        src = [_PRELUDE % {"nslots": max(nslots, 1)}]
        src.append(f"#define LB_VL {k.vl}")
        src.append(f"#define LB_TS {k.ts}")
        src.append(f'extern "C" __global__ void __launch_bounds__({k.block}) {k.name}(const LbParams P) {{')
        src.append(f"  unsigned long long* const lb_E = (unsigned long long*)P.s[{E}];")
        src.append(f"  unsigned long long* const lb_C = (unsigned long long*)P.s[{Cn}];")
        src.append(f"  const long long lb_eb = (long long)P.s[{EB}];")
        src.append("  const int lb_lane = (int)(threadIdx.x % LB_VL);")
        src.append("  const int lb_tt = (int)(threadIdx.x / LB_VL);")
        src.append("  const long long lb_gid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / LB_VL;")
        src.append("  const long long lb_ngroups = ((long long)gridDim.x * blockDim.x) / LB_VL;")
        src.append("  const unsigned lb_gmask = (LB_VL == 32) ? 0xffffffffu : "
                   "((0xffffffffu >> (32 - LB_VL)) << ((threadIdx.x & 31u) & ~(unsigned)(LB_VL - 1)));")
        src.append("  (void)lb_E; (void)lb_C; (void)lb_lane; (void)lb_tt; (void)lb_gid; "
                   "(void)lb_ngroups; (void)lb_gmask;")
        if self.max_team_acc:
            src.append(f"  __shared__ unsigned long long lb_slots[{self.max_team_acc} * LB_TS];")
        for i in range(ncnt):
            src.append(f"  unsigned long long lb_cnt{i} = 0;")
        for h in self._head:
            src.append("  " + h)
        src.extend(body)
        for i in range(ncnt):
            src.append(f"  if (lb_cnt{i}) atomicAdd(&lb_C[{i}], lb_cnt{i});")
        src.append("}")
        if fold_src:
            src.append(fold_src)
        k.source = "\n".join(src) + "\n"
        return k

    def emit_top_contrib(self, top, inits, index_expr: str, ctx: _Ctx) -> None:
        """A top-level reduce returns scalars to the host: each index writes its
        contribution; a one-thread fold kernel combines them in index order."""
        if not inits:
            return
        red = self.reduce_info(top, inits)
        k = self.k
        for r, (kind, comb, region, contrib) in enumerate(red):
            s = self.slot("aux", aux=f"contrib{r}")
            c = self.scalar(contrib)
            self.emit(f"if ({ctx.canon}) (({CTYPE[kind]}*)P.s[{s}])[{index_expr}] = {c};")
            k.top_reduce.append((kind, comb, region, inits[r]))

    def fold_kernel(self) -> str:
        k = self.k
        k.fold_name = k.name + "_fold"
        self.lines = []
        self.ind = 1
        n = self.slot("aux", aux="fold_n")
        lines_head = [f'extern "C" __global__ void __launch_bounds__(32) {k.fold_name}(const LbParams P) {{',
                      "  if (threadIdx.x != 0 || blockIdx.x != 0) return;",
                      f"  unsigned long long* const lb_E = (unsigned long long*)P.s[{self.slot('aux', aux='errors')}];",
                      f"  const long long lb_eb = (long long)P.s[{self.slot('aux', aux='errbase')}];",
                      "  (void)lb_E; (void)lb_eb;",
                      f"  const long long lb_n = (long long)P.s[{n}];"]
        for r, (kind, comb, region, init) in enumerate(k.top_reduce):
            c = self.slot("aux", aux=f"contrib{r}")
            o = self.slot("aux", aux=f"out{r}")
            i0 = self.slot("aux", aux=f"init{r}")
            ct = CTYPE[kind]
            if kind == "f64":
                self.emit(f"double acc{r} = __longlong_as_double((long long)P.s[{i0}]);")
            elif kind == "f32":
                self.emit(f"float acc{r} = __int_as_float((int)(unsigned)P.s[{i0}]);")
            else:
                self.emit(f"{ct} acc{r} = ({ct})(long long)P.s[{i0}];")
            self.emit(f"for (long long i = 0; i < lb_n; ++i) {{")
            self.ind += 1
            self.emit(f"const {ct} x = (({ct}*)P.s[{c}])[i];")
            self.combine(f"acc{r}", "x", kind, comb, region)
            self.ind -= 1
            self.emit("}")
            self.emit(f"(({ct}*)P.s[{o}])[0] = acc{r};")
        return "\n".join(lines_head + self.lines + ["}"])


def generate(top, name: str, vl: int = 1, ts: int | None = None, count_loads=()) -> Kernel:
    """CUDA source + parameter layout for one top-level nest.  Loads from the
    memref values in ``count_loads`` are counted (category "stale")."""
    return NestGen(top, name, vl=vl, ts=ts, count_loads=count_loads).generate()


# --------------------------------------------------------------- library ops
class LibGen(NestGen):
    """The library ops (linalg.*, kokkos.gemm / gemv, sparse.spmv_csr) as
    generated kernels: one thread per output element, the reduction in the
    interpreter's sequential order (interp.py:704-812, 949-976).  This is the
    exact path (``run(..., exact=True)``) and the path for element types the
    hand-written kernels do not take; shape errors are raised on the host
    before launch (runtime.py)."""

    def arith(self, kind: str, sym: str, a: str, b: str) -> str:
        if kind in FLOAT_KINDS:
            return f"({a} {sym} {b})"
        u = UTYPE[kind]
        return self.wrap(kind, f"({u}){a} {sym} ({u}){b}")

    def load(self, op, view, idx: list) -> str:
        kind = view.type.element.kind
        base, ext, st = self.memref(view)
        eid = self.error_id(op)
        ok = self.fresh("ok")
        self.emit(f"bool {ok} = true;")
        for d, (i, e) in enumerate(zip(idx, ext)):
            self.emit(f"if ({ok} && !((unsigned long long)({i}) < (unsigned long long){e})) "
                      f"{{ {ok} = false; lb_err(lb_E, {ERR_OOB}, lb_eb + {eid}, (long long)({i}), {e}, {d}); }}")
        flat = " + ".join(f"(long long)({i}) * {s}" for i, s in zip(idx, st)) or "0"
        v = self.fresh("ld")
        self.emit(f"{CTYPE[kind]} {v} = 0;")
        self.emit(f"if ({ok}) {v} = ({CTYPE[kind]}){base}[{flat}];")
        return v

    def store(self, view, idx: list, val: str) -> None:
        kind = view.type.element.kind
        base, ext, st = self.memref(view)
        flat = " + ".join(f"(long long)({i}) * {s}" for i, s in zip(idx, st)) or "0"
        conv = f"(unsigned char)(({val}) & 1)" if kind == "i1" else val
        self.emit(f"{base}[{flat}] = {conv};")

    def generate(self) -> Kernel:
        op = self.top
        self._head = []
        self._unpacked = set()
        E = self.slot("aux", aux="errors")
        Cn = self.slot("aux", aux="counters")
        EB = self.slot("aux", aux="errbase")
        k = self.k
        k.mapping, k.vl, k.ts, k.block = "range", 1, BLOCK, BLOCK
        name = op.name
        if name == "linalg.fill":
            out = op.operands[1]
            dims = self.memref(out)[1]
            idx = self.open_range(dims)
            self.store(out, idx, self.scalar(op.operands[0]))
        elif name == "linalg.elementwise":
            ins, out = op.operands[:-1], op.operands[-1]
            dims = self.memref(out)[1]
            idx = self.open_range(dims)
            body = op.region(0)
            for arg, view in zip(body.args, ins):
                v = self.load(op, view, idx)
                self.define(arg, CTYPE[_kind(arg)], v)
            ctx = _Ctx("range", "true")
            for o in body.ops[:-1]:
                if o.name in ("memref.load", "memref.store"):
                    raise GenError("memory access inside an elementwise body", o)
                self.emit_op(o, ctx)
            self.store(out, idx, self.scalar(body.ops[-1].operands[0]))
        elif name == "linalg.reduce":
            src, dst = op.operands[0], op.operands[1]
            axes = list(op.attrs["axes"])
            comb = op.attrs["combiner"]
            kind = src.type.element.kind
            sdims = self.memref(src)[1]
            kept = [d for d in range(len(sdims)) if d not in axes]
            idx = self.open_range([sdims[d] for d in kept])
            acc = self.fresh("acc")
            self.emit(f"{CTYPE[kind]} {acc} = {identity_literal(comb, kind)};")
            full = [None] * len(sdims)
            for d, i in zip(kept, idx):
                full[d] = i
            opened = 0
            for d in axes:
                r = self.fresh("r")
                self.emit(f"for (long long {r} = 0; {r} < {sdims[d]}; ++{r}) {{")
                self.ind += 1
                opened += 1
                full[d] = r
            v = self.load(op, src, full)
            self.combine(acc, v, kind, comb, None)
            for _ in range(opened):
                self.ind -= 1
                self.emit("}")
            self.store(dst, idx, acc)
        elif name in ("linalg.matmul", "kokkos.gemm", "linalg.batch_matmul"):
            a, b, c = op.operands[:3]
            kind = c.type.element.kind
            cd = self.memref(c)[1]
            ad = self.memref(a)[1]
            idx = self.open_range(cd)
            kk = ad[-1]
            acc = self.fresh("acc")
            self.emit(f"{CTYPE[kind]} {acc} = 0;")
            r = self.fresh("k")
            self.emit(f"for (long long {r} = 0; {r} < {kk}; ++{r}) {{")
            self.ind += 1
            lead = idx[:-2]
            x = self.load(op, a, lead + [idx[-2], r])
            y = self.load(op, b, lead + [r, idx[-1]])
            p = self.fresh("p")
            self.emit(f"const {CTYPE[kind]} {p} = {self.arith(kind, '*', x, y)};")
            self.emit(f"{acc} = {self.arith(kind, '+', acc, p)};")
            self.ind -= 1
            self.emit("}")
            self.store(c, idx, acc)
        elif name in ("linalg.matvec", "kokkos.gemv"):
            a, x, y = op.operands[:3]
            kind = y.type.element.kind
            ad = self.memref(a)[1]
            idx = self.open_range([self.memref(y)[1][0]])
            acc = self.fresh("acc")
            self.emit(f"{CTYPE[kind]} {acc} = 0;")
            r = self.fresh("j")
            self.emit(f"for (long long {r} = 0; {r} < {ad[1]}; ++{r}) {{")
            self.ind += 1
            u = self.load(op, a, [idx[0], r])
            w = self.load(op, x, [r])
            p = self.fresh("p")
            self.emit(f"const {CTYPE[kind]} {p} = {self.arith(kind, '*', u, w)};")
            self.emit(f"{acc} = {self.arith(kind, '+', acc, p)};")
            self.ind -= 1
            self.emit("}")
            self.store(y, idx, acc)
        elif name in ("sparse.spmv_csr", "kokkos.spmv_csr"):
            rp, ci, vals, x, y = op.operands
            kind = y.type.element.kind
            rpd = self.memref(rp)[1]
            idx = self.open_range([f"({rpd[0]} - 1)"])
            i = idx[0]
            b = self.load(op, rp, [i])
            e = self.load(op, rp, [f"({i} + 1)"])
            acc = self.fresh("acc")
            self.emit(f"{CTYPE[kind]} {acc} = 0;")
            j = self.fresh("j")
            self.emit(f"for (long long {j} = (long long){b}; {j} < (long long){e}; ++{j}) {{")
            self.ind += 1
            col = self.load(op, ci, [j])
            v = self.load(op, vals, [j])
            xv = self.load(op, x, [col])
            p = self.fresh("p")
            self.emit(f"const {CTYPE[kind]} {p} = {self.arith(kind, '*', v, xv)};")
            self.emit(f"{acc} = {self.arith(kind, '+', acc, p)};")
            self.ind -= 1
            self.emit("}")
            self.store(y, idx, acc)
        else:
            raise GenError(f"no generated kernel for {name}", op)
        self.ind -= 1
        self.emit("}")
        body = self.lines
        src = [_PRELUDE % {"nslots": max(len(k.slots), 1)}]
        src.append(f"#define LB_VL 1")
        src.append(f"#define LB_TS {BLOCK}")
        src.append(f'extern "C" __global__ void __launch_bounds__({BLOCK}) {k.name}(const LbParams P) {{')
        src.append(f"  unsigned long long* const lb_E = (unsigned long long*)P.s[{E}];")
        src.append(f"  const long long lb_eb = (long long)P.s[{EB}];")
        src.append(f"  (void)P.s[{Cn}];")
        for h in self._head:
            src.append("  " + h)
        src.extend(body)
        src.append("}")
        k.source = "\n".join(src) + "\n"
        return k

    def open_range(self, dims: list) -> list:
        """Grid-stride loop over the row-major index space `dims`; returns the
        per-dimension index names (the loop stays open until generate())."""
        total = " * ".join(f"(long long)({d})" for d in dims) or "1LL"
        self._head.append(f"const long long lb_total = {total};")
        self.emit("for (long long lb_t = (long long)blockIdx.x * blockDim.x + threadIdx.x; "
                  "lb_t < lb_total; lb_t += (long long)gridDim.x * blockDim.x) {")
        self.ind += 1
        self.emit("long long lb_r = lb_t;")
        names = [None] * len(dims)
        for d in range(len(dims) - 1, -1, -1):
            n = self.fresh("i")
            self.emit(f"const long long {n} = lb_r % ({dims[d]}); lb_r /= ({dims[d]});")
            names[d] = n
        return names


def identity_literal(comb: str, kind: str) -> str:
    """The combiner identity (interp.py:186-195)."""
    if kind in FLOAT_KINDS:
        v = {"add": 0.0, "mul": 1.0, "min": float("inf"), "max": float("-inf")}[comb]
        return literal(v, kind)
    w = WIDTH[kind]
    v = {"add": 0, "mul": 1, "min": (1 << (w - 1)) - 1, "max": -(1 << (w - 1))}[comb]
    if kind == "i1":
        return str(v)  # the interpreter keeps -1 unwrapped as the i1 max identity
    return literal(v, kind)


LIBRARY_OPS = ("linalg.fill", "linalg.elementwise", "linalg.reduce", "linalg.matmul", "kokkos.gemm",
               "linalg.batch_matmul", "linalg.matvec", "kokkos.gemv", "sparse.spmv_csr",
               "kokkos.spmv_csr")


def generate_library(op, name: str) -> Kernel:
    return LibGen(op, name).generate()
