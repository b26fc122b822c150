"""PyTorch frontend: a torch.fx graph of a small sparse model -> LAPIS IR.

The paper drives LAPIS from PyTorch through torch-mlir / MPACT (PAPER.md:148,
298-313, 362): ``torch.mv(A_csr, x)`` becomes ``sparse.spmv_csr``,
``torch.matmul`` becomes ``linalg.matmul``, and a GCN layer becomes one
function of loop nests (oracle/ir/gcn_f32.mlir).  The reference
artifact ships no such frontend, so this module is the thin equivalent for the
model family the BASELINE names (config 4: SpMM + dense matmul + ReLU):

  * ``torch.fx.symbolic_trace`` the module;
  * map each node onto the IR the reference's own fixtures use —
      torch.sparse.mm / torch.mm / matmul / @ with a sparse CSR left operand
          -> the loop-nest SpMM of oracle/ir/spmm.mlir (2-D result) or
             sparse.spmv_csr (1-D result, tests/fixtures/spmv.mlir)
      nn.Linear(bias=False), torch.mm / matmul of two dense operands
          -> linalg.matmul (the Linear's weight enters as its transpose W)
      torch.relu / F.relu / nn.ReLU
          -> linalg.elementwise { cmpf ogt ; select }
  * emit the function text, parse it with the reference's parser and lower it
    with the reference's own pipeline (``run_pipeline(..., PassPipeline.preset(),
    TargetConfig())``);
  * run it with ``paper_2509_25605_b200.runtime.run`` (the B200 drop-in for
    ``lapis.interp.run``) or, for checking, with the reference interpreter.

Anything outside that op set raises ``FrontendError`` — no silent fallback.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

_DT = {torch.float32: "f32", torch.float64: "f64"}
_NP = {torch.float32: np.float32, torch.float64: np.float64}


class FrontendError(Exception):
    pass


@dataclass
class Lowered:
    """IR text of the traced model plus how to build its argument list."""
    text: str
    entry: str
    args: list = field(default_factory=list)     # ("csr", name) | ("dense", name) | ("param", tensor^T)
    out_shape_of: object = None                  # callable(inputs) -> output shape

    def inputs(self, *tensors) -> list:
        """numpy argument list for (lapis.interp | runtime).run from the
        model's forward arguments (CSR tensors are split into rowptr /
        colind / values)."""
        out, it = [], iter(tensors)
        for kind, v in self.args:
            if kind == "csr":
                a = next(it)
                out += [a.crow_indices().cpu().numpy().astype(np.int64),
                        a.col_indices().cpu().numpy().astype(np.int32),
                        a.values().cpu().numpy()]
            elif kind == "dense":
                out.append(np.ascontiguousarray(next(it).detach().cpu().numpy()))
            elif kind == "param":
                out.append(np.ascontiguousarray(v))
        shape, dtype = self.out_shape_of(tensors)
        out.append(np.zeros(shape, dtype=dtype))
        return out


class _Emitter:
    def __init__(self, dt: str):
        self.dt = dt
        self.lines: list[str] = []
        self.n = 0
        self.consts_done = False

    def fresh(self, stem: str) -> str:
        self.n += 1
        return f"%{stem}{self.n}"

    def consts(self):
        if not self.consts_done:
            self.lines += ["  %c0 = arith.constant 0 : index", "  %c1 = arith.constant 1 : index"]
            self.consts_done = True

    def dim(self, v: str, i: int) -> str:
        d = self.fresh("d")
        self.lines.append(f"  {d} = memref.dim({v}) {{index = {i}}}")
        return d

    def alloc(self, *dims) -> str:
        t = self.fresh("t")
        ty = "x".join(["?"] * len(dims)) + f"x{self.dt}"
        self.lines.append(f"  {t} = memref.alloc({', '.join(dims)}) : memref<{ty}>")
        return t

    # loop-nest SpMM, exactly the nest of oracle/ir/spmm.mlir / gcn_f32.mlir
    def spmm(self, rp, ci, vals, x, out, nrows, k):
        dt = self.dt
        i, c = self.fresh("i"), self.fresh("c")
        b, e, ln, s = self.fresh("b"), self.fresh("e"), self.fresh("len"), self.fresh("sum")
        inx, z, jj, j = self.fresh("in"), self.fresh("z"), self.fresh("jj"), self.fresh("j")
        v, c32, col, xv, p = (self.fresh("v"), self.fresh("col32"), self.fresh("col"),
                              self.fresh("xv"), self.fresh("p"))
        ra, rb, rs = self.fresh("ra"), self.fresh("rb"), self.fresh("rs")
        self.lines += [
            f"  scf.parallel ({i}, {c}) = (%c0, %c0) to ({nrows}, {k}) step (%c1, %c1) {{",
            f"    {b} = memref.load {rp}[{i}]",
            f"    {inx} = arith.addi({i}, %c1)",
            f"    {e} = memref.load {rp}[{inx}]",
            f"    {ln} = arith.subi({e}, {b})",
            f"    {z} = arith.constant 0.0 : {dt}",
            f"    {s} = scf.parallel {jj} = %c0 to {ln} step %c1 init({z}) {{",
            f"      {j} = arith.addi({b}, {jj})",
            f"      {v} = memref.load {vals}[{j}]",
            f"      {c32} = memref.load {ci}[{j}]",
            f"      {col} = arith.index_cast({c32}) : index",
            f"      {xv} = memref.load {x}[{col}, {c}]",
            f"      {p} = arith.mulf({v}, {xv})",
            f"      scf.reduce({p}) {{",
            f"        ^({ra}: {dt}, {rb}: {dt}):",
            f"          {rs} = arith.addf({ra}, {rb})",
            f"          scf.reduce.return({rs})",
            "      }",
            "    }",
            f"    memref.store {s}, {out}[{i}, {c}]",
            "    scf.yield",
            "  }",
        ]

    def relu(self, src, dst):
        dt = self.dt
        v, z, pos, r = self.fresh("rv"), self.fresh("rz"), self.fresh("rpos"), self.fresh("rr")
        self.lines += [
            f"  linalg.elementwise({src}, {dst}) {{",
            f"    ^({v}: {dt}):",
            f"      {z} = arith.constant 0.0 : {dt}",
            f"      {pos} = arith.cmpf({v}, {z}) {{predicate = \"ogt\"}}",
            f"      {r} = arith.select({pos}, {v}, {z})",
            f"      scf.yield({r})",
            "  }",
        ]


def _is_sparse(t) -> bool:
    return isinstance(t, torch.Tensor) and t.layout == torch.sparse_csr


def lower_module(module: torch.nn.Module, *example, entry: str = "forward") -> Lowered:
    """Trace `module` with torch.fx and emit its LAPIS IR (see module docstring).
    `example` are forward arguments (a torch.sparse_csr_tensor for each sparse
    operand); they fix the element type and which operands are sparse."""
    import torch.fx as fx
    gm = fx.symbolic_trace(module)
    mods = dict(gm.named_modules())
    dense_dt = next((t.dtype for t in example if isinstance(t, torch.Tensor) and not _is_sparse(t)),
                    torch.float32)
    if dense_dt not in _DT:
        raise FrontendError(f"unsupported element type {dense_dt}")
    dt = _DT[dense_dt]
    em = _Emitter(dt)
    sig, args = [], []
    env: dict = {}          # fx node -> ("csr", (rp, ci, v, nrows_sym)) | ("dense", name, rank)
    ph = iter(example)
    for node in gm.graph.nodes:
        if node.op != "placeholder":
            continue
        t = next(ph)
        nm = node.name
        if _is_sparse(t):
            sig += [f"%{nm}_rowptr: memref<?xindex>", f"%{nm}_colind: memref<?xi32>",
                    f"%{nm}_values: memref<?x{dt}>"]
            args.append(("csr", nm))
            env[node] = ("csr", (f"%{nm}_rowptr", f"%{nm}_colind", f"%{nm}_values"))
        else:
            rank = t.dim()
            sig.append(f"%{nm}: memref<{'x'.join(['?'] * rank)}x{dt}>")
            args.append(("dense", nm))
            env[node] = ("dense", f"%{nm}", rank)
    em.consts()
    pending_out = []      # (value name, rank) of the node feeding `output`

    def dense_of(n):
        kind = env[n]
        if kind[0] != "dense":
            raise FrontendError(f"{n} must be dense here")
        return kind[1], kind[2]

    def rows_of(csr):
        rp = csr[0]
        nb = em.dim(rp, 0)
        nr = em.fresh("nrows")
        em.lines.append(f"  {nr} = arith.subi({nb}, %c1)")
        return nr

    def matmul(a, b):
        m, k2 = em.dim(a, 0), em.dim(b, 1)
        t = em.alloc(m, k2)
        em.lines.append(f"  linalg.matmul({a}, {b}, {t})")
        return t

    params = {}
    for node in gm.graph.nodes:
        if node.op in ("placeholder",):
            continue
        if node.op == "output":
            src = node.args[0]
            if isinstance(src, (tuple, list)):
                if len(src) != 1:
                    raise FrontendError("one output only")
                src = src[0]
            pending_out.append(env[src])
            continue
        target = node.target
        if node.op == "call_module":
            sub = mods[target]
            if isinstance(sub, torch.nn.Linear):
                if sub.bias is not None:
                    raise FrontendError("nn.Linear with bias is not in the supported op set")
                w = f"%{node.name}_w"
                sig.append(f"{w}: memref<?x?x{dt}>")
                wt = sub.weight.detach().t().contiguous().cpu().numpy().astype(_NP[dense_dt])
                args.append(("param", wt))
                a, _ = dense_of(node.args[0])
                env[node] = ("dense", matmul(a, w), 2)
            elif isinstance(sub, torch.nn.ReLU):
                a, r = dense_of(node.args[0])
                dims = [em.dim(a, i) for i in range(r)]
                t = em.alloc(*dims)
                em.relu(a, t)
                env[node] = ("dense", t, r)
            else:
                raise FrontendError(f"module {type(sub).__name__} is not in the supported op set")
            continue
        if node.op == "get_attr":
            p = getattr(gm, target)
            if not isinstance(p, torch.Tensor) or p.dim() != 2:
                raise FrontendError("only rank-2 dense parameters are supported")
            w = f"%{node.name}"
            sig.append(f"{w}: memref<?x?x{dt}>")
            args.append(("param", p.detach().cpu().numpy().astype(_NP[dense_dt])))
            env[node] = ("dense", w, 2)
            params[node] = p
            continue
        if node.op == "call_method" and target in ("t",) and node.args[0] in params:
            p = params[node.args[0]].t().contiguous()
            args[-1] = ("param", p.detach().cpu().numpy().astype(_NP[dense_dt]))
            env[node] = env[node.args[0]]
            continue
        if node.op not in ("call_function", "call_method"):
            raise FrontendError(f"unsupported node {node.op} {target}")
        name = getattr(target, "__name__", str(target))
        if name in ("mm", "matmul", "matmul_", "__matmul__", "mv") or target in (
                torch.sparse.mm, torch.mm, torch.matmul, torch.mv):
            lhs, rhs = node.args[0], node.args[1]
            if env[lhs][0] == "csr":
                csr = env[lhs][1]
                x, r = dense_of(rhs)
                nr = rows_of(csr)
                if r == 1:
                    y = em.alloc(nr)
                    em.lines.append(f"  sparse.spmv_csr({', '.join(csr)}, {x}, {y})")
                    env[node] = ("dense", y, 1)
                else:
                    k = em.dim(x, 1)
                    y = em.alloc(nr, k)
                    em.spmm(*csr, x, y, nr, k)
                    env[node] = ("dense", y, 2)
            else:
                a, ra = dense_of(lhs)
                b, rb = dense_of(rhs)
                if ra != 2 or rb != 2:
                    raise FrontendError("dense matmul of rank-2 operands only")
                env[node] = ("dense", matmul(a, b), 2)
            continue
        if name in ("relu",) or target in (torch.relu, torch.nn.functional.relu):
            a, r = dense_of(node.args[0])
            dims = [em.dim(a, i) for i in range(r)]
            t = em.alloc(*dims)
            em.relu(a, t)
            env[node] = ("dense", t, r)
            continue
        raise FrontendError(f"op {name} is not in the supported op set")
    if len(pending_out) != 1 or pending_out[0][0] != "dense":
        raise FrontendError("the model must return one dense tensor")
    _, res, rank = pending_out[0]
    sig.append(f"%out: memref<{'x'.join(['?'] * rank)}x{dt}>")
    # the last temporary IS the caller's output buffer: drop its alloc and
    # rename it (the reference fixtures write results into an argument)
    import re
    alloc = re.compile(r"^\s*" + re.escape(res) + r" = memref\.alloc\(")
    if not any(alloc.match(ln) for ln in em.lines):
        raise FrontendError("the model's result must be computed by a supported op")
    em.lines = [ln for ln in em.lines if not alloc.match(ln)]
    pat = re.compile(re.escape(res) + r"(?![0-9A-Za-z_])")
    em.lines = [pat.sub("%out", ln) for ln in em.lines]
    ty = "x".join(["?"] * rank) + f"x{dt}"
    text = (f"// generated by paper_2509_25605_b200.frontend from {type(module).__name__}\n"
            f"func @{entry}({', '.join(sig)}) -> (memref<{ty}>) {{\n" + "\n".join(em.lines) +
            "\n  func.return(%out)\n}\n")

    def out_shape_of(tensors):
        with torch.no_grad():
            o = module(*[t for t in tensors])
        return tuple(o.shape), _NP[dense_dt]

    return Lowered(text=text, entry=entry, args=args, out_shape_of=out_shape_of)


def compile_module(module, *example, lowered_pipeline: bool = True):
    """(Lowered, program) — the program parsed by the reference parser and,
    by default, lowered by the reference's preset pipeline."""
    from lapis.parser import parse
    low = lower_module(module, *example)
    program = parse(low.text)
    if lowered_pipeline:
        from lapis.passes import PassPipeline, TargetConfig, run_pipeline
        program = run_pipeline(program, PassPipeline.preset(), TargetConfig()).program
    return low, program


def run_module(module, *tensors, backend: str = "b200", config=None):
    """Run the traced model on `tensors`: backend "b200" uses
    paper_2509_25605_b200.runtime.run, "interp" the reference interpreter.
    Returns (output ndarray, RunResult)."""
    low, program = compile_module(module, *tensors)
    inputs = low.inputs(*tensors)
    if backend == "interp":
        from lapis.interp import run
    else:
        from .runtime import run
    res = run(program, low.entry, inputs, config)
    return np.asarray(res.outputs[0]), res
