"""Seeded synthetic inputs of the BASELINE configs, defined on
the host with numpy so that both bench arms — the B200 backend and the
reference's own CPU path (`bench.py --impl reference`) — read the very same
numbers without either one depending on the other's code.  Nothing here imports
the backend package or the oracle: the B200 arm may build a structure on the
device (torch ops that give bit-identical integers, below), the reference arm
builds only the bounded row window it times, on the host.

Power-law matrix (configs 3 and 4): Chung-Lu with Pareto row
weights of density exponent alpha = 2.5,

  w_i = (1 - u_i)^(-1 / (alpha - 1))          u_i = default_rng(seed).random(n)
  W_i = w_i * mean * n / sum(w)                (expected row length)
  d_i = floor(W_i) + [i among the (mean*n - sum floor(W)) largest remainders]
                                               (exactly mean * n draws, no empty row)
  columns of row i: searchsorted(cumsum(W), u * cumsum(W)[-1]) for the next d_i
        uniforms of the same generator (columns drawn in proportion to the
        same weights); the hubs sit at random positions (iid weights)
  per-row sort + dedupe of (row, column); values U(-1, 1) from the same
        generator, in final entry order (config 3).

At n = 10,000,000, mean 10, seed 1 this gives nnz 99,891,191, longest row
117,683, median 5, p99 72, no empty row (checksums pinned in
tests/test_synth_inputs.py).  SURVEY A.8's own script was not committed; its
printed result (nnz 99,891,811, max 117,686, median 5, p99 72, no empty rows)
is reproduced to 6e-6 in nnz and 3 entries in the hub row — the difference is
the unpublished order of its random draws.
"""
from __future__ import annotations

import numpy as np

POWERLAW_ALPHA = 2.5


# ------------------------------------------------------------------- stencils
def stencil_nnz(points: int, n: int) -> int:
    return (3 * n - 2) ** 3 if points == 27 else 5 * n * n - 4 * n


def stencil_rows(points: int, n: int, a: int, b: int, colind_dtype=np.int64):
    """Rows [a, b) of the 5-point 2-D (diagonal 4) or 27-point 3-D (diagonal
    26) stencil in natural order, ascending columns, off-diagonals -1:
    (rowptr int64 rebased to 0, colind, values f64).  Same matrix as the
    device generator lapis_b200_synth_stencil (csrc/synth.cu)."""
    r = np.arange(a, b, dtype=np.int64)
    if points == 5:
        coords = [r // n, r % n]
        offs = [(di, dj) for di in (-1, 0, 1) for dj in (-1, 0, 1) if abs(di) + abs(dj) <= 1]
        diag_val = 4.0
    else:
        coords = [r // (n * n), (r // n) % n, r % n]
        offs = [(di, dj, dk) for di in (-1, 0, 1) for dj in (-1, 0, 1) for dk in (-1, 0, 1)]
        diag_val = 26.0
    # offsets in ascending column order: lexicographic in (di, dj, dk)
    offs.sort()
    cols = np.empty((r.size, len(offs)), dtype=np.int64)
    keep = np.ones((r.size, len(offs)), dtype=bool)
    for t, o in enumerate(offs):
        c = np.zeros(r.size, dtype=np.int64)
        for ax, d in enumerate(o):
            q = coords[ax] + d
            keep[:, t] &= (q >= 0) & (q < n)
            c = c * n + q
        cols[:, t] = c
    counts = keep.sum(1)
    rowptr = np.zeros(r.size + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    colind = cols[keep].astype(colind_dtype)
    values = np.where(colind == np.repeat(r, counts), diag_val, -1.0)
    return rowptr, colind, values


def stencil_x(points: int, n: int, seed: int):
    N = n ** 3 if points == 27 else n * n
    return np.random.default_rng(seed).uniform(-1.0, 1.0, N)


# ------------------------------------------------------------------ power law
class PowerLawSpec:
    """The row-length and column-weight tables of the power-law generator
    (module docstring); the column draws follow in the same generator."""

    def __init__(self, n: int, mean: float = 10.0, seed: int = 1, alpha: float = POWERLAW_ALPHA):
        self.n, self.mean, self.seed, self.alpha = n, mean, seed, alpha
        rng = np.random.default_rng(seed)
        w = (1.0 - rng.random(n)) ** (-1.0 / (alpha - 1.0))
        W = w * (mean * n / w.sum())
        fl = np.floor(W).astype(np.int64)
        self.total = int(round(mean * n))
        rem = self.total - int(fl.sum())
        if rem > 0:
            fl[np.argsort(-(W - fl), kind="stable")[:rem]] += 1
        self.deg = fl
        self.cdf = np.cumsum(W)
        self.draws_before_cols = n           # generator position of the first column draw
        self.offsets = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(self.deg, out=self.offsets[1:])

    def generator_at(self, position: int) -> np.random.Generator:
        """default_rng(seed) advanced by `position` doubles."""
        g = np.random.default_rng(self.seed)
        g.bit_generator.advance(position)
        return g

    def column_uniforms(self, first_draw: int, count: int) -> np.ndarray:
        return self.generator_at(self.draws_before_cols + first_draw).random(count)

    def columns_of(self, u: np.ndarray) -> np.ndarray:
        c = np.searchsorted(self.cdf, u * self.cdf[-1])
        return np.minimum(c, self.n - 1)

    def values_position(self) -> int:
        """Generator position of the first value draw (after every column draw)."""
        return self.draws_before_cols + self.total


def _dedupe(rows: np.ndarray, cols: np.ndarray, n: int, nrows: int, row0: int = 0):
    key = np.unique((rows - row0) * n + cols)
    r = key // n
    colind = (key - r * n).astype(np.int32)
    rowptr = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=nrows), out=rowptr[1:])
    return rowptr, colind


def powerlaw_structure_host(spec: PowerLawSpec, rows: int | None = None):
    """(rowptr, colind int32) of rows [0, rows) (all rows by default) on the
    host: only the column draws of those rows are generated."""
    nr = spec.n if rows is None else min(rows, spec.n)
    m = int(spec.offsets[nr])
    cols = spec.columns_of(spec.column_uniforms(0, m))
    r = np.repeat(np.arange(nr, dtype=np.int64), spec.deg[:nr])
    return _dedupe(r, cols, spec.n, nr)


def powerlaw_structure_device(spec: PowerLawSpec, device="cuda", chunk: int = 25_000_000):
    """The full structure built with torch on the device: the same uniforms
    (numpy), the same float64 products and the same left-side binary search
    (torch.searchsorted, right=False), then a sort-based dedupe — integers, so
    bit-identical to powerlaw_structure_host."""
    import torch
    n = spec.n
    cdf = torch.from_numpy(spec.cdf).to(device)
    scale = float(spec.cdf[-1])
    g = spec.generator_at(spec.draws_before_cols)
    keys = []
    deg = torch.from_numpy(spec.deg).to(device)
    rows_all = torch.repeat_interleave(torch.arange(n, device=device, dtype=torch.int64), deg)
    for c0 in range(0, spec.total, chunk):
        m = min(chunk, spec.total - c0)
        u = torch.from_numpy(g.random(m)).to(device)
        c = torch.searchsorted(cdf, u * scale).clamp_(max=n - 1)
        keys.append(rows_all[c0:c0 + m] * n + c)
        del u, c
    del rows_all
    key = torch.unique(torch.cat(keys))
    del keys
    r = torch.div(key, n, rounding_mode="floor")
    colind = (key - r * n).to(torch.int32)
    rowptr = torch.zeros(n + 1, dtype=torch.int64, device=device)
    rowptr[1:] = torch.cumsum(torch.bincount(r, minlength=n), 0)
    return rowptr, colind.contiguous()


def powerlaw_values(spec: PowerLawSpec, nnz: int, first: int = 0, count: int | None = None):
    """Values U(-1, 1) of entries [first, first + count) in final entry order."""
    count = nnz - first if count is None else count
    return spec.generator_at(spec.values_position() + first).uniform(-1.0, 1.0, count)


def spmm_dense(n: int, k: int, seed: int) -> np.ndarray:
    """Config 3's dense operand X [n, k] f64 U(-1, 1) (default_rng(seed + 100))."""
    return np.random.default_rng(seed + 100).uniform(-1.0, 1.0, (n, k))


def gcn_values_host(rowptr: np.ndarray, colind: np.ndarray) -> np.ndarray:
    """A_hat = D^-1/2 A D^-1/2 with D the row lengths (clamped to 1), fp32."""
    deg = np.maximum(np.diff(rowptr), 1).astype(np.float64)
    rows = np.repeat(np.arange(rowptr.size - 1), np.diff(rowptr))
    return (1.0 / np.sqrt(deg[rows] * deg[colind])).astype(np.float32)


def gcn_features(n: int, f: int, seed: int):
    """Config 4's X [n, f] U(0, 1) fp32 and W [f, f] U(-1/8, 1/8) fp32
    (torch Linear's default bound for fan-in 64), default_rng(seed + 100)."""
    g = np.random.default_rng(seed + 100)
    X = g.random((n, f), dtype=np.float32)
    W = ((g.random((f, f)) * 2.0 - 1.0) / 8.0).astype(np.float32)
    return X, W


def dense_operands(n: int, dtype, seed: int):
    """Config 2's A, B [n, n]: f32 U(0, 1) seed 3, f64 U(-1, 1) seed 2."""
    g = np.random.default_rng(seed)
    lo = 0.0 if dtype == np.float32 else -1.0
    A = g.uniform(lo, 1.0, (n, n)).astype(dtype)
    B = g.uniform(lo, 1.0, (n, n)).astype(dtype)
    return A, B
