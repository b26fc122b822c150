"""Host logic of the row-block-sharded SpMV (paper_2509_25605_b200/sharded.py)
on 2 and 3 CPU processes over gloo: the exchange plan moves exactly the needed
x slabs, the assembled x window equals the global x on every referenced
column, and per-shard products (checked with the oracle) reassemble the
global y bit for bit."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_25605_b200 import sharded


def _worker(rank, world, port, points, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(__file__))
        from matrices import stencil_csr
        from oracle import oracle as O
        rowptr, colind, values = stencil_csr(points, n)
        N = rowptr.size - 1
        ranges = sharded.balanced_row_ranges(N, world)
        r0, r1 = ranges[rank]
        lrp = torch.from_numpy(rowptr[r0:r1 + 1] - rowptr[r0])
        lci = torch.from_numpy(colind[rowptr[r0]:rowptr[r1]].astype(np.int64))
        plan = sharded.build_exchange_plan(lci, ranges, rank, world)
        x = np.random.default_rng(5).uniform(-1, 1, N)
        x_full = torch.full((N,), float("nan"), dtype=torch.float64)
        x_full[r0:r1] = torch.from_numpy(x[r0:r1])
        reqs = sharded.exchange(plan, x_full)
        for r in reqs:
            r.wait()
        used = np.unique(lci.numpy())
        assert np.array_equal(x_full.numpy()[used], x[used])
        a, b = sharded.interior_run(lrp, lci, (r0, r1))
        y = O.spmv_csr(lrp.numpy(), lci.numpy(), values[rowptr[r0]:rowptr[r1]], x_full.numpy())
        q.put((rank, plan.needs, plan.sends, (a, b), y.tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,points,n", [(2, 5, 30), (3, 27, 9), (2, 27, 7)])
def test_sharded_exchange_and_reassembly(world, points, n):
    from matrices import stencil_csr
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + world * 10 + points + n
    procs = [ctx.Process(target=_worker, args=(r, world, port, points, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    rowptr, colind, values = stencil_csr(points, n)
    N = rowptr.size - 1
    x = np.random.default_rng(5).uniform(-1, 1, N)
    want = O.spmv_csr(rowptr, colind, values, x)
    got = np.concatenate([np.frombuffer(r[4], dtype=np.float64) for r in res])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    halo = n * n + n + 1 if points == 27 else n
    ranges = sharded.balanced_row_ranges(N, world)
    for rank, needs, sends, (a, b), _ in res:
        # sends of p to q == needs of q from p
        for p in range(world):
            if p != rank:
                assert tuple(res[p][1][rank]) == tuple(sends[p])
        # neighbours exchange at most the stencil halo
        for p, (lo, hi) in enumerate(needs):
            if p != rank:
                assert hi - lo <= halo
        r0, r1 = ranges[rank]
        assert 0 <= a <= b <= r1 - r0
        assert (b - a) >= (r1 - r0) - 2 * halo


def _spmm_worker(rank, world, port, nrows, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(__file__))
        from matrices import powerlaw_csr
        from oracle import oracle as O
        rowptr, colind, values = powerlaw_csr(np.random.default_rng(7), nrows, mean=6.0)
        X = np.random.default_rng(8).uniform(-1, 1, (nrows, k))
        ranges = sharded.equal_row_ranges(nrows, world)
        r0, r1 = ranges[rank]
        lrp = torch.from_numpy(rowptr[r0:r1 + 1] - rowptr[r0])
        lci = torch.from_numpy(colind[rowptr[r0]:rowptr[r1]])
        lv = torch.from_numpy(values[rowptr[r0]:rowptr[r1]])
        op = sharded.RowBlockSpmm(lrp, lci, lv, nrows, k, rank, world)
        assert (op.row_begin, op.row_end) == (r0, r1)
        op.x_local.copy_(torch.from_numpy(X[r0:r1]))
        op.gather()
        # every rank now holds all of X at its global row indices
        assert np.array_equal(op.X_full[:nrows].numpy(), X)
        Y = O.spmm_csr(lrp.numpy(), lci.numpy(), lv.numpy(), op.X_full[:nrows].numpy())
        q.put((rank, Y.tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nrows", [(2, 301), (3, 250)])
def test_sharded_spmm_allgather_reassembly(world, nrows):
    from matrices import powerlaw_csr
    from oracle import oracle as O
    k = 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + world * 10 + nrows % 7
    procs = [ctx.Process(target=_spmm_worker, args=(r, world, port, nrows, k, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rowptr, colind, values = powerlaw_csr(np.random.default_rng(7), nrows, mean=6.0)
    X = np.random.default_rng(8).uniform(-1, 1, (nrows, k))
    want = O.spmm_csr(rowptr, colind, values, X)
    got = np.concatenate([np.frombuffer(r[1], dtype=np.float64).reshape(-1, k) for r in res])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
