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


def _gemm_worker(rank, world, port, m, k, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        A = np.random.default_rng(2).uniform(-1, 1, (m, k))
        Bfull = np.random.default_rng(3).uniform(-1, 1, (k, n))
        r0, r1 = sharded.equal_row_ranges(m, world)[rank]
        # only rank 0 holds B: the operator broadcasts it once
        B = torch.from_numpy(Bfull.copy()) if rank == 0 else torch.full((k, n), float("nan"),
                                                                         dtype=torch.float64)
        op = sharded.RowBlockGemm(torch.from_numpy(A[r0:r1].copy()), B, m, rank, world)
        assert np.array_equal(op.B.numpy(), Bfull)
        assert (op.row_begin, op.row_end) == (r0, r1)
        C_local = torch.from_numpy(O.matmul(op.A_local.numpy(), op.B.numpy()))
        full = op.gather_c(C_local)
        q.put((rank, full.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m", [(2, 37), (3, 64)])
def test_sharded_gemm_broadcast_and_reassembly(world, m):
    from oracle import oracle as O
    k, n = 24, 16
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + world * 10 + m % 7
    procs = [ctx.Process(target=_gemm_worker, args=(r, world, port, m, k, n, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = np.random.default_rng(2).uniform(-1, 1, (m, k))
    B = np.random.default_rng(3).uniform(-1, 1, (k, n))
    want = O.matmul(A, B)
    for _, buf in res:   # every rank holds the whole C after gather_c
        got = np.frombuffer(buf, dtype=np.float64).reshape(m, n)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def _gcn_worker(rank, world, port, nrows, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(__file__)))
        import synth_inputs as S
        from oracle import oracle as O
        spec = S.PowerLawSpec(nrows, mean=6.0, seed=4)
        rowptr, colind = S.powerlaw_structure_host(spec)
        values = S.gcn_values_host(rowptr, colind)
        X, Wf = S.gcn_features(nrows, 16, 4)
        r0, r1 = sharded.equal_row_ranges(nrows, world)[rank]
        lrp = torch.from_numpy(rowptr[r0:r1 + 1] - rowptr[r0])
        lci = torch.from_numpy(colind[rowptr[r0]:rowptr[r1]])
        lv = torch.from_numpy(values[rowptr[r0]:rowptr[r1]])
        W = torch.from_numpy(Wf.copy()) if rank == 0 else torch.zeros((16, 16), dtype=torch.float32)
        op = sharded.RowBlockGcn(lrp, lci, lv, W, nrows, rank, world)
        op.x_local.copy_(torch.from_numpy(X[r0:r1]))
        op.gather()
        assert np.array_equal(op.spmm.X_full[:nrows].numpy(), X)
        assert np.array_equal(op.W.numpy(), Wf)
        H = O.gcn(lrp.numpy(), lci.numpy(), lv.numpy(), op.spmm.X_full[:nrows].numpy(),
                  op.W.numpy())
        q.put((rank, H.tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nrows", [(2, 301), (3, 250)])
def test_sharded_gcn_reassembly(world, nrows):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(__file__)))
    import synth_inputs as S
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29900 + world * 10 + nrows % 7
    procs = [ctx.Process(target=_gcn_worker, args=(r, world, port, nrows, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = S.PowerLawSpec(nrows, mean=6.0, seed=4)
    rowptr, colind = S.powerlaw_structure_host(spec)
    values = S.gcn_values_host(rowptr, colind)
    X, W = S.gcn_features(nrows, 16, 4)
    want = O.gcn(rowptr, colind, values, X, W)
    got = np.concatenate([np.frombuffer(r[1], dtype=np.float32).reshape(-1, 16) for r in res])
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
