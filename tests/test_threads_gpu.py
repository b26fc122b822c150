"""Concurrent callers (SURVEY 8(b) threading): several host threads, each on
its own CUDA stream, call the C ABI at the same time — SpMV through a shared
plan and without one, SpMM, GEMM, GCN — and every result is bit-identical to
the same call made alone.  Per-call workspaces are stream-ordered
(cudaMallocAsync), plans are read-only after creation, error state is
thread-local."""
import threading

import numpy as np
import pytest
import torch

import paper_2509_25605_b200 as lb
from conftest import bits_equal
from matrices import powerlaw_csr, stencil_csr

pytestmark = pytest.mark.gpu


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _run_threads(fns, reps=4):
    errors, outs = [], [None] * len(fns)

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(reps):
                    r = fns[i](s)
                s.synchronize()
            outs[i] = r.cpu()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    return outs


def test_concurrent_calls_match_serial(cuda_device):
    rng = np.random.default_rng(11)
    rp5, ci5, v5 = stencil_csr(27, 30)
    x5 = rng.uniform(-1, 1, rp5.size - 1)
    rpp, cip, vpp = powerlaw_csr(rng, 50_000, mean=12.0)
    xp = rng.uniform(-1, 1, 50_000)
    X = rng.uniform(-1, 1, (50_000, 64))
    A = rng.uniform(0, 1, (384, 512)).astype(np.float32)
    B = rng.uniform(0, 1, (512, 256)).astype(np.float32)
    W = rng.uniform(-1, 1, (64, 64)).astype(np.float32)
    d = {k: cu(v) for k, v in dict(rp5=rp5, ci5=ci5, v5=v5, x5=x5, rpp=rpp, cip=cip, vpp=vpp, xp=xp,
                                     X=X, A=A, B=B, W=W, Xf=X.astype(np.float32),
                                     vpf=vpp.astype(np.float32)).items()}
    plan = lb.CsrPlan(d["rp5"], exact=True)
    fns = [
        lambda s: plan.spmv(d["ci5"], d["v5"], d["x5"], stream=s),
        lambda s: lb.spmv_csr(d["rpp"], d["cip"], d["vpp"], d["xp"], stream=s),
        lambda s: lb.spmm_csr(d["rpp"], d["cip"], d["vpp"], d["X"], stream=s),
        lambda s: lb.gemm(d["A"], d["B"], stream=s),
        lambda s: lb.gcn_layer(d["rpp"], d["cip"], d["vpf"], d["Xf"], d["W"], stream=s),
        lambda s: plan.spmv(d["ci5"], d["v5"], d["x5"], stream=s),
    ]
    serial = []
    for f in fns:
        r = f(torch.cuda.current_stream())
        torch.cuda.synchronize()
        serial.append(r.cpu())
    for _ in range(3):
        outs = _run_threads(fns)
        for i, (a, b) in enumerate(zip(outs, serial)):
            assert bits_equal(a.numpy(), b.numpy()), i


def test_errors_are_thread_local(cuda_device):
    # a failing call on one thread leaves another thread's error state alone
    msgs = {}

    def bad():
        for _ in range(50):
            try:  # rejected inside the C ABI (vector length not a power of two)
                lb.spmv_csr(cu(np.array([0, 1], np.int64)), cu(np.array([0], np.int32)),
                            cu(np.array([2.0])), cu(np.array([3.0])), vector_length=3)
            except lb.BackendError as e:
                msgs["bad"] = str(e)

    def good():
        for _ in range(50):
            y = lb.spmv_csr(cu(np.array([0, 1], np.int64)), cu(np.array([0], np.int32)),
                            cu(np.array([2.0])), cu(np.array([3.0])))
            msgs["good"] = float(y.item())

    ts = [threading.Thread(target=bad), threading.Thread(target=good)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert "vector_length" in msgs["bad"] and msgs["good"] == 6.0
