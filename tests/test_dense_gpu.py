"""Parity of the dense kernels (matmul, matvec, batch_matmul, parallel_reduce,
ReLU) with the reference fixtures; the EXACT mode and the row-sequential
kernels follow the reference order and must be bit-identical."""
import numpy as np
import pytest
import torch

import paper_2509_25605_b200 as lb
from conftest import bits_equal, golden_names, load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("name", ["matmul_i32", "matmul_f64", "matmul_f64_kl", "matmul_dyn_f32",
                                  "matmul_dyn_f64"])
def test_golden_matmul_exact_mode(cuda_device, name):
    g = load_golden(name)
    A, B = g["inputs"][:2]
    assert bits_equal(host(lb.gemm(cu(A), cu(B), mode="exact")), g["outputs"][0])


@pytest.mark.parametrize("name", ["matmul_f64", "matmul_dyn_f32", "matmul_dyn_f64", "matmul_i32"])
def test_golden_matmul_auto_mode(cuda_device, name):
    g = load_golden(name)
    A, B = g["inputs"][:2]
    got = host(lb.gemm(cu(A), cu(B)))
    want = g["outputs"][0]
    tol = {np.dtype(np.float64): 1e-12, np.dtype(np.float32): 1e-5}.get(want.dtype, 0)
    ok, msg = O.diff_outputs([got], [want], tol)
    assert ok, msg


@pytest.mark.parametrize("name", ["matvec_f64", "matvec_f64_kl", "matvec_dyn"])
def test_golden_matvec_bitexact(cuda_device, name):
    g = load_golden(name)
    A, x = g["inputs"][:2]
    assert bits_equal(host(lb.gemv(cu(A), cu(x))), g["outputs"][0])


def test_golden_batch_matmul_bitexact(cuda_device):
    g = load_golden("batch_matmul_f32")
    A, B = g["inputs"]
    assert bits_equal(host(lb.batch_gemm(cu(A), cu(B), mode="exact")), g["outputs"][0])


@pytest.mark.parametrize("name", golden_names("reduce_"))
def test_golden_reduce_bitexact(cuda_device, name):
    g = load_golden(name)
    if name == "reduce_add_f64":
        comb, axis = "add", 1
    else:
        _, comb, ax, _ = name.split("_")
        axis = int(ax[2:])
    assert bits_equal(host(lb.reduce2d(cu(g["inputs"][0]), axis, comb)), g["outputs"][0])


def test_relu_select_semantics(cuda_device):
    x = np.array([1.5, -2.0, 0.0, -0.0, np.nan, np.inf, -np.inf, 3e-310])
    assert bits_equal(host(lb.relu(cu(x))), O.relu(x))
    assert bits_equal(host(lb.relu(cu(x.astype(np.float32)))), O.relu(x.astype(np.float32)))


@pytest.mark.parametrize("m,n,k", [(129, 65, 257), (1, 300, 5), (64, 64, 64)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32, np.int32, np.int64])
def test_exact_gemm_random_shapes(cuda_device, m, n, k, dtype):
    rng = np.random.default_rng(m * n + k)
    if np.issubdtype(dtype, np.integer):
        A = rng.integers(-2**20, 2**20, (m, k)).astype(dtype)
        B = rng.integers(-2**20, 2**20, (k, n)).astype(dtype)
    else:
        A = rng.uniform(-1, 1, (m, k)).astype(dtype)
        B = rng.uniform(-1, 1, (k, n)).astype(dtype)
    assert bits_equal(host(lb.gemm(cu(A), cu(B), mode="exact")), O.matmul(A, B))


def test_gemv_large_bitexact(cuda_device):
    rng = np.random.default_rng(2)
    A = rng.uniform(-1, 1, (3001, 777))
    x = rng.uniform(-1, 1, 777)
    assert bits_equal(host(lb.gemv(cu(A), cu(x))), O.matvec(A, x))


@pytest.mark.parametrize("m,n,k", [(128, 256, 32), (129, 65, 257), (1, 300, 5), (300, 257, 1000),
                                   (1024, 1024, 1024), (45, 70, 130), (7, 9, 3)])
def test_tf32x3_gemm_fp32_contract(cuda_device, m, n, k):
    # tcgen05 3xTF32 path: within the fp32 contract (1e-5, diff_outputs) on U(0,1)
    rng = np.random.default_rng(m + 7 * n + 13 * k)
    A = rng.uniform(0, 1, (m, k)).astype(np.float32)
    B = rng.uniform(0, 1, (k, n)).astype(np.float32)
    got = host(lb.gemm(cu(A), cu(B), mode="tf32x3"))
    ok, msg = O.diff_outputs([got], [O.matmul(A, B)], 1e-5)
    assert ok, msg


def test_tf32x3_batched(cuda_device):
    rng = np.random.default_rng(1)
    A = rng.uniform(0, 1, (3, 70, 90)).astype(np.float32)
    B = rng.uniform(0, 1, (3, 90, 300)).astype(np.float32)
    got = host(lb.batch_gemm(cu(A), cu(B), mode="tf32x3"))
    ok, msg = O.diff_outputs([got], [O.batch_matmul(A, B)], 1e-5)
    assert ok, msg


@pytest.mark.parametrize("m,n,k", [(128, 128, 16), (130, 66, 258), (1000, 600, 512), (32, 32, 32),
                                   (2, 2, 2), (257, 129, 33), (64, 4, 1024)])
def test_dmma_gemm_fp64_contract(cuda_device, m, n, k):
    # DMMA path (odd extents fall back to the exact kernel): within the 1e-12 contract
    rng = np.random.default_rng(m * 3 + n * 5 + k)
    A = rng.uniform(-1, 1, (m, k))
    B = rng.uniform(-1, 1, (k, n))
    got = host(lb.gemm(cu(A), cu(B), mode="dmma"))
    ok, msg = O.diff_outputs([got], [O.matmul(A, B)], 1e-12)
    assert ok, msg


@pytest.mark.parametrize("dt,tol,lo", [(np.float64, 1e-12, -1.0), (np.float32, 1e-5, 0.0)])
@pytest.mark.parametrize("m,n,k", [(96, 80, 160), (200, 300, 517), (257, 129, 1000), (512, 512, 4096)])
def test_ozaki_int8_within_tolerance(cuda_device, dt, tol, lo, m, n, k):
    """Ozaki digit split on the int8 tensor cores vs the reference-order
    sequential sum (oracle), the reference's parity criterion."""
    rng = np.random.default_rng(m + n + k)
    A = rng.uniform(lo, 1, (m, k)).astype(dt)
    B = rng.uniform(lo, 1, (k, n)).astype(dt)
    got = host(lb.gemm(cu(A), cu(B), mode="ozaki"))
    ok, msg = O.diff_outputs([got], [O.matmul(A, B)], tol)
    assert ok, msg


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_ozaki_scaled_rows_and_zeros(cuda_device, dt):
    """Rows / columns of very different magnitude (per-row / per-column
    exponents), an all-zero row and column."""
    rng = np.random.default_rng(7)
    lo = -1.0 if dt == np.float64 else 0.0   # fp32: U(0,1)
    A = rng.uniform(lo, 1, (64, 300)).astype(dt) * np.logspace(-20, 20, 64)[:, None].astype(dt)
    B = rng.uniform(lo, 1, (300, 48)).astype(dt) * np.logspace(-10, 10, 48)[None, :].astype(dt)
    A[5] = 0
    B[:, 7] = 0
    got = host(lb.gemm(cu(A), cu(B), mode="ozaki"))
    ok, msg = O.diff_outputs([got], [O.matmul(A, B)], 1e-12 if dt == np.float64 else 1e-5)
    assert ok, msg


@pytest.mark.parametrize("bad", [np.inf, -np.inf, np.nan])
def test_ozaki_non_finite_falls_back_to_reference_order(cuda_device, bad):
    rng = np.random.default_rng(3)
    A = rng.uniform(-1, 1, (40, 64))
    B = rng.uniform(-1, 1, (64, 24))
    A[3, 5] = bad
    got = host(lb.gemm(cu(A), cu(B), mode="ozaki"))
    assert bits_equal(got, O.matmul(A, B))


@pytest.mark.parametrize("dt,lo", [(np.float64, -1.0), (np.float32, 0.0)])
def test_ozaki_certification_falls_back(cuda_device, dt, lo):
    """A row whose largest element dwarfs the rest while the product
    cancels it: the a-priori bound cannot certify the contract, so the
    certified fallback (fp64 DMMA / fp32 3xTF32) produces C."""
    rng = np.random.default_rng(11)
    A = rng.uniform(lo, 1, (48, 512)).astype(dt)
    B = rng.uniform(lo, 1, (512, 40)).astype(dt)
    A[:, 0] = 1e10
    B[0, :] = 0.0
    got = host(lb.gemm(cu(A), cu(B), mode="ozaki"))
    ok, msg = O.diff_outputs([got], [O.matmul(A, B)], 1e-12 if dt == np.float64 else 1e-5)
    assert ok, msg


@pytest.mark.parametrize("m,n,dtype", [(1000, 1537, np.float64), (333, 4096, np.float32),
                                       (70, 4100, np.float64), (65, 3, np.float32),
                                       (129, 2050, np.int64), (40, 999, np.int32)])
def test_gemv_pipelined_fold_bitexact(cuda_device, m, n, dtype):
    # both copy paths of row_fold_pipe_kernel (16-byte when the row pitch and n
    # allow, element-wise otherwise), partial row blocks and column panels
    rng = np.random.default_rng(m + n)
    if np.issubdtype(dtype, np.integer):
        A = rng.integers(-2**30, 2**30, (m, n)).astype(dtype)   # wraps
        x = rng.integers(-9, 9, n).astype(dtype)
    else:
        A = rng.uniform(-1, 1, (m, n)).astype(dtype)
        x = rng.uniform(-1, 1, n).astype(dtype)
    assert bits_equal(host(lb.gemv(cu(A), cu(x))), O.matvec(A, x))


@pytest.mark.parametrize("comb", ["add", "mul", "min", "max"])
@pytest.mark.parametrize("dtype", [np.float64, np.int64, np.float32])
def test_reduce_rows_pipelined_bitexact(cuda_device, comb, dtype):
    rng = np.random.default_rng(3)
    src = (rng.integers(-5, 6, (300, 517)) if np.issubdtype(dtype, np.integer)
           else rng.uniform(0.5, 1.5, (300, 517))).astype(dtype)
    assert bits_equal(host(lb.reduce2d(cu(src), 1, comb)), O.reduce2d(src, 1, comb))


@pytest.mark.parametrize("m,n,k", [(256, 200, 300), (384, 130, 517), (1024, 512, 2048)])
def test_auto_f32_sign_gate(cuda_device, m, n, k):
    """AUTO f32: non-negative operands take the certified Ozaki path (even and
    odd row-block counts: 2-CTA clusters or single CTAs), operands with a
    negative entry the 3xTF32 path; both within the 1e-5 contract."""
    rng = np.random.default_rng(m * 7 + k)
    A = rng.uniform(0, 1, (m, k)).astype(np.float32)
    B = rng.uniform(0, 1, (k, n)).astype(np.float32)
    ok, msg = O.diff_outputs([host(lb.gemm(cu(A), cu(B)))], [O.matmul(A, B)], 1e-5)
    assert ok, msg
    A[m // 2, k // 3] = -0.25   # one negative entry trips the gate
    ok, msg = O.diff_outputs([host(lb.gemm(cu(A), cu(B)))], [O.matmul(A, B)], 1e-5)
    assert ok, msg
    B2 = B.copy()
    B2[k - 1, n - 1] = -1.0
    ok, msg = O.diff_outputs([host(lb.gemm(cu(np.abs(A)), cu(B2)))], [O.matmul(np.abs(A), B2)], 1e-5)
    assert ok, msg


def test_auto_f32_non_finite_reference_order(cuda_device):
    rng = np.random.default_rng(4)
    A = rng.uniform(0, 1, (130, 96)).astype(np.float32)
    B = rng.uniform(0, 1, (96, 70)).astype(np.float32)
    A[7, 9] = np.inf
    assert bits_equal(host(lb.gemm(cu(A), cu(B))), O.matmul(A, B))


@pytest.mark.parametrize("dt,lo,tol", [(np.float32, 0.0, 1e-5), (np.float64, -1.0, 1e-12)])
def test_auto_batched_ozaki(cuda_device, dt, lo, tol):
    """batch_gemm in AUTO mode through the Ozaki paths (per-batch splits, the
    cluster kernels on an even row-block count)."""
    rng = np.random.default_rng(17)
    A = rng.uniform(lo, 1, (3, 256, 192)).astype(dt)
    B = rng.uniform(lo, 1, (3, 192, 160)).astype(dt)
    got = host(lb.batch_gemm(cu(A), cu(B)))
    for b in range(3):
        ok, msg = O.diff_outputs([got[b]], [O.matmul(A[b], B[b])], tol)
        assert ok, (b, msg)
