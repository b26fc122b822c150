"""The reference's own emitted C++ on its serial stub (oracle/_ref, built by
oracle/build.py) agrees bit for bit with the reference interpreter fixtures and
with the C oracle; the row-block thread split used for the all-cores CPU
baseline leaves every output bit unchanged."""
import numpy as np
import pytest

from conftest import bits_equal, load_golden
from oracle import oracle as O
from oracle import ref as R

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("name", ["spmv4", "spmv_random100_s31", "spmv_ragged400",
                                  "spmv_mean1434", "spmv_allempty", "spmv_identity"])
def test_emitted_spmv_matches_interpreter(name):
    g = load_golden(name)
    rowptr, colind, values, x, _ = g["inputs"]
    y, _ = R.spmv_csr(rowptr, colind, values, x)
    assert bits_equal(y, g["outputs"][0])
    y32, _ = R.spmv_csr(rowptr, colind.astype(np.int32), values, x)
    assert bits_equal(y32, g["outputs"][0])


def test_transfer_counters_match_interpreter_trace():
    # compile_smoke.test.ts:81-142: driver counters == `lapis run --trace`
    g = load_golden("spmv4")
    h2d = [e for e in g["trace"] if e.startswith("H2D")]
    d2h = [e for e in g["trace"] if e.startswith("D2H")]
    hb = sum(int(e.split("bytes=")[1]) for e in h2d)
    db = sum(int(e.split("bytes=")[1]) for e in d2h)
    assert R.spmv_transfer_probe() == (len(h2d), len(d2h), hb, db) == (4, 1, 152, 32)


def test_thread_split_is_bitwise_identical():
    rng = np.random.default_rng(9)
    n = 3000
    counts = rng.integers(0, 40, n)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum(counts)
    colind = rng.integers(0, n, rowptr[-1]).astype(np.int32)
    values = rng.uniform(-1, 1, rowptr[-1])
    x = rng.uniform(-1, 1, n)
    y1, _ = R.spmv_csr(rowptr, colind, values, x, threads=1)
    y4, _ = R.spmv_csr(rowptr, colind, values, x, reps=2, threads=4)
    assert bits_equal(y1, y4)
    assert bits_equal(y1, O.spmv_csr(rowptr, colind, values, x))


def test_emitted_spmm_and_gcn_match_interpreter():
    g = load_golden("spmm_k8")
    rowptr, colind, values, X, _ = g["inputs"]
    Y, _ = R.spmm_csr(rowptr, colind, values, X, threads=3)
    assert bits_equal(Y, g["outputs"][0])
    g = load_golden("gcn_small")
    rowptr, colind, values, X, W, _ = g["inputs"]
    H, _ = R.gcn(rowptr, colind, values, X, W, threads=2)
    assert bits_equal(H, g["outputs"][0])


def test_emitted_dense_match_interpreter():
    for name in ("matmul_dyn_f32", "matmul_dyn_f64"):
        g = load_golden(name)
        A, B = g["inputs"][:2]
        Cm, _ = R.matmul(A, B, threads=2)
        assert bits_equal(Cm, g["outputs"][0])
    g = load_golden("matvec_dyn")
    y, _ = R.matvec(*g["inputs"][:2])
    assert bits_equal(y, g["outputs"][0])


def test_spmm_gcn_relabelled_blocks_bitwise():
    """The driver hands each thread block only the X rows it references
    (relabelled columns): outputs stay bitwise equal to the oracle at any
    thread count."""
    import synth_inputs as S
    spec = S.PowerLawSpec(4000, mean=8.0, seed=9)
    rowptr, colind = S.powerlaw_structure_host(spec)
    values = S.powerlaw_values(spec, int(rowptr[-1]))
    X = np.random.default_rng(1).uniform(-1, 1, (4000, 16))
    want = O.spmm_csr(rowptr, colind, values, X)
    for t in (1, 5, 16):
        Y, _ = R.spmm_csr(rowptr, colind, values, X, threads=t)
        assert np.array_equal(Y.view(np.uint64), want.view(np.uint64)), t
    vf = S.gcn_values_host(rowptr, colind)
    Xf, Wf = S.gcn_features(4000, 16, 4)
    wantH = O.gcn(rowptr, colind, vf, Xf, Wf)
    for t in (1, 7):
        H, _ = R.gcn(rowptr, colind, vf, Xf, Wf, threads=t)
        assert np.array_equal(H.view(np.uint32), wantH.view(np.uint32)), t
