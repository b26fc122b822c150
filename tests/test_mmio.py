"""Matrix Market reader (native, host-side) against scipy.io.mmread on
general / symmetric / skew-symmetric / pattern / integer files, blank and
comment lines, empty rows; malformed files raise."""
import numpy as np
import pytest

from paper_2509_25605_b200 import mmio
from paper_2509_25605_b200._capi import BackendError

scipy_io = pytest.importorskip("scipy.io")
sparse = pytest.importorskip("scipy.sparse")


def _write(tmp_path, name, A, field="real", symmetry="general"):
    p = tmp_path / name
    scipy_io.mmwrite(str(p), A, field=field, symmetry=symmetry)
    return p if p.suffix == ".mtx" else p.with_suffix(".mtx")


def _check(path, index_dtype=np.int32):
    rowptr, colind, values, shape = mmio.read_matrix_market(path, index_dtype=index_dtype)
    want = sparse.csr_matrix(scipy_io.mmread(str(path)))
    want.sort_indices()
    assert shape == want.shape
    assert np.array_equal(rowptr, want.indptr.astype(np.int64))
    assert np.array_equal(colind, want.indices.astype(index_dtype))
    assert np.array_equal(values, want.data.astype(np.float64))


@pytest.mark.parametrize("index_dtype", [np.int32, np.int64])
def test_general_real(tmp_path, index_dtype):
    rng = np.random.default_rng(0)
    A = sparse.random(300, 200, density=0.03, random_state=1, format="coo")
    A.data = rng.uniform(-1, 1, A.nnz)
    _check(_write(tmp_path, "g.mtx", A), index_dtype)


@pytest.mark.parametrize("symmetry", ["symmetric", "skew-symmetric"])
def test_symmetric_storage_expanded(tmp_path, symmetry):
    B = sparse.random(150, 150, density=0.05, random_state=2, format="csr")
    A = (B - B.T) if symmetry == "skew-symmetric" else (B + B.T)
    A = sparse.coo_matrix(A)
    _check(_write(tmp_path, "s.mtx", A, symmetry=symmetry))


def test_pattern_and_integer(tmp_path):
    A = sparse.random(80, 90, density=0.1, random_state=3, format="coo")
    A.data = np.round(A.data * 100)
    _check(_write(tmp_path, "i.mtx", A, field="integer"))
    p = tmp_path / "p.mtx"
    rows, cols = A.row + 1, A.col + 1
    p.write_text("%%MatrixMarket matrix coordinate pattern general\n% comment\n\n"
                 f"80 90 {A.nnz}\n" + "".join(f"{r} {c}\n" for r, c in zip(rows, cols)))
    rowptr, colind, values, _ = mmio.read_matrix_market(p)
    want = sparse.csr_matrix((np.ones(A.nnz), (A.row, A.col)), shape=(80, 90))
    want.sort_indices()
    assert np.array_equal(rowptr, want.indptr) and np.array_equal(colind, want.indices)
    assert np.all(values == 1.0)


def test_empty_rows_and_info(tmp_path):
    p = tmp_path / "e.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n5 4 3\n1 1 2.5\n4 2 -1\n4 1 3e-3\n")
    info = mmio.matrix_market_info(p)
    assert info == {"nrows": 5, "ncols": 4, "nnz": 3, "field": "real", "symmetry": "general"}
    rowptr, colind, values, _ = mmio.read_matrix_market(p)
    assert rowptr.tolist() == [0, 1, 1, 1, 3, 3]
    assert colind.tolist() == [0, 0, 1] and values.tolist() == [2.5, 3e-3, -1.0]


@pytest.mark.parametrize("text", [
    "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "not a matrix market file\n",
])
def test_malformed_files_raise(tmp_path, text):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(BackendError):
        mmio.read_matrix_market(p)
