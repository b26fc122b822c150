// CSR SpMV with int64 row pointers and int32 column indices (the layout the
// B200 kernels stream).  Same op as the reference fixture
// tests/fixtures/spmv.mlir; dialect.py:797-812 admits i32 colind and
// spmv_lowering.py:15-18 inserts the index_cast.
func @spmv(%rowptr: memref<?xindex>, %colind: memref<?xi32>, %values: memref<?xf64>,
           %x: memref<?xf64>, %y: memref<?xf64>) -> (memref<?xf64>) {
  sparse.spmv_csr(%rowptr, %colind, %values, %x, %y)
  func.return(%y)
}
