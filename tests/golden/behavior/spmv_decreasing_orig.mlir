func.func @spmv(%0: memref<?xindex>, %1: memref<?xindex>, %2: memref<?xf64>, %3: memref<?xf64>, %4: memref<?xf64>) -> (memref<?xf64>) {
  sparse.spmv_csr(%0, %1, %2, %3, %4)
  func.return(%4)
}
