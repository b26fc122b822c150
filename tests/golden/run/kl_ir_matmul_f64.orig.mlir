func.func @matmul(%0: memref<?x?xf64>, %1: memref<?x?xf64>, %2: memref<?x?xf64>) -> (memref<?x?xf64>) {
  linalg.matmul(%0, %1, %2)
  func.return(%2)
}
