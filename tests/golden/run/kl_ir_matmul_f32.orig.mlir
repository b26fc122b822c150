func.func @matmul(%0: memref<?x?xf32>, %1: memref<?x?xf32>, %2: memref<?x?xf32>) -> (memref<?x?xf32>) {
  linalg.matmul(%0, %1, %2)
  func.return(%2)
}
