func.func @matvec(%0: memref<?x?xf64>, %1: memref<?xf64>, %2: memref<?xf64>) -> (memref<?xf64>) {
  linalg.matvec(%0, %1, %2)
  func.return(%2)
}
