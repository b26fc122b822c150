func.func @matmul(%0: memref<32x32xf64>, %1: memref<32x32xf64>) -> (memref<32x32xf64>) {
  %2 = memref.alloc : memref<32x32xf64>
  linalg.matmul(%0, %1, %2)
  func.return(%2)
}
