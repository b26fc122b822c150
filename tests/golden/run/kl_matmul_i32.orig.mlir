func.func @matmul(%0: memref<16x16xi32>, %1: memref<16x16xi32>) -> (memref<16x16xi32>) {
  %2 = memref.alloc : memref<16x16xi32>
  linalg.matmul(%0, %1, %2)
  func.return(%2)
}
