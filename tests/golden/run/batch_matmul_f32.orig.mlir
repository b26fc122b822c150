func.func @bmm(%0: memref<4x8x8xf32>, %1: memref<4x8x8xf32>) -> (memref<4x8x8xf32>) {
  %2 = memref.alloc : memref<4x8x8xf32>
  linalg.batch_matmul(%0, %1, %2)
  func.return(%2)
}
