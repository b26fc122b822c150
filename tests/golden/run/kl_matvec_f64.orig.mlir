func.func @matvec(%0: memref<64x64xf64>, %1: memref<64xf64>) -> (memref<64xf64>) {
  %2 = memref.alloc : memref<64xf64>
  linalg.matvec(%0, %1, %2)
  func.return(%2)
}
