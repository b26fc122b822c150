func.func @fillit() -> (memref<8x8xf64>) {
  %0 = memref.alloc : memref<8x8xf64>
  %1 = arith.constant 3.5 : f64
  linalg.fill(%1, %0)
  func.return(%0)
}
