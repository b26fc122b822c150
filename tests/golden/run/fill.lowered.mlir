func.func @fillit() -> (memref<8x8xf64, dualview>) {
  %0 = memref.alloc : memref<8x8xf64, dualview>
  %1 = arith.constant 3.5 : f64
  %2 = arith.constant 8 : index
  %3 = arith.constant 8 : index
  %4 = arith.constant 0 : index
  %5 = arith.constant 1 : index
  kokkos.range_parallel (%6, %7) in (%2, %3) {executionSpace = device, parallelLevel = topmdrange} {
    memref.store %1, %0[%6, %7]
    kokkos.yield
  }
  kokkos.modify(%0) {space = device}
  func.return(%0)
}
