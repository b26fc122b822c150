func.func @f(%0: memref<4xf64, dualview>) -> (f64) {
  %1 = arith.constant 0 : index
  %2 = arith.constant 4 : index
  %3 = memref.alloc : memref<4xf64, device>
  kokkos.sync(%0) {space = device}
  kokkos.range_parallel (%4) in (%2) {executionSpace = device, parallelLevel = toprange} {
    %5 = memref.load %0[%4]
    memref.store %5, %3[%4]
    kokkos.yield
  }
  %6 = memref.load %3[%1]
  func.return(%6)
}
