func.func @f(%0: memref<4xf64, dualview>, %1: memref<4xf64, dualview>) -> (memref<4xf64, dualview>) {
  %2 = arith.constant 0 : index
  %3 = arith.constant 4 : index
  %4 = arith.constant 9.0 : f64
  kokkos.sync(%0) {space = device}
  memref.store %4, %0[%2]
  kokkos.modify(%0) {space = host}
  kokkos.range_parallel (%5) in (%3) {executionSpace = device, parallelLevel = toprange} {
    %6 = memref.load %0[%5]
    memref.store %6, %1[%5]
    kokkos.yield
  }
  kokkos.modify(%1) {space = device}
  func.return(%1)
}
