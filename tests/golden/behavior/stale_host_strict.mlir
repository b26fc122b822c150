func.func @f(%0: memref<4xf64, dualview>) -> (memref<4xf64, dualview>) {
  %1 = arith.constant 0 : index
  %2 = arith.constant 1 : index
  %3 = arith.constant 4 : index
  %4 = arith.constant 2.0 : f64
  kokkos.sync(%0) {space = device}
  kokkos.range_parallel (%5) in (%3) {executionSpace = device, parallelLevel = toprange} {
    %6 = memref.load %0[%5]
    %7 = arith.mulf(%6, %4)
    memref.store %7, %0[%5]
    kokkos.yield
  }
  kokkos.modify(%0) {space = device}
  %8 = memref.load %0[%1]
  memref.store %8, %0[%2]
  func.return(%0)
}
