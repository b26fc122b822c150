func.func @f(%0: memref<8xf64, dualview>) -> (f64, memref<8xf64, dualview>) {
  %1 = arith.constant 2 : index
  %2 = arith.constant 4 : index
  %3 = arith.constant 1 : index
  %4 = arith.constant 3 : index
  %5 = arith.constant 0 : index
  %6 = arith.constant 42.0 : f64
  %7 = memref.subview %0[%1][%2]
  memref.store %6, %7[%3]
  kokkos.modify(%0) {space = host}
  kokkos.sync(%0) {space = device}
  kokkos.range_parallel (%8) in (%2) {executionSpace = device, parallelLevel = toprange} {
    %9 = memref.load %7[%8]
    %10 = arith.addf(%9, %6)
    memref.store %10, %7[%8]
    kokkos.yield
  }
  kokkos.modify(%0) {space = device}
  kokkos.sync(%0) {space = host}
  %11 = memref.load %0[%4]
  func.return(%11, %0)
}
