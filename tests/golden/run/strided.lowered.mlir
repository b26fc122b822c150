func.func @strided(%0: memref<16xf64, dualview>) -> (memref<16xf64, dualview>) {
  %1 = arith.constant 3 : index
  %2 = arith.constant 11 : index
  %3 = arith.constant 2 : index
  %4 = arith.constant 1.0 : f64
  %5 = arith.constant 0 : index
  %6 = arith.constant 1 : index
  %7 = arith.constant 4 : index
  kokkos.sync(%0) {space = device}
  kokkos.range_parallel (%8) in (%7) {executionSpace = device, parallelLevel = toprange} {
    %9 = arith.muli(%8, %3)
    %10 = arith.addi(%1, %9)
    %11 = memref.load %0[%10]
    %12 = arith.addf(%11, %4)
    memref.store %12, %0[%10]
    kokkos.yield
  }
  kokkos.modify(%0) {space = device}
  func.return(%0)
}
