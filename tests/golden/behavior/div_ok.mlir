func.func @f(%0: memref<?xi64, dualview>, %1: memref<?xi64, dualview>, %2: memref<?xi64, dualview>) -> (memref<?xi64, dualview>) {
  %3 = arith.constant 0 : index
  %4 = arith.constant 1 : index
  %5 = memref.dim(%0) {index = 0}
  kokkos.sync(%0) {space = device}
  kokkos.sync(%1) {space = device}
  kokkos.range_parallel (%6) in (%5) {executionSpace = device, parallelLevel = toprange} {
    %7 = memref.load %0[%6]
    %8 = memref.load %1[%6]
    %9 = arith.divi(%7, %8)
    %10 = arith.ceildivsi(%7, %8)
    %11 = arith.addi(%9, %10)
    memref.store %11, %2[%6]
    kokkos.yield
  }
  kokkos.modify(%2) {space = device}
  func.return(%2)
}
