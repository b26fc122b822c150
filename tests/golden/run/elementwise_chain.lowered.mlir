func.func @ewchain(%0: memref<?x?xf64, dualview>, %1: memref<?x?xf64, dualview>) -> (memref<?x?xf64, dualview>) {
  %2 = memref.dim(%0) {index = 0}
  %3 = memref.dim(%0) {index = 1}
  %4 = memref.alloc(%2, %3) : memref<?x?xf64, device>
  %5 = memref.alloc(%2, %3) : memref<?x?xf64, dualview>
  %6 = memref.dim(%4) {index = 0}
  %7 = memref.dim(%4) {index = 1}
  %8 = arith.constant 0 : index
  %9 = arith.constant 1 : index
  kokkos.sync(%0) {space = device}
  kokkos.sync(%1) {space = device}
  kokkos.range_parallel (%10, %11) in (%6, %7) {executionSpace = device, parallelLevel = topmdrange} {
    %12 = memref.load %0[%10, %11]
    %13 = memref.load %1[%10, %11]
    %14 = arith.mulf(%12, %13)
    memref.store %14, %4[%10, %11]
    kokkos.yield
  }
  %15 = memref.dim(%5) {index = 0}
  %16 = memref.dim(%5) {index = 1}
  %17 = arith.constant 0 : index
  %18 = arith.constant 1 : index
  kokkos.range_parallel (%19, %20) in (%15, %16) {executionSpace = device, parallelLevel = topmdrange} {
    %21 = memref.load %4[%19, %20]
    %22 = memref.load %0[%19, %20]
    %23 = arith.addf(%21, %22)
    memref.store %23, %5[%19, %20]
    kokkos.yield
  }
  kokkos.modify(%5) {space = device}
  func.return(%5)
}
