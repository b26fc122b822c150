memref.global @weights {value = dense<[0.5, 1.5, 2.5, 3.5]>} : memref<4xf64, dualview>

func.func @apply_weights(%0: memref<4xf64, dualview>) -> (memref<4xf64, dualview>) {
  %1 = arith.constant 0 : index
  %2 = arith.constant 1 : index
  %3 = arith.constant 4 : index
  %4 = memref.get_global @weights : memref<4xf64, dualview>
  %5 = memref.alloc : memref<4xf64, dualview>
  kokkos.sync(%0) {space = device}
  %6 = memref.get_global @weights : memref<4xf64, dualview>
  kokkos.sync(%6) {space = device}
  kokkos.range_parallel (%7) in (%3) {executionSpace = device, parallelLevel = toprange} {
    %8 = memref.load %0[%7]
    %9 = memref.load %4[%7]
    %10 = arith.mulf(%8, %9)
    memref.store %10, %5[%7]
    kokkos.yield
  }
  kokkos.modify(%5) {space = device}
  func.return(%5)
}
