memref.global @weights {value = dense<[0.5, 1.5, 2.5, 3.5]>} : memref<4xf64>

func.func @apply_weights(%0: memref<4xf64>) -> (memref<4xf64>) {
  %1 = arith.constant 0 : index
  %2 = arith.constant 1 : index
  %3 = arith.constant 4 : index
  %4 = memref.get_global @weights : memref<4xf64>
  %5 = memref.alloc : memref<4xf64>
  scf.parallel %6 = %1 to %3 step %2 {
    %7 = memref.load %0[%6]
    %8 = memref.load %4[%6]
    %9 = arith.mulf(%7, %8)
    memref.store %9, %5[%6]
    scf.yield
  }
  func.return(%5)
}
