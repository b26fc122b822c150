func.func @hostloop(%0: memref<8x4xf64>, %1: memref<8xf64>) -> (memref<8xf64>) {
  %2 = arith.constant 0 : index
  %3 = arith.constant 1 : index
  %4 = arith.constant 8 : index
  %5 = arith.constant 4 : index
  %6 = arith.constant 3 : index
  %7 = arith.constant 2.0 : f64
  scf.parallel %8 = %2 to %4 step %3 {
    %9 = memref.alloc : memref<4xf64>
    scf.for %10 = %2 to %5 step %3 {
      %11 = memref.load %0[%8, %10]
      %12 = arith.mulf(%11, %7)
      memref.store %12, %9[%10]
      scf.yield
    }
    %13 = memref.load %9[%6]
    memref.store %13, %1[%8]
    memref.dealloc(%9)
    scf.yield
  }
  func.return(%1)
}
