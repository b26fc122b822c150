func.func @wave(%0: memref<2x3x4x8xf64>) -> (memref<2x3x4x8xf64>) {
  %1 = arith.constant 0 : index
  %2 = arith.constant 1 : index
  %3 = arith.constant 2 : index
  %4 = arith.constant 3 : index
  %5 = arith.constant 4 : index
  %6 = arith.constant 8 : index
  %7 = arith.constant 2.0 : f64
  scf.parallel %8 = %1 to %3 step %2 {
    scf.parallel %9 = %1 to %4 step %2 {
      scf.parallel %10 = %1 to %5 step %2 {
        scf.parallel %11 = %1 to %6 step %2 {
          %12 = memref.load %0[%8, %9, %10, %11]
          %13 = arith.mulf(%12, %7)
          memref.store %13, %0[%8, %9, %10, %11]
          scf.yield
        }
        scf.yield
      }
      scf.yield
    }
    scf.yield
  }
  func.return(%0)
}
