func.func @dot(%0: memref<?xf64>, %1: memref<?xf64>) -> (f64) {
  %2 = arith.constant 0 : index
  %3 = arith.constant 1 : index
  %4 = memref.dim(%0) {index = 0}
  %5 = arith.constant 0.0 : f64
  %6 = scf.parallel %7 = %2 to %4 step %3 init(%5) {
    %8 = memref.load %0[%7]
    %9 = memref.load %1[%7]
    %10 = arith.mulf(%8, %9)
    scf.reduce(%10) {
      ^(%11: f64, %12: f64):
      %13 = arith.addf(%11, %12)
      scf.reduce.return(%13)
    }
  }
  func.return(%6)
}
