func.func @scale(%0: memref<128xf64>, %1: memref<128xf64>) -> (memref<128xf64>) {
  %2 = arith.constant 0 : index
  %3 = arith.constant 1 : index
  %4 = arith.constant 128 : index
  %5 = arith.constant 2.0 : f64
  scf.parallel %6 = %2 to %4 step %3 {
    %7 = memref.load %0[%6]
    %8 = arith.mulf(%7, %5)
    memref.store %8, %1[%6]
    scf.yield
  }
  func.return(%1)
}
