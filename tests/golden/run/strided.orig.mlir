func.func @strided(%0: memref<16xf64>) -> (memref<16xf64>) {
  %1 = arith.constant 3 : index
  %2 = arith.constant 11 : index
  %3 = arith.constant 2 : index
  %4 = arith.constant 1.0 : f64
  scf.parallel %5 = %1 to %2 step %3 {
    %6 = memref.load %0[%5]
    %7 = arith.addf(%6, %4)
    memref.store %7, %0[%5]
    scf.yield
  }
  func.return(%0)
}
