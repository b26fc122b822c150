func.func @rowsums(%0: memref<16x8xf64>, %1: memref<16xf64>) -> (memref<16xf64>) {
  %2 = arith.constant 0 : index
  %3 = arith.constant 1 : index
  %4 = arith.constant 16 : index
  %5 = arith.constant 8 : index
  scf.parallel %6 = %2 to %4 step %3 {
    %7 = arith.constant 0.0 : f64
    %8 = scf.parallel %9 = %2 to %5 step %3 init(%7) {
      %10 = memref.load %0[%6, %9]
      scf.reduce(%10) {
        ^(%11: f64, %12: f64):
        %13 = arith.addf(%11, %12)
        scf.reduce.return(%13)
      }
    }
    memref.store %8, %1[%6]
    scf.yield
  }
  func.return(%1)
}
