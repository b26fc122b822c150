func.func @teams(%0: memref<4x8xf64>, %1: memref<4x8xf64>, %2: memref<4xf64>) -> (memref<4xf64>) {
  %3 = arith.constant 0 : index
  %4 = arith.constant 1 : index
  %5 = arith.constant 4 : index
  %6 = arith.constant 8 : index
  scf.parallel %7 = %3 to %5 step %4 {
    scf.parallel %8 = %3 to %6 step %4 {
      %9 = arith.constant 0.0 : f64
      %10 = scf.parallel %11 = %3 to %6 step %4 init(%9) {
        %12 = memref.load %0[%7, %11]
        %13 = memref.load %0[%7, %8]
        %14 = arith.mulf(%12, %13)
        scf.reduce(%14) {
          ^(%15: f64, %16: f64):
          %17 = arith.addf(%15, %16)
          scf.reduce.return(%17)
        }
      }
      memref.store %10, %1[%7, %8]
      scf.yield
    }
    %18 = memref.load %1[%7, %3]
    memref.store %18, %2[%7]
    %19 = arith.constant 0.0 : f64
    %20 = scf.parallel %21 = %3 to %6 step %4 init(%19) {
      %22 = memref.load %1[%7, %21]
      scf.reduce(%22) {
        ^(%23: f64, %24: f64):
        %25 = arith.addf(%23, %24)
        scf.reduce.return(%25)
      }
    }
    memref.store %20, %2[%7]
    scf.yield
  }
  func.return(%2)
}
