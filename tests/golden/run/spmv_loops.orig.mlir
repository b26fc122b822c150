func.func @spmv(%0: memref<?xindex>, %1: memref<?xindex>, %2: memref<?xf64>, %3: memref<?xf64>, %4: memref<?xf64>) -> (memref<?xf64>) {
  %5 = arith.constant 0 : index
  %6 = arith.constant 1 : index
  %7 = memref.dim(%0) {index = 0}
  %8 = arith.subi(%7, %6)
  scf.parallel %9 = %5 to %8 step %6 {
    %10 = memref.load %0[%9]
    %11 = arith.addi(%9, %6)
    %12 = memref.load %0[%11]
    %13 = arith.subi(%12, %10)
    %14 = arith.constant 0.0 : f64
    %15 = scf.parallel %16 = %5 to %13 step %6 init(%14) {
      %17 = arith.addi(%10, %16)
      %18 = memref.load %2[%17]
      %19 = memref.load %1[%17]
      %20 = memref.load %3[%19]
      %21 = arith.mulf(%18, %20)
      scf.reduce(%21) {
        ^(%22: f64, %23: f64):
        %24 = arith.addf(%22, %23)
        scf.reduce.return(%24)
      }
    }
    memref.store %15, %4[%9]
    scf.yield
  }
  func.return(%4)
}
