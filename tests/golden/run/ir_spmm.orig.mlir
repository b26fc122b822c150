func.func @spmm(%0: memref<?xindex>, %1: memref<?xi32>, %2: memref<?xf64>, %3: memref<?x?xf64>, %4: memref<?x?xf64>) -> (memref<?x?xf64>) {
  %5 = arith.constant 0 : index
  %6 = arith.constant 1 : index
  %7 = memref.dim(%0) {index = 0}
  %8 = arith.subi(%7, %6)
  %9 = memref.dim(%3) {index = 1}
  scf.parallel (%10, %11) = (%5, %5) to (%8, %9) step (%6, %6) {
    %12 = memref.load %0[%10]
    %13 = arith.addi(%10, %6)
    %14 = memref.load %0[%13]
    %15 = arith.subi(%14, %12)
    %16 = arith.constant 0.0 : f64
    %17 = scf.parallel %18 = %5 to %15 step %6 init(%16) {
      %19 = arith.addi(%12, %18)
      %20 = memref.load %2[%19]
      %21 = memref.load %1[%19]
      %22 = arith.index_cast(%21) : index
      %23 = memref.load %3[%22, %11]
      %24 = arith.mulf(%20, %23)
      scf.reduce(%24) {
        ^(%25: f64, %26: f64):
        %27 = arith.addf(%25, %26)
        scf.reduce.return(%27)
      }
    }
    memref.store %17, %4[%10, %11]
    scf.yield
  }
  func.return(%4)
}
