func.func @m(%0: memref<?x?xf64, dualview>) -> (f64) {
  %1 = arith.constant 0 : index
  %2 = arith.constant 1 : index
  %3 = memref.dim(%0) {index = 0}
  %4 = memref.dim(%0) {index = 1}
  %5 = arith.constant -1e+300 : f64
  kokkos.sync(%0) {space = device}
  %6 = kokkos.range_parallel (%7, %8) in (%3, %4) init(%5) {executionSpace = device, parallelLevel = topmdrange} {
    %9 = memref.load %0[%7, %8]
    scf.reduce(%9) {
      ^(%10: f64, %11: f64):
      %12 = arith.cmpf(%10, %11) {predicate = ogt}
      %13 = arith.select(%12, %10, %11)
      scf.reduce.return(%13)
    }
  }
  func.return(%6)
}
