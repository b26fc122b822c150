func.func @c(%0: memref<?xf64, dualview>) -> (f64) {
  %1 = arith.constant 0 : index
  %2 = arith.constant 1 : index
  %3 = memref.dim(%0) {index = 0}
  %4 = arith.constant 1.0 : f64
  kokkos.sync(%0) {space = device}
  %5 = kokkos.range_parallel (%6) in (%3) init(%4) {executionSpace = device, parallelLevel = toprange} {
    %7 = memref.load %0[%6]
    scf.reduce(%7) {
      ^(%8: f64, %9: f64):
      %10 = arith.subf(%8, %9)
      scf.reduce.return(%10)
    }
  }
  func.return(%5)
}
