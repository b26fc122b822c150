func.func @matvec(%0: memref<?x?xf64, dualview>, %1: memref<?xf64, dualview>, %2: memref<?xf64, dualview>) -> (memref<?xf64, dualview>) {
  %3 = memref.dim(%0) {index = 0}
  %4 = memref.dim(%0) {index = 1}
  %5 = arith.constant 0 : index
  %6 = arith.constant 1 : index
  kokkos.sync(%0) {space = device}
  kokkos.sync(%1) {space = device}
  kokkos.thread_parallel (%7) in (%3) {executionSpace = device} {
    %8 = arith.constant 0.0 : f64
    %9 = arith.constant 0 : index
    %10 = arith.constant 1 : index
    %11 = kokkos.range_parallel (%12) in (%4) init(%8) {parallelLevel = threadvector} {
      %13 = memref.load %0[%7, %12]
      %14 = memref.load %1[%12]
      %15 = arith.mulf(%13, %14)
      scf.reduce(%15) {
        ^(%16: f64, %17: f64):
        %18 = arith.addf(%16, %17)
        scf.reduce.return(%18)
      }
    }
    kokkos.single {level = perThread} {
      memref.store %11, %2[%7]
      kokkos.yield
    }
    kokkos.yield
  }
  kokkos.modify(%2) {space = device}
  func.return(%2)
}
