func.func @matmul(%0: memref<?x?xf32, dualview>, %1: memref<?x?xf32, dualview>, %2: memref<?x?xf32, dualview>) -> (memref<?x?xf32, dualview>) {
  %3 = memref.dim(%0) {index = 0}
  %4 = memref.dim(%1) {index = 1}
  %5 = memref.dim(%0) {index = 1}
  %6 = arith.constant 0 : index
  %7 = arith.constant 1 : index
  kokkos.sync(%0) {space = device}
  kokkos.sync(%1) {space = device}
  kokkos.team_parallel (%8, %9) in (%3) {executionSpace = device} {
    %10 = arith.constant 0 : index
    %11 = arith.constant 1 : index
    kokkos.range_parallel (%12) in (%4) {parallelLevel = teamthread} {
      %13 = arith.constant 0.0 : f32
      %14 = arith.constant 0 : index
      %15 = arith.constant 1 : index
      %16 = kokkos.range_parallel (%17) in (%5) init(%13) {parallelLevel = threadvector} {
        %18 = memref.load %0[%8, %17]
        %19 = memref.load %1[%17, %12]
        %20 = arith.mulf(%18, %19)
        scf.reduce(%20) {
          ^(%21: f32, %22: f32):
          %23 = arith.addf(%21, %22)
          scf.reduce.return(%23)
        }
      }
      kokkos.single {level = perThread} {
        memref.store %16, %2[%8, %12]
        kokkos.yield
      }
      kokkos.yield
    }
    kokkos.team_barrier
    kokkos.yield
  }
  kokkos.modify(%2) {space = device}
  func.return(%2)
}
