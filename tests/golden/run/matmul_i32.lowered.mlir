func.func @matmul(%0: memref<16x16xi32, dualview>, %1: memref<16x16xi32, dualview>) -> (memref<16x16xi32, dualview>) {
  %2 = memref.alloc : memref<16x16xi32, dualview>
  %3 = arith.constant 16 : index
  %4 = arith.constant 16 : index
  %5 = arith.constant 16 : index
  %6 = arith.constant 0 : index
  %7 = arith.constant 1 : index
  %8 = arith.constant 16 : index
  kokkos.sync(%0) {space = device}
  kokkos.sync(%1) {space = device}
  kokkos.team_parallel (%9, %10) in (%3) vector_length(%8) {executionSpace = device} {
    %11 = arith.constant 0 : index
    %12 = arith.constant 1 : index
    kokkos.range_parallel (%13) in (%4) {parallelLevel = teamthread} {
      %14 = arith.constant 0 : i32
      %15 = arith.constant 0 : index
      %16 = arith.constant 1 : index
      %17 = kokkos.range_parallel (%18) in (%5) init(%14) {parallelLevel = threadvector} {
        %19 = memref.load %0[%9, %18]
        %20 = memref.load %1[%18, %13]
        %21 = arith.muli(%19, %20)
        scf.reduce(%21) {
          ^(%22: i32, %23: i32):
          %24 = arith.addi(%22, %23)
          scf.reduce.return(%24)
        }
      }
      kokkos.single {level = perThread} {
        memref.store %17, %2[%9, %13]
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
