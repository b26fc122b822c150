func.func @bmm(%0: memref<4x8x8xf32, dualview>, %1: memref<4x8x8xf32, dualview>) -> (memref<4x8x8xf32, dualview>) {
  %2 = memref.alloc : memref<4x8x8xf32, dualview>
  %3 = arith.constant 4 : index
  %4 = arith.constant 8 : index
  %5 = arith.constant 8 : index
  %6 = arith.constant 8 : index
  %7 = arith.constant 0 : index
  %8 = arith.constant 1 : index
  %9 = arith.constant 8 : index
  kokkos.sync(%0) {space = device}
  kokkos.sync(%1) {space = device}
  kokkos.team_parallel (%10, %11) in (%3) vector_length(%9) {executionSpace = device} {
    %12 = arith.constant 0 : index
    %13 = arith.constant 1 : index
    kokkos.range_parallel (%14) in (%4) {parallelLevel = teamthread} {
      %15 = arith.constant 0 : index
      %16 = arith.constant 1 : index
      %17 = arith.constant 0 : index
      %18 = arith.constant 1 : index
      scf.for %19 = %17 to %5 step %18 {
        %20 = arith.constant 0.0 : f32
        %21 = arith.constant 0 : index
        %22 = arith.constant 1 : index
        %23 = kokkos.range_parallel (%24) in (%6) init(%20) {parallelLevel = threadvector} {
          %25 = memref.load %0[%10, %14, %24]
          %26 = memref.load %1[%10, %24, %19]
          %27 = arith.mulf(%25, %26)
          scf.reduce(%27) {
            ^(%28: f32, %29: f32):
            %30 = arith.addf(%28, %29)
            scf.reduce.return(%30)
          }
        }
        kokkos.single {level = perThread} {
          memref.store %23, %2[%10, %14, %19]
          kokkos.yield
        }
        scf.yield
      }
      kokkos.yield
    }
    kokkos.team_barrier
    kokkos.yield
  }
  kokkos.modify(%2) {space = device}
  func.return(%2)
}
