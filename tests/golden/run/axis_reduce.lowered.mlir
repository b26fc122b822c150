func.func @rowsum(%0: memref<16x8xf64, dualview>) -> (memref<16xf64, dualview>) {
  %1 = memref.alloc : memref<16xf64, dualview>
  %2 = arith.constant 16 : index
  %3 = arith.constant 8 : index
  %4 = arith.constant 0 : index
  %5 = arith.constant 1 : index
  %6 = arith.constant 8 : index
  kokkos.sync(%0) {space = device}
  kokkos.thread_parallel (%7) in (%2) vector_length(%6) {executionSpace = device} {
    %8 = arith.constant 0.0 : f64
    %9 = arith.constant 0 : index
    %10 = arith.constant 1 : index
    %11 = kokkos.range_parallel (%12) in (%3) init(%8) {parallelLevel = threadvector} {
      %13 = memref.load %0[%7, %12]
      scf.reduce(%13) {
        ^(%14: f64, %15: f64):
        %16 = arith.addf(%14, %15)
        scf.reduce.return(%16)
      }
    }
    kokkos.single {level = perThread} {
      memref.store %11, %1[%7]
      kokkos.yield
    }
    kokkos.yield
  }
  kokkos.modify(%1) {space = device}
  func.return(%1)
}
