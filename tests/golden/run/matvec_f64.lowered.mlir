func.func @matvec(%0: memref<64x64xf64, dualview>, %1: memref<64xf64, dualview>) -> (memref<64xf64, dualview>) {
  %2 = memref.alloc : memref<64xf64, dualview>
  %3 = arith.constant 64 : index
  %4 = arith.constant 64 : index
  %5 = arith.constant 0 : index
  %6 = arith.constant 1 : index
  %7 = arith.constant 32 : index
  kokkos.sync(%0) {space = device}
  kokkos.sync(%1) {space = device}
  kokkos.thread_parallel (%8) in (%3) vector_length(%7) {executionSpace = device} {
    %9 = arith.constant 0.0 : f64
    %10 = arith.constant 0 : index
    %11 = arith.constant 1 : index
    %12 = kokkos.range_parallel (%13) in (%4) init(%9) {parallelLevel = threadvector} {
      %14 = memref.load %0[%8, %13]
      %15 = memref.load %1[%13]
      %16 = arith.mulf(%14, %15)
      scf.reduce(%16) {
        ^(%17: f64, %18: f64):
        %19 = arith.addf(%17, %18)
        scf.reduce.return(%19)
      }
    }
    kokkos.single {level = perThread} {
      memref.store %12, %2[%8]
      kokkos.yield
    }
    kokkos.yield
  }
  kokkos.modify(%2) {space = device}
  func.return(%2)
}
