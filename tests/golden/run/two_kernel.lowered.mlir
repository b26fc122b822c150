func.func @two_kernel(%0: memref<64xf64, dualview>) -> (memref<64xf64, dualview>) {
  %1 = arith.constant 0 : index
  %2 = arith.constant 1 : index
  %3 = arith.constant 64 : index
  %4 = arith.constant 2.0 : f64
  %5 = arith.constant 1.0 : f64
  %6 = arith.constant 3.0 : f64
  %7 = memref.alloc : memref<64xf64, dualview>
  %8 = memref.alloc : memref<64xf64, device>
  %9 = memref.alloc : memref<64xf64, dualview>
  scf.for %10 = %1 to %3 step %2 {
    %11 = memref.load %0[%10]
    %12 = arith.mulf(%11, %4)
    memref.store %12, %7[%10]
    scf.yield
  }
  kokkos.modify(%7) {space = host}
  kokkos.sync(%7) {space = device}
  kokkos.range_parallel (%13) in (%3) {executionSpace = device, parallelLevel = toprange} {
    %14 = memref.load %7[%13]
    %15 = arith.addf(%14, %5)
    memref.store %15, %8[%13]
    kokkos.yield
  }
  kokkos.range_parallel (%16) in (%3) {executionSpace = device, parallelLevel = toprange} {
    %17 = memref.load %7[%16]
    %18 = arith.mulf(%17, %6)
    memref.store %18, %9[%16]
    kokkos.yield
  }
  kokkos.modify(%9) {space = device}
  func.return(%9)
}
