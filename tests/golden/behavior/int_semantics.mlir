func.func @f(%0: memref<?xi64, dualview>, %1: memref<?xi64, dualview>, %2: memref<?xi32, dualview>, %3: memref<?xi64, dualview>) -> (memref<?xi32, dualview>, memref<?xi64, dualview>) {
  %4 = arith.constant 0 : index
  %5 = arith.constant 1 : index
  %6 = memref.dim(%0) {index = 0}
  %7 = arith.constant 3 : i64
  kokkos.sync(%0) {space = device}
  kokkos.sync(%1) {space = device}
  kokkos.range_parallel (%8) in (%6) {executionSpace = device, parallelLevel = toprange} {
    %9 = memref.load %0[%8]
    %10 = memref.load %1[%8]
    %11 = arith.muli(%9, %10)
    %12 = arith.index_cast(%11) : index
    %13 = arith.index_cast(%12) : i32
    memref.store %13, %2[%8]
    %14 = arith.cmpi(%9, %10) {predicate = ult}
    %15 = arith.shli(%9, %7)
    %16 = arith.select(%14, %15, %11)
    %17 = arith.maxsi(%16, %10)
    memref.store %17, %3[%8]
    kokkos.yield
  }
  kokkos.modify(%2) {space = device}
  kokkos.modify(%3) {space = device}
  func.return(%2, %3)
}
