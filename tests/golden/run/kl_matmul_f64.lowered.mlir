func.func @matmul(%0: memref<32x32xf64, dualview>, %1: memref<32x32xf64, dualview>) -> (memref<32x32xf64, dualview>) {
  %2 = memref.alloc : memref<32x32xf64, dualview>
  kokkos.sync(%0) {space = device}
  kokkos.sync(%1) {space = device}
  kokkos.gemm(%0, %1, %2)
  kokkos.modify(%2) {space = device}
  func.return(%2)
}
