func.func @matmul(%0: memref<?x?xf64, dualview>, %1: memref<?x?xf64, dualview>, %2: memref<?x?xf64, dualview>) -> (memref<?x?xf64, dualview>) {
  kokkos.sync(%0) {space = device}
  kokkos.sync(%1) {space = device}
  kokkos.gemm(%0, %1, %2)
  kokkos.modify(%2) {space = device}
  func.return(%2)
}
