func.func @matvec(%0: memref<64x64xf64, dualview>, %1: memref<64xf64, dualview>) -> (memref<64xf64, dualview>) {
  %2 = memref.alloc : memref<64xf64, dualview>
  kokkos.sync(%0) {space = device}
  kokkos.sync(%1) {space = device}
  kokkos.gemv(%0, %1, %2)
  kokkos.modify(%2) {space = device}
  func.return(%2)
}
