// Dense C = A * B with runtime extents, C passed in (overwritten).  Same op
// as tests/fixtures/matmul_f64.mlir; dynamic shapes so one emitted kernel
// serves every size including the 4096^3 benchmark.
func @matmul(%a: memref<?x?xf32>, %b: memref<?x?xf32>, %c: memref<?x?xf32>) -> (memref<?x?xf32>) {
  linalg.matmul(%a, %b, %c)
  func.return(%c)
}
