// Dense C = A * B with runtime extents, C passed in (overwritten).  Same op
// as tests/fixtures/matmul_f64.mlir; dynamic shapes so one emitted kernel
// serves every size including the 4096^3 benchmark.
func @matmul(%a: memref<?x?xf64>, %b: memref<?x?xf64>, %c: memref<?x?xf64>) -> (memref<?x?xf64>) {
  linalg.matmul(%a, %b, %c)
  func.return(%c)
}
