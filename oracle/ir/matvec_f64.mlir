// Dense y = A * x with runtime extents (tests/fixtures/matvec_f64.mlir, dynamic).
func @matvec(%a: memref<?x?xf64>, %x: memref<?xf64>, %y: memref<?xf64>) -> (memref<?xf64>) {
  linalg.matvec(%a, %x, %y)
  func.return(%y)
}
