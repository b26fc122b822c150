func.func @rowsum(%0: memref<16x8xf64>) -> (memref<16xf64>) {
  %1 = memref.alloc : memref<16xf64>
  linalg.reduce(%0, %1) {axes = [1], combiner = add}
  func.return(%1)
}
