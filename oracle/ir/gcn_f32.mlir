// GCN layer H = relu((A_hat * X) * W) as one function (SURVEY A.5 / config 4):
// loop-nest SpMM (f32), linalg.matmul, linalg.elementwise ReLU (cmpf ogt +
// select).  Temporaries are device-local allocations.
func @gcn(%rowptr: memref<?xindex>, %colind: memref<?xi32>, %values: memref<?xf32>,
          %x: memref<?x?xf32>, %w: memref<?x?xf32>, %h: memref<?x?xf32>) -> (memref<?x?xf32>) {
  %c0 = arith.constant 0 : index
  %c1 = arith.constant 1 : index
  %nb = memref.dim(%rowptr) {index = 0}
  %nrows = arith.subi(%nb, %c1)
  %nfeat = memref.dim(%x) {index = 1}
  %nout = memref.dim(%w) {index = 1}
  %ax = memref.alloc(%nrows, %nfeat) : memref<?x?xf32>
  %t = memref.alloc(%nrows, %nout) : memref<?x?xf32>
  scf.parallel (%i, %c) = (%c0, %c0) to (%nrows, %nfeat) step (%c1, %c1) {
    %begin = memref.load %rowptr[%i]
    %inext = arith.addi(%i, %c1)
    %end = memref.load %rowptr[%inext]
    %len = arith.subi(%end, %begin)
    %zero = arith.constant 0.0 : f32
    %sum = scf.parallel %jj = %c0 to %len step %c1 init(%zero) {
      %j = arith.addi(%begin, %jj)
      %v = memref.load %values[%j]
      %col32 = memref.load %colind[%j]
      %col = arith.index_cast(%col32) : index
      %xv = memref.load %x[%col, %c]
      %prod = arith.mulf(%v, %xv)
      scf.reduce(%prod) {
        ^(%a: f32, %b: f32):
          %s = arith.addf(%a, %b)
          scf.reduce.return(%s)
      }
    }
    memref.store %sum, %ax[%i, %c]
    scf.yield
  }
  linalg.matmul(%ax, %w, %t)
  linalg.elementwise(%t, %h) {
    ^(%v: f32):
      %z = arith.constant 0.0 : f32
      %pos = arith.cmpf(%v, %z) {predicate = "ogt"}
      %r = arith.select(%pos, %v, %z)
      scf.yield(%r)
  }
  func.return(%h)
}
