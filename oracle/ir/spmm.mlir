// CSR x dense SpMM, Y[i, c] = sum_j values[j] * X[colind[j], c].
// The reference has no SpMM op (dialect.py:215-222); this is the loop-nest
// form (SURVEY A.5): a 2-D outer parallel over (row, rhs column) wrapping the
// CSR add-reduce.  The preset maps it to thread_parallel over N*K with the
// CSR vector-length hint.
func @spmm(%rowptr: memref<?xindex>, %colind: memref<?xi32>, %values: memref<?xf64>,
           %x: memref<?x?xf64>, %y: memref<?x?xf64>) -> (memref<?x?xf64>) {
  %c0 = arith.constant 0 : index
  %c1 = arith.constant 1 : index
  %nb = memref.dim(%rowptr) {index = 0}
  %nrows = arith.subi(%nb, %c1)
  %ncols = memref.dim(%x) {index = 1}
  scf.parallel (%i, %c) = (%c0, %c0) to (%nrows, %ncols) step (%c1, %c1) {
    %begin = memref.load %rowptr[%i]
    %inext = arith.addi(%i, %c1)
    %end = memref.load %rowptr[%inext]
    %len = arith.subi(%end, %begin)
    %zero = arith.constant 0.0 : f64
    %sum = scf.parallel %jj = %c0 to %len step %c1 init(%zero) {
      %j = arith.addi(%begin, %jj)
      %v = memref.load %values[%j]
      %col32 = memref.load %colind[%j]
      %col = arith.index_cast(%col32) : index
      %xv = memref.load %x[%col, %c]
      %prod = arith.mulf(%v, %xv)
      scf.reduce(%prod) {
        ^(%a: f64, %b: f64):
          %s = arith.addf(%a, %b)
          scf.reduce.return(%s)
      }
    }
    memref.store %sum, %y[%i, %c]
    scf.yield
  }
  func.return(%y)
}
