func.func @gcn(%0: memref<?xindex>, %1: memref<?xi32>, %2: memref<?xf32>, %3: memref<?x?xf32>, %4: memref<?x?xf32>, %5: memref<?x?xf32>) -> (memref<?x?xf32>) {
  %6 = arith.constant 0 : index
  %7 = arith.constant 1 : index
  %8 = memref.dim(%0) {index = 0}
  %9 = arith.subi(%8, %7)
  %10 = memref.dim(%3) {index = 1}
  %11 = memref.dim(%4) {index = 1}
  %12 = memref.alloc(%9, %10) : memref<?x?xf32>
  %13 = memref.alloc(%9, %11) : memref<?x?xf32>
  scf.parallel (%14, %15) = (%6, %6) to (%9, %10) step (%7, %7) {
    %16 = memref.load %0[%14]
    %17 = arith.addi(%14, %7)
    %18 = memref.load %0[%17]
    %19 = arith.subi(%18, %16)
    %20 = arith.constant 0.0 : f32
    %21 = scf.parallel %22 = %6 to %19 step %7 init(%20) {
      %23 = arith.addi(%16, %22)
      %24 = memref.load %2[%23]
      %25 = memref.load %1[%23]
      %26 = arith.index_cast(%25) : index
      %27 = memref.load %3[%26, %15]
      %28 = arith.mulf(%24, %27)
      scf.reduce(%28) {
        ^(%29: f32, %30: f32):
        %31 = arith.addf(%29, %30)
        scf.reduce.return(%31)
      }
    }
    memref.store %21, %12[%14, %15]
    scf.yield
  }
  linalg.matmul(%12, %4, %13)
  linalg.elementwise(%13, %5) {
    ^(%32: f32):
    %33 = arith.constant 0.0 : f32
    %34 = arith.cmpf(%32, %33) {predicate = ogt}
    %35 = arith.select(%34, %32, %33)
    scf.yield(%35)
  }
  func.return(%5)
}
