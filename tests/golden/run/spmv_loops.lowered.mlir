func.func @spmv(%0: memref<?xindex, dualview>, %1: memref<?xindex, dualview>, %2: memref<?xf64, dualview>, %3: memref<?xf64, dualview>, %4: memref<?xf64, dualview>) -> (memref<?xf64, dualview>) {
  %5 = arith.constant 0 : index
  %6 = arith.constant 1 : index
  %7 = memref.dim(%0) {index = 0}
  %8 = arith.subi(%7, %6)
  %9 = arith.constant 1 : index
  %10 = memref.dim(%0) {index = 0}
  %11 = arith.subi(%10, %9)
  %12 = memref.load %0[%11]
  %13 = arith.maxsi(%11, %9)
  %14 = arith.ceildivsi(%12, %13)
  %15 = arith.constant 32 : index
  %16 = arith.constant 16 : index
  %17 = arith.cmpi(%14, %16) {predicate = sle}
  %18 = arith.select(%17, %16, %15)
  %19 = arith.constant 8 : index
  %20 = arith.cmpi(%14, %19) {predicate = sle}
  %21 = arith.select(%20, %19, %18)
  %22 = arith.constant 4 : index
  %23 = arith.cmpi(%14, %22) {predicate = sle}
  %24 = arith.select(%23, %22, %21)
  %25 = arith.constant 2 : index
  %26 = arith.cmpi(%14, %25) {predicate = sle}
  %27 = arith.select(%26, %25, %24)
  %28 = arith.constant 1 : index
  %29 = arith.cmpi(%14, %28) {predicate = sle}
  %30 = arith.select(%29, %28, %27)
  kokkos.sync(%0) {space = device}
  kokkos.sync(%2) {space = device}
  kokkos.sync(%1) {space = device}
  kokkos.sync(%3) {space = device}
  kokkos.thread_parallel (%31) in (%8) vector_length(%30) {executionSpace = device} {
    %32 = memref.load %0[%31]
    %33 = arith.addi(%31, %6)
    %34 = memref.load %0[%33]
    %35 = arith.subi(%34, %32)
    %36 = arith.constant 0.0 : f64
    %37 = kokkos.range_parallel (%38) in (%35) init(%36) {parallelLevel = threadvector} {
      %39 = arith.addi(%32, %38)
      %40 = memref.load %2[%39]
      %41 = memref.load %1[%39]
      %42 = memref.load %3[%41]
      %43 = arith.mulf(%40, %42)
      scf.reduce(%43) {
        ^(%44: f64, %45: f64):
        %46 = arith.addf(%44, %45)
        scf.reduce.return(%46)
      }
    }
    kokkos.single {level = perThread} {
      memref.store %37, %4[%31]
      kokkos.yield
    }
    kokkos.yield
  }
  kokkos.modify(%4) {space = device}
  func.return(%4)
}
