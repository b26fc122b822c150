func.func @spmm(%0: memref<?xindex, dualview>, %1: memref<?xi32, dualview>, %2: memref<?xf64, dualview>, %3: memref<?x?xf64, dualview>, %4: memref<?x?xf64, dualview>) -> (memref<?x?xf64, dualview>) {
  %5 = arith.constant 0 : index
  %6 = arith.constant 1 : index
  %7 = memref.dim(%0) {index = 0}
  %8 = arith.subi(%7, %6)
  %9 = memref.dim(%3) {index = 1}
  %10 = arith.constant 0 : index
  %11 = arith.constant 1 : index
  %12 = arith.muli(%8, %9)
  %13 = arith.constant 1 : index
  %14 = memref.dim(%0) {index = 0}
  %15 = arith.subi(%14, %13)
  %16 = memref.load %0[%15]
  %17 = arith.maxsi(%15, %13)
  %18 = arith.ceildivsi(%16, %17)
  %19 = arith.constant 32 : index
  %20 = arith.constant 16 : index
  %21 = arith.cmpi(%18, %20) {predicate = sle}
  %22 = arith.select(%21, %20, %19)
  %23 = arith.constant 8 : index
  %24 = arith.cmpi(%18, %23) {predicate = sle}
  %25 = arith.select(%24, %23, %22)
  %26 = arith.constant 4 : index
  %27 = arith.cmpi(%18, %26) {predicate = sle}
  %28 = arith.select(%27, %26, %25)
  %29 = arith.constant 2 : index
  %30 = arith.cmpi(%18, %29) {predicate = sle}
  %31 = arith.select(%30, %29, %28)
  %32 = arith.constant 1 : index
  %33 = arith.cmpi(%18, %32) {predicate = sle}
  %34 = arith.select(%33, %32, %31)
  kokkos.sync(%0) {space = device}
  kokkos.sync(%2) {space = device}
  kokkos.sync(%1) {space = device}
  kokkos.sync(%3) {space = device}
  kokkos.thread_parallel (%35) in (%12) vector_length(%34) {executionSpace = device} {
    %36 = arith.divi(%35, %9)
    %37 = arith.muli(%36, %9)
    %38 = arith.subi(%35, %37)
    %39 = memref.load %0[%36]
    %40 = arith.addi(%36, %6)
    %41 = memref.load %0[%40]
    %42 = arith.subi(%41, %39)
    %43 = arith.constant 0.0 : f64
    %44 = kokkos.range_parallel (%45) in (%42) init(%43) {parallelLevel = threadvector} {
      %46 = arith.addi(%39, %45)
      %47 = memref.load %2[%46]
      %48 = memref.load %1[%46]
      %49 = arith.index_cast(%48) : index
      %50 = memref.load %3[%49, %38]
      %51 = arith.mulf(%47, %50)
      scf.reduce(%51) {
        ^(%52: f64, %53: f64):
        %54 = arith.addf(%52, %53)
        scf.reduce.return(%54)
      }
    }
    kokkos.single {level = perThread} {
      memref.store %44, %4[%36, %38]
      kokkos.yield
    }
    kokkos.yield
  }
  kokkos.modify(%4) {space = device}
  func.return(%4)
}
