func.func @gcn(%0: memref<?xindex, dualview>, %1: memref<?xi32, dualview>, %2: memref<?xf32, dualview>, %3: memref<?x?xf32, dualview>, %4: memref<?x?xf32, dualview>, %5: memref<?x?xf32, dualview>) -> (memref<?x?xf32, dualview>) {
  %6 = arith.constant 0 : index
  %7 = arith.constant 1 : index
  %8 = memref.dim(%0) {index = 0}
  %9 = arith.subi(%8, %7)
  %10 = memref.dim(%3) {index = 1}
  %11 = memref.dim(%4) {index = 1}
  %12 = memref.alloc(%9, %10) : memref<?x?xf32, device>
  %13 = memref.alloc(%9, %11) : memref<?x?xf32, device>
  %14 = arith.constant 0 : index
  %15 = arith.constant 1 : index
  %16 = arith.muli(%9, %10)
  %17 = arith.constant 1 : index
  %18 = memref.dim(%0) {index = 0}
  %19 = arith.subi(%18, %17)
  %20 = memref.load %0[%19]
  %21 = arith.maxsi(%19, %17)
  %22 = arith.ceildivsi(%20, %21)
  %23 = arith.constant 32 : index
  %24 = arith.constant 16 : index
  %25 = arith.cmpi(%22, %24) {predicate = sle}
  %26 = arith.select(%25, %24, %23)
  %27 = arith.constant 8 : index
  %28 = arith.cmpi(%22, %27) {predicate = sle}
  %29 = arith.select(%28, %27, %26)
  %30 = arith.constant 4 : index
  %31 = arith.cmpi(%22, %30) {predicate = sle}
  %32 = arith.select(%31, %30, %29)
  %33 = arith.constant 2 : index
  %34 = arith.cmpi(%22, %33) {predicate = sle}
  %35 = arith.select(%34, %33, %32)
  %36 = arith.constant 1 : index
  %37 = arith.cmpi(%22, %36) {predicate = sle}
  %38 = arith.select(%37, %36, %35)
  kokkos.sync(%0) {space = device}
  kokkos.sync(%2) {space = device}
  kokkos.sync(%1) {space = device}
  kokkos.sync(%3) {space = device}
  kokkos.thread_parallel (%39) in (%16) vector_length(%38) {executionSpace = device} {
    %40 = arith.divi(%39, %10)
    %41 = arith.muli(%40, %10)
    %42 = arith.subi(%39, %41)
    %43 = memref.load %0[%40]
    %44 = arith.addi(%40, %7)
    %45 = memref.load %0[%44]
    %46 = arith.subi(%45, %43)
    %47 = arith.constant 0.0 : f32
    %48 = kokkos.range_parallel (%49) in (%46) init(%47) {parallelLevel = threadvector} {
      %50 = arith.addi(%43, %49)
      %51 = memref.load %2[%50]
      %52 = memref.load %1[%50]
      %53 = arith.index_cast(%52) : index
      %54 = memref.load %3[%53, %42]
      %55 = arith.mulf(%51, %54)
      scf.reduce(%55) {
        ^(%56: f32, %57: f32):
        %58 = arith.addf(%56, %57)
        scf.reduce.return(%58)
      }
    }
    kokkos.single {level = perThread} {
      memref.store %48, %12[%40, %42]
      kokkos.yield
    }
    kokkos.yield
  }
  %59 = memref.dim(%12) {index = 0}
  %60 = memref.dim(%4) {index = 1}
  %61 = memref.dim(%12) {index = 1}
  %62 = arith.constant 0 : index
  %63 = arith.constant 1 : index
  kokkos.sync(%4) {space = device}
  kokkos.team_parallel (%64, %65) in (%59) {executionSpace = device} {
    %66 = arith.constant 0 : index
    %67 = arith.constant 1 : index
    kokkos.range_parallel (%68) in (%60) {parallelLevel = teamthread} {
      %69 = arith.constant 0.0 : f32
      %70 = arith.constant 0 : index
      %71 = arith.constant 1 : index
      %72 = kokkos.range_parallel (%73) in (%61) init(%69) {parallelLevel = threadvector} {
        %74 = memref.load %12[%64, %73]
        %75 = memref.load %4[%73, %68]
        %76 = arith.mulf(%74, %75)
        scf.reduce(%76) {
          ^(%77: f32, %78: f32):
          %79 = arith.addf(%77, %78)
          scf.reduce.return(%79)
        }
      }
      kokkos.single {level = perThread} {
        memref.store %72, %13[%64, %68]
        kokkos.yield
      }
      kokkos.yield
    }
    kokkos.team_barrier
    kokkos.yield
  }
  %80 = memref.dim(%5) {index = 0}
  %81 = memref.dim(%5) {index = 1}
  %82 = arith.constant 0 : index
  %83 = arith.constant 1 : index
  kokkos.range_parallel (%84, %85) in (%80, %81) {executionSpace = device, parallelLevel = topmdrange} {
    %86 = memref.load %13[%84, %85]
    %87 = arith.constant 0.0 : f32
    %88 = arith.cmpf(%86, %87) {predicate = ogt}
    %89 = arith.select(%88, %86, %87)
    memref.store %89, %5[%84, %85]
    kokkos.yield
  }
  kokkos.modify(%5) {space = device}
  func.return(%5)
}
