#!/bin/bash
# ncu --set full of the exact SpMV variants on a 24M-row 27-point stencil
OUT=gpurun_out/${1:-ncu_exact}; mkdir -p $OUT
P="python scripts/spmv_variant.py"
$P tree; $P exact; LAPIS_B200_SPMV_EXACT_KIND=1 LAPIS_B200_SPMV_KERNEL=vec $P exact; LAPIS_B200_SPMV_KERNEL=vec $P exact; LAPIS_B200_RS_CFG=1 $P exact
NC="timeout 600 ncu --set full --clock-control none -s 3 -c 1"
$NC -k regex:spmv_vector_kernel -o $OUT/tree $P tree > /dev/null 2>&1
LAPIS_B200_SPMV_KERNEL=vec $NC -k regex:spmv_vector_kernel -o $OUT/vec_exact $P exact > /dev/null 2>&1
LAPIS_B200_SPMV_EXACT_KIND=1 LAPIS_B200_SPMV_KERNEL=vec $NC -k regex:spmv_vector_chunk -o $OUT/chunk8 $P exact > /dev/null 2>&1
LAPIS_B200_RS_CFG=1 $NC -k regex:spmv_rowstream -o $OUT/rs1 $P exact > /dev/null 2>&1
ls $OUT
for r in $OUT/*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  python scripts/ncu_summary.py $r --json $b.summary.json > $b.summary.txt 2>&1
  rm -f $r
done
du -sh $OUT
