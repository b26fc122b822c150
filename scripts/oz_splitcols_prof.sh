#!/bin/bash
OUT=gpurun_out/${1:-ozsc}; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none -k regex:ozaki_split_cols_f32 -s 2 -c 1 -o $OUT/sc python scripts/gemm_f32_mixed_launches.py > /dev/null 2>&1
ncu -i $OUT/sc.ncu-rep --page raw --csv > $OUT/sc.raw.csv 2>/dev/null
python scripts/ncu_summary.py $OUT/sc.ncu-rep > $OUT/sc.txt 2>&1
rm -f $OUT/sc.ncu-rep
cat $OUT/sc.txt
