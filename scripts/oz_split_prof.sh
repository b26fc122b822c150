#!/bin/bash
OUT=gpurun_out/${1:-ozsplit}; mkdir -p $OUT
for K in ozaki_split_rows ozaki_split_cols ozaki_colmax; do
  timeout 600 ncu --set full --clock-control none -k regex:$K -s 2 -c 1 -o $OUT/$K python scripts/gemm_f32_mixed_launches.py > /dev/null 2>&1
  LAPIS_X=1 python scripts/ncu_summary.py $OUT/$K.ncu-rep > $OUT/$K.txt 2>&1
  rm -f $OUT/$K.ncu-rep
  echo "== $K"; grep -E "duration|dram_gbs|issue_active|warps_active|top_stalls" -A3 $OUT/$K.txt | head -14
done
