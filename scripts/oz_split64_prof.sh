#!/bin/bash
OUT=gpurun_out/${1:-ozs64}; mkdir -p $OUT
for K in ozaki_split_rows ozaki_split_cols; do
timeout 600 ncu --set full --clock-control none -k regex:$K -s 1 -c 1 -o $OUT/$K python scripts/oz_prof_run.py > /dev/null 2>&1
ncu -i $OUT/$K.ncu-rep --page raw --csv > $OUT/$K.raw.csv 2>/dev/null
python scripts/ncu_summary.py $OUT/$K.ncu-rep > $OUT/$K.txt 2>&1
rm -f $OUT/$K.ncu-rep
grep -E "duration|dram_read|dram_write|issue_active|warps_active|warp_instructions" $OUT/$K.txt; grep -A4 top_stalls $OUT/$K.txt
done
