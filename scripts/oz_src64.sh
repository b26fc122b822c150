#!/bin/bash
OUT=gpurun_out/${1:-ozsrc64}; mkdir -p $OUT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ozaki_split_rows -s 1 -c 1 -o $OUT/r python scripts/oz_prof_run.py > /dev/null 2>&1
ncu -i $OUT/r.ncu-rep --page source --csv > $OUT/r.source.csv 2>/dev/null
rm -f $OUT/r.ncu-rep
