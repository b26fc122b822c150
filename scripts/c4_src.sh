#!/bin/bash
OUT=gpurun_out/${1:-c4src}; mkdir -p $OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_batch2 -s 3 -c 1 -o $OUT/r python bench.py --workload c4 --steps 1 --warmup 3 --extra none --no-cpu --e2e-steps 1 > /dev/null 2>&1
ncu -i $OUT/r.ncu-rep --page source --csv > $OUT/r.source.csv 2>/dev/null
rm -f $OUT/r.ncu-rep
