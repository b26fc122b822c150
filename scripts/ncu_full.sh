#!/bin/bash
# ncu --set full of one kernel of a bench workload; raw CSV + summary, the report removed
# usage: bash scripts/ncu_full.sh TAG WORKLOAD KERNEL_REGEX [SKIP]
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$3" -s ${4:-3} -c 1 -o $OUT/$2 \
  python bench.py --workload $2 --steps 1 --warmup 3 --extra none --no-cpu --e2e-steps 1 > $OUT/ncu.log 2>&1
ncu -i $OUT/$2.ncu-rep --page raw --csv > $OUT/$2.raw.csv 2>/dev/null
ncu -i $OUT/$2.ncu-rep --page source --csv > $OUT/$2.source.csv 2>/dev/null
python scripts/ncu_summary.py $OUT/$2.ncu-rep --json $OUT/$2.summary.json > /dev/null 2>&1
rm -f $OUT/$2.ncu-rep
ls -la $OUT; cat $OUT/$2.summary.json
