#!/bin/bash
# ncu --set full of one kernel (regex $1) in workload $2; writes gpurun_out/$3/
OUT=gpurun_out/$3; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${SKIP:-3} -c 1 \
  -o $OUT/full_$2 python bench.py --workload $2 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu_$2.log 2>&1
ncu -i $OUT/full_$2.ncu-rep --page raw --csv > $OUT/raw_$2.csv 2>/dev/null
python - $OUT/raw_$2.csv <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "l1tex__t_sector_hit_rate.pct",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
for w in want:
    if w in h:
        i = h.index(w); print(w, v[i], u[i])
PY
