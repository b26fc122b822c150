#!/bin/bash
# DRAM bytes per launch of each workload's dominant kernel (ncu, one launch)
OUT=gpurun_out/${1:-traffic}; mkdir -p $OUT
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
run() {  # workload regex
  timeout 900 ncu --metrics $M --clock-control none -k regex:"$2" -s 3 -c 1 --csv python bench.py --workload $1 --steps 1 --warmup 3 --extra none --no-cpu --e2e-steps 1 2>/dev/null > $OUT/$1.csv
  python - "$OUT/$1.csv" "$1" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
i = [k for k, r in enumerate(rows) if 'Kernel Name' in r][0]
h, rows = rows[i], rows[i + 1:]
d = {r[h.index('Metric Name')]: float(r[h.index('Metric Value')]) for r in rows}
print(sys.argv[2], rows[0][h.index('Kernel Name')][:90], d)
PY
}
[ -n "$ONLY_SPMV" ] || run c2f32 gemm_ozaki_2p
[ -n "$ONLY_SPMV" ] || run c2f64 gemm_ozaki_2p
[ -n "$ONLY_SPMV" ] || run c3 spmm_batch2
[ -n "$ONLY_SPMV" ] || run c4 spmm_batch2
run c1 spmv_vector
run c5 spmv_rowstream
