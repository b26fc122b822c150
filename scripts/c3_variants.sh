#!/bin/bash
# config-3 SpMM plan variants: step time and the batch kernel's instruction count / DRAM bytes
OUT=gpurun_out/${1:-c3var}; mkdir -p $OUT
M=smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for V in ${VARIANTS:-"X=0" "LAPIS_B200_SPMM_NOHOT=1" "LAPIS_B200_SPMM_HINT=0" "LAPIS_B200_SPMM_NOHOT=1 LAPIS_B200_SPMM_HINT=0"}; do
  env $V timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 --extra none --no-cpu --e2e-steps 1 > $OUT/b.json 2> $OUT/b.err
  python -c "import json;d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]);print('$V', d['ms_per_step'], d['value'], d['roofline']['frac'])" || tail -3 $OUT/b.err
  env $V timeout 900 ncu --metrics $M --clock-control none -k regex:spmm_batch -s 3 -c 1 --csv python bench.py --workload c3 --steps 1 --warmup 3 --extra none --no-cpu --e2e-steps 1 2>/dev/null > $OUT/n.csv
  python - "$OUT/n.csv" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
i = [k for k, r in enumerate(rows) if 'Kernel Name' in r][0]
h, rows = rows[i], rows[i + 1:]
print("   ", rows[0][h.index('Kernel Name')][:60], {r[h.index('Metric Name')]: r[h.index('Metric Value')] for r in rows})
PY
done
