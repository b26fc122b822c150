#!/bin/bash
OUT=gpurun_out/${1:-c4var}; mkdir -p $OUT
M=smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct
for V in ${VARIANTS:-"X=0"}; do
  env $V timeout 900 python bench.py --workload c4 --steps 20 --warmup 3 --extra none --no-cpu --e2e-steps 1 > $OUT/b.json 2> $OUT/b.err
  python -c "import json;d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]);print('$V', d['ms_per_step'], d['value'], d['roofline']['frac'])" || tail -3 $OUT/b.err
  env $V timeout 900 ncu --metrics $M --clock-control none -k regex:"spmm_batch|gcn_dense|seq_long" -s 3 -c 3 --csv python bench.py --workload c4 --steps 1 --warmup 3 --extra none --no-cpu --e2e-steps 1 2>/dev/null > $OUT/n.csv
  python - "$OUT/n.csv" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
i = [k for k, r in enumerate(rows) if 'Kernel Name' in r][0]
h, rows = rows[i], rows[i + 1:]
d = collections.OrderedDict()
for r in rows:
    d.setdefault(r[h.index('Kernel Name')][:40], {})[r[h.index('Metric Name')].split('.')[0]] = r[h.index('Metric Value')]
for k, v in d.items():
    print("   ", k, v)
PY
done
