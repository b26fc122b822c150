#!/bin/bash
for U in 16 163; do LAPIS_B200_SPMV_WB_U=$U timeout 300 python scripts/spmv_irregular_probe.py 1; done
for V in "X=0" "LAPIS_B200_SPMM_MB3=1"; do
  env LAPIS_BENCH_SPMM_PLAN=0 $V timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 --extra none --no-cpu --e2e-steps 1 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('noplan $V', d['ms_per_step'], d['value'])" || tail -3 /tmp/b.err
done
