#!/bin/bash
# SpMM plan A/B on config 3: hot-row budget x persisting window
TAG=${1:-r2i}; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() {  # name env...
  env "${@:2}" timeout 600 python bench.py --workload c3 --extra none --no-cpu --e2e-steps 1 --steps 10 > $OUT/$1.json 2> $OUT/$1.err
  python -c "import json;d=json.loads(open('$OUT/$1.json').read().strip().splitlines()[-1]);print('$1',d['ms_per_step'],d['workload_detail'].get('spmm_plan'))" || tail -3 $OUT/$1.err
}
run noplan LAPIS_BENCH_SPMM_PLAN=0
for MB in 8 12 16 24; do
  run hot${MB}_win LAPIS_BENCH_SPMM_HOT_MB=$MB
  run hot${MB}_nowin LAPIS_BENCH_SPMM_HOT_MB=$MB LAPIS_B200_SPMM_WINDOW=0
done
run noplan_v1 LAPIS_BENCH_SPMM_PLAN=0 LAPIS_B200_SPMM_V1=1
run noplan_again LAPIS_BENCH_SPMM_PLAN=0
