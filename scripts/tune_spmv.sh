#!/bin/bash
# SpMV kernel-shape sweep (LAPIS_B200_SPMV_CFG) on config 5 and config 1.
TAG=${1:-tune}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python -m pytest tests/test_spmv_gpu.py -q -x > $OUT/pytest_spmv.txt 2>&1; tail -2 $OUT/pytest_spmv.txt
for cfg in ${CFGS:-0 1 2 3}; do
  for W in c5 c1; do
    LAPIS_B200_SPMV_CFG=$cfg timeout 300 python bench.py --workload $W --steps 10 --no-cpu --e2e-steps 1 > $OUT/cfg${cfg}_$W.json 2>$OUT/cfg${cfg}_$W.err
    python -c "import json;d=json.load(open('$OUT/cfg${cfg}_$W.json'));print('cfg',$cfg,'$W',d['value'],d['roofline']['frac'],d['ms_per_step'])" || tail -3 $OUT/cfg${cfg}_$W.err
  done
done
