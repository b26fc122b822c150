#!/bin/bash
TAG=${1:-vl}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for W in c5 c1; do for vl in ${VLS:-1 2 4 8 16}; do
  timeout 300 python bench.py --workload $W --steps 10 --no-cpu --e2e-steps 1 --vl $vl > $OUT/${W}_vl$vl.json 2>$OUT/${W}_vl$vl.err
  python -c "import json;d=json.load(open('$OUT/${W}_vl$vl.json'));print('$W vl',$vl,d['value'],d['roofline']['frac'])" || tail -3 $OUT/${W}_vl$vl.err
done; done
