#!/bin/bash
TAG=${1:-r2j}; OUT=gpurun_out/$TAG; mkdir -p $OUT
bash scripts/gpu_plan_ab.sh $TAG/plan 2>&1 | grep -v "^$"
for V in 0 1; do
  LAPIS_B200_NO_SIDE_STREAM=$V timeout 600 python bench.py --workload c4 --extra none --no-cpu --e2e-steps 1 > $OUT/c4_ns$V.json 2> $OUT/c4_ns$V.err
  python -c "import json;d=json.loads(open('$OUT/c4_ns$V.json').read().strip().splitlines()[-1]);print('c4 noside=$V',d['ms_per_step'])" || tail -3 $OUT/c4_ns$V.err
done
timeout 600 python bench.py --workload c1 --extra none --no-cpu --e2e-steps 1 > $OUT/c1.json 2> $OUT/c1.err
python -c "import json;d=json.loads(open('$OUT/c1.json').read().strip().splitlines()[-1]);r=d['roofline'];print('c1',d['value'],d['ms_per_step'],r['frac'],r.get('launch_floor_us'),r.get('frac_floor_corrected'), d.get('exact_mode'))" || tail -3 $OUT/c1.err
