#!/bin/bash
OUT=gpurun_out/${1:-c1vl}; mkdir -p $OUT
for v in 1 2 4 8; do
  LAPIS_B200_SPMV_VL=$v timeout 300 python bench.py --workload c1 --steps 200 --no-cpu --e2e-steps 1 > $OUT/c1_vl$v.json 2>$OUT/c1_vl$v.err
  python -c "import json;d=json.loads(open('$OUT/c1_vl$v.json').read().strip().splitlines()[-1]);print('VL',$v,d['value'],d['ms_per_step'],d['roofline']['kernel'],d['exact_mode']['value'])" || tail -3 $OUT/c1_vl$v.err
done
