#!/bin/bash
OUT=gpurun_out/${1:-c5ex}; mkdir -p $OUT
for v in 1 2 4 8; do
  LAPIS_B200_SPMV_VL=$v timeout 400 python bench.py --workload c5 --steps 5 --no-cpu --e2e-steps 1 > $OUT/c5_vl$v.json 2>$OUT/c5_vl$v.err
  python -c "import json;d=json.loads(open('$OUT/c5_vl$v.json').read().strip().splitlines()[-1]);print('VL',$v,'tree',d['value'],'exact',d['exact_mode']['value'])" || tail -3 $OUT/c5_vl$v.err
done
