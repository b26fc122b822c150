#!/bin/bash
OUT=gpurun_out/${1:-grid}; mkdir -p $OUT
for b in ${BPS:-8 16 32 64 256}; do
  LAPIS_B200_SPMV_BLOCKS_PER_SM=$b timeout 300 python bench.py --workload c5 --steps 10 --no-cpu --e2e-steps 1 > $OUT/c5_b$b.json 2>$OUT/c5_b$b.err
  python -c "import json;d=json.loads(open('$OUT/c5_b$b.json').read().strip().splitlines()[-1]);print('blocks/SM',$b,d['value'],d['ms_per_step'],d['roofline']['frac'])" || tail -3 $OUT/c5_b$b.err
done
