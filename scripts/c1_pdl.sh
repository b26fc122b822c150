#!/bin/bash
# A/B: config-1 SpMV launched with programmatic dependent launch (LAPIS_B200_PDL)
mkdir -p gpurun_out
for r in 1 2 3; do for P in 0 1; do
  LAPIS_B200_PDL=$P timeout 600 python bench.py --workload c1 --steps 200 --warmup 5 --extra none --no-cpu --e2e-steps 1 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('pdl=$P', d['ms_per_step'], d['value'], d['roofline']['frac'])" || tail -3 /tmp/b.err
done; done 2>&1 | tee gpurun_out/c1_pdl.txt
LAPIS_B200_PDL=1 timeout 600 python -m pytest tests/test_spmv_gpu.py tests/test_configs_gpu.py -q -x 2>&1 | tail -2
