#!/bin/bash
for r in 1 2; do for B in 0 1024; do
  LAPIS_B200_SPMV_BLOCKS_PER_SM=$B timeout 600 python bench.py --workload c1 --steps 50 --warmup 5 --extra none --no-cpu --e2e-steps 1 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('blocks/SM env=$B', d['ms_per_step'], d['value'], d['roofline']['frac'])" || tail -3 /tmp/b.err
done; done
