#!/bin/bash
# A/B: config-1 timed steps replaying one graph per step vs one graph of all
# rotation copies per len(rot) steps (LAPIS_B200_BENCH_GROUP)
mkdir -p gpurun_out
for r in 1 2; do for G in 0 1; do for K in 200 203; do
  LAPIS_B200_BENCH_GROUP=$G timeout 600 python bench.py --workload c1 --steps $K --warmup 5 --extra none --no-cpu --e2e-steps 1 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('group=$G K=$K', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline'].get('launch_floor_us'), d.get('parity'), d['config'].get('launch', '')[:50])" || tail -3 /tmp/b.err
done; done; done 2>&1 | tee gpurun_out/c1_group.txt
