#!/bin/bash
LAPIS_B200_SPMV_ROW2=1 timeout 600 python -m pytest tests/test_spmv_gpu.py -q -x > /tmp/t.txt 2>&1; tail -1 /tmp/t.txt
for r in 1 2; do for V in 0 1; do for B in 0 16; do
  LAPIS_B200_SPMV_ROW2=$V LAPIS_B200_SPMV_BLOCKS_PER_SM=$B timeout 600 python bench.py --workload c1 --steps 50 --warmup 5 --extra none --no-cpu --e2e-steps 1 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('row2=$V blocks=$B', d['ms_per_step'], d['value'], d['roofline']['frac'], d['parity']['bitexact_vs_reference'] if 'parity' in d else '')" || tail -3 /tmp/b.err
done; done; done
