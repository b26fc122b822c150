#!/bin/bash
timeout 600 python -m pytest tests/test_spmv_gpu.py tests/test_rowstream_gpu.py -q -x > /tmp/t.txt 2>&1; tail -1 /tmp/t.txt
for W in c1 c5; do
  timeout 900 python bench.py --workload $W --steps 20 --warmup 5 --extra none --no-cpu --e2e-steps 1 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('$W', d['ms_per_step'], d['value'], d['roofline']['frac'], (d.get('exact_mode') or {}).get('value'))" || tail -3 /tmp/b.err
done
