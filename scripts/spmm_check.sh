#!/bin/bash
timeout 900 python -m pytest tests/test_spmm_gpu.py tests/test_gcn_gpu.py tests/test_configs_gpu.py tests/test_interop_gpu.py tests/test_threads_gpu.py -q -x > /tmp/sp.txt 2>&1; tail -1 /tmp/sp.txt
for P in 1 0; do
  LAPIS_BENCH_SPMM_PLAN=$P timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 --extra none --no-cpu --e2e-steps 1 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('c3 plan=$P', d['ms_per_step'], d['value'])" || tail -3 /tmp/b.err
done
timeout 900 python bench.py --workload c4 --steps 20 --warmup 3 --extra none --no-cpu --e2e-steps 1 > /tmp/b.json 2>/tmp/b.err
python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('c4', d['ms_per_step'], d['value'])" || tail -3 /tmp/b.err
