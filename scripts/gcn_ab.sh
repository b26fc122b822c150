#!/bin/bash
OUT=gpurun_out/${1:-gcn}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gcn_gpu.py tests/test_runtime_gpu.py -q -x > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
tail -3 $OUT/pytest.txt
WORKLOADS="c1 c4" bash scripts/quick.sh ${1:-gcn}
LAPIS_B200_GCN_UNFUSED=1 timeout 600 python bench.py --workload c4 --no-cpu > $OUT/bench_c4_unfused.json 2>$OUT/bench_c4_unfused.err
python -c "
import json; d=json.loads(open('$OUT/bench_c4_unfused.json').read().strip().splitlines()[-1]); print('unfused', d['value'], d['ms_per_step'], d.get('kernels'))"
python -c "
import json; d=json.loads(open('$OUT/bench_c4.json').read().strip().splitlines()[-1]); print('fused', d['value'], d['ms_per_step'], d.get('kernels'))
d=json.loads(open('$OUT/bench_c1.json').read().strip().splitlines()[-1]); print('c1', d['value'], d['ms_per_step'], d.get('kernels'), d['config'])"
