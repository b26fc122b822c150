#!/bin/bash
OUT=gpurun_out/${1:-ring}; mkdir -p $OUT
LAPIS_B200_SPMM_RING=1 timeout 900 python -m pytest tests/test_spmm_gpu.py tests/test_gcn_gpu.py tests/test_configs_gpu.py -q -x > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
tail -n 2 $OUT/pytest.txt; grep -E "^E  |FAILED" $OUT/pytest.txt | head -5
for W in c3 c4; do for R in 0 1; do
  LAPIS_B200_SPMM_RING=$R timeout 900 python bench.py --workload $W --steps 10 --warmup 3 --extra none --no-cpu --e2e-steps 1 > $OUT/b.json 2> $OUT/b.err
  python -c "import json;d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]);print('$W ring=$R', d['ms_per_step'], d['value'], d['roofline']['frac'])" || tail -3 $OUT/b.err
done; done
