#!/bin/bash
OUT=gpurun_out/${1:-u16}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_spmm_gpu.py tests/test_gcn_gpu.py -q -x > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
LAPIS_B200_SPMM_U=32 timeout 900 python -m pytest tests/test_spmm_gpu.py tests/test_gcn_gpu.py -q -x > $OUT/pytest32.txt 2>&1; echo "rc=$?" >> $OUT/pytest32.txt
tail -1 $OUT/pytest.txt $OUT/pytest32.txt
for W in c4; do for U in 8 16 32 -1; do
  LAPIS_B200_SPMM_U=$U timeout 900 python bench.py --workload $W --steps 20 --warmup 3 --extra none --no-cpu --e2e-steps 1 > $OUT/b.json 2> $OUT/b.err
  python -c "import json;d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]);print('$W U=$U', d['ms_per_step'], d['value'], d['roofline']['frac'])" || tail -3 $OUT/b.err
done; done
