#!/bin/bash
# A/B of the SpMM kernels on configs 3 and 4 + the SpMM/GCN/runtime GPU tests.
OUT=gpurun_out/${1:-ab_spmm}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_spmm_gpu.py tests/test_gcn_gpu.py tests/test_runtime_gpu.py -q -p no:cacheprovider > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
for W in c3 c4; do
  timeout 600 python bench.py --workload $W --steps 10 --no-cpu --e2e-steps 1 > $OUT/new_$W.json 2> $OUT/new_$W.err
  LAPIS_B200_SPMM_ROW=1 timeout 600 python bench.py --workload $W --steps 10 --no-cpu --e2e-steps 1 > $OUT/row_$W.json 2> $OUT/row_$W.err
  for V in new row; do python -c "import json;d=json.loads(open('$OUT/${V}_$W.json').read().strip().splitlines()[-1]);print('$V $W', d['value'], d['unit'], d['ms_per_step'], d.get('parity'))" || tail -3 $OUT/${V}_$W.err; done
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_batch -s 2 -c 1 \
    -o $OUT/batch_c3 python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu.log 2>&1; tail -2 $OUT/ncu.log
fi
