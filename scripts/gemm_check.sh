#!/bin/bash
TAG=${1:-gm}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 300 python -m pytest tests/test_dense_gpu.py -q -x > $OUT/pytest.txt 2>&1; tail -3 $OUT/pytest.txt
for W in c2f32 c2f64; do
  timeout 300 python bench.py --workload $W --steps 10 --cpu-reps 1 > $OUT/$W.json 2> $OUT/$W.err
  python -c "import json;d=json.load(open('$OUT/$W.json'));print('$W',d['value'],d['roofline']['frac'],d['ms_per_step'],d.get('parity'))" || tail -5 $OUT/$W.err
done
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32x3 -s 1 -c 1 \
    -o $OUT/tf32x3 python bench.py --workload c2f32 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_dmma -s 1 -c 1 \
    -o $OUT/dmma python bench.py --workload c2f64 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu2.log 2>&1
tail -1 $OUT/ncu.log $OUT/ncu2.log
fi
