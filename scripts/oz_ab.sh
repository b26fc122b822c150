#!/bin/bash
# A/B of the Ozaki GEMM variants (env knobs) on C2 f64 / f32 (mode ozaki)
TAG=${1:-oz}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 300 python -m pytest tests/test_dense_gpu.py -q -x > $OUT/pytest.txt 2>&1; tail -3 $OUT/pytest.txt
for V in "LAPIS_B200_OZAKI_SPLIT=0" "LAPIS_B200_OZAKI_SPLIT=1" ${EXTRA_VARIANTS}; do
  for W in c2f64; do
    env $V timeout 300 python bench.py --workload $W --steps 20 --no-cpu > $OUT/$W.$V.json 2> $OUT/$W.$V.err
    python -c "import json;d=json.load(open('$OUT/$W.$V.json'));print('$W $V',d['value'],d['roofline']['frac'],d['ms_per_step'],d.get('parity'))" || tail -5 $OUT/$W.$V.err
  done
  env $V timeout 300 python bench.py --workload c2f32 --gemm-mode ozaki --steps 20 --no-cpu > $OUT/c2f32oz.$V.json 2> $OUT/c2f32oz.$V.err
  python -c "import json;d=json.load(open('$OUT/c2f32oz.$V.json'));print('c2f32oz $V',d['value'],d['roofline']['frac'],d['ms_per_step'],d.get('parity'))" || tail -5 $OUT/c2f32oz.$V.err
done
if [ -n "$PROF" ]; then
  LAPIS_B200_OZAKI_PROF=1 timeout 300 python bench.py --workload c2f64 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 2>&1 | grep "ozaki prof" | tail -2
fi
