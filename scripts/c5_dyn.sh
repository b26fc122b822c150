#!/bin/bash
# row-stream tile split: static share vs counter share (LAPIS_B200_RS_DYN %),
# C5 exact per-launch times + the per-CTA end-time spread
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_rowstream_gpu.py -x -q 2>&1 | tail -3
for D in 0 10 15 25 50 100; do
  echo "== RS_DYN=$D"
  LAPIS_B200_RS_DYN=$D timeout 300 python scripts/rs_times.py 2>&1 | tail -6
done
