#!/bin/bash
# warp-block SpMV on the config-3 power-law matrix: blocks per counter claim (LAPIS_B200_WB_RUN)
for r in 1 2; do for R in 1 2 4 8; do
  LAPIS_B200_WB_RUN=$R timeout 300 python scripts/spmv_irregular_probe.py 1 2>&1 | sed "s/^/run=$R /" | tail -1
done; done
