#!/bin/bash
P="timeout 300 python scripts/spmv_variant.py"
for n in 585 300 585; do $P tree $n; $P exact $n; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
