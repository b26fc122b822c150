#!/bin/bash
timeout 600 python -m pytest tests/test_rowstream_gpu.py tests/test_spmv_gpu.py -q -x > /tmp/t.txt 2>&1; tail -1 /tmp/t.txt
P="timeout 300 python scripts/spmv_variant.py"
for n in 300 585; do $P exact $n; LAPIS_B200_RS_STATIC=1 $P exact $n; done
