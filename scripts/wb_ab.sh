#!/bin/bash
# A/B of the SpMV warp-block kernel against the vector kernel (c1, c5)
OUT=gpurun_out/${1:-wb}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_spmv_gpu.py -q -x > $OUT/pytest_spmv.txt 2>&1; echo "rc=$?" >> $OUT/pytest_spmv.txt
for K in wb vec; do
  for W in c1 c5; do
    LAPIS_B200_SPMV_KERNEL=$K timeout 600 python bench.py --workload $W --no-cpu --e2e-steps 3 > $OUT/bench_${W}_$K.json 2> $OUT/bench_${W}_$K.err
  done
done
tail -2 $OUT/pytest_spmv.txt
for f in $OUT/bench_*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], d["roofline"]["frac"], d["roofline"].get("kernel"), d.get("exact_mode", d.get("exact")))
PY
done
