#!/bin/bash
# SpMM/GCN tests, then per-kernel launch times + bench lines for configs 3 and 4.
OUT=gpurun_out/${1:-spl}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gcn_gpu.py tests/test_spmm_gpu.py tests/test_runtime_gpu.py -q -p no:cacheprovider 2>&1 | tail -1
for W in ${WORKLOADS:-c3 c4}; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
  python bench.py --workload $W --steps 10 --e2e-steps 1 2>/dev/null | tail -1 > $OUT/bench_$W.json
done
