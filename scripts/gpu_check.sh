#!/bin/bash
# One gpurun call: GPU tests, smoke, benches, ncu launch list + one full capture.
# usage (from the repo root, on the GPU box): bash scripts/gpu_check.sh [tag]
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi.txt
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
for W in ${WORKLOADS:-c5 c1}; do
  timeout 900 python bench.py --workload $W > $OUT/bench_$W.json 2> $OUT/bench_$W.err
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_tile -s 4 -c 1 \
    -o $OUT/spmv_tile_c5 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu_full.log 2>&1
fi
tail -3 $OUT/pytest_gpu.txt; cat $OUT/smoke.txt
for W in ${WORKLOADS:-c5 c1}; do cat $OUT/bench_$W.json; tail -3 $OUT/bench_$W.err; done
