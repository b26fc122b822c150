#!/bin/bash
# One gpurun call: GPU tests, smoke, every workload's bench line, the c5 launch list
# and (NCU=1) one full ncu capture of the SpMM kernel on config 3.
# usage (repo root, on the GPU box): bash scripts/gpu_full.sh [tag]
TAG=${1:-full}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi.txt
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
for W in ${WORKLOADS:-c5 c1 c3 c4 c2f32 c2f64 gemv}; do
  timeout 900 python bench.py --workload $W ${BENCH_ARGS} > $OUT/bench_$W.json 2> $OUT/bench_$W.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
if [ -n "$NCU" ]; then
  for W in ${NCU_WORKLOADS:-c3 c4}; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
  done
  if [ -n "$NCU_FULL" ]; then
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_FULL" -s ${NCU_SKIP:-3} -c 1 \
      -o $OUT/full_${NCU_W:-c3} python bench.py --workload ${NCU_W:-c3} --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu_full.log 2>&1
  fi
fi
tail -3 $OUT/pytest_gpu.txt; cat $OUT/smoke.txt; tail -c 400 $OUT/bench_reference.json
for W in ${WORKLOADS:-c5 c1 c3 c4 c2f32 c2f64 gemv}; do
  python - "$OUT/bench_$W.json" <<'PY' || tail -5 $OUT/bench_$W.err
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["config"]["workload"], d["value"], d["unit"], "frac", d["roofline"]["frac"],
      "e2e", d["e2e"]["value"], "cpu", d["cpu_baseline"]["value"], "parity", d.get("parity"))
PY
done
