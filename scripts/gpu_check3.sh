#!/bin/bash
# GCN tensor-core stage + census + c3/c4 launch lists and the gcn_dense ncu capture
TAG=${1:-r2c}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest ${TESTS:-tests/test_gcn_gpu.py tests/test_spmm_gpu.py} -m gpu -q -x > $OUT/pytest.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest.txt
tail -5 $OUT/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -2 $OUT/smoke.txt
for W in ${WORKLOADS:-c4 c3}; do
  timeout 900 python bench.py --workload $W --extra none ${BENCH_ARGS} > $OUT/bench_$W.json 2> $OUT/bench_$W.err
  python - "$OUT/bench_$W.json" <<'PY' || tail -5 $OUT/bench_$W.err
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["config"]["workload"], d["value"], d["unit"], d["ms_per_step"], "frac", d["roofline"]["frac"], "parity", d.get("parity"))
print(" launches", d.get("gpu_launches"), d.get("gpu_launches_source"))
for k, v in (d.get("kernels") or {}).items(): print("   ", k, v)
PY
done
if [ -n "$NCU" ]; then
  for W in ${NCU_WORKLOADS:-c4 c3}; do
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --extra none > /dev/null 2>&1
    python scripts/launch_table.py $OUT/launches_$W.csv 2>/dev/null | tail -15
  done
fi
if [ -n "$NCU_FULL" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_FULL" -s ${NCU_SKIP:-3} -c 1 \
    -o $OUT/full_${NCU_W:-c4} python bench.py --workload ${NCU_W:-c4} --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --extra none > $OUT/ncu_full.log 2>&1
  tail -3 $OUT/ncu_full.log
fi
