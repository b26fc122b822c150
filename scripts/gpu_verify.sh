#!/bin/bash
# One gpurun call: GPU tests, smoke, the default bench line (c5 + workloads), the reference arm,
# and the c5 launch list (ncu gpu__time_duration, cold-cache, serialised).
# usage (repo root, on the GPU box): bash scripts/gpu_verify.sh [tag]
TAG=${1:-verify}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
fi
timeout 180 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1
timeout 1200 python bench.py ${BENCH_ARGS} > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference ${BENCH_ARGS} > $OUT/bench_reference.json 2> $OUT/bench_reference.err
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 400 \
    --log-file $OUT/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --extra none > /dev/null 2>&1
fi
tail -3 $OUT/pytest_gpu.txt 2>/dev/null; cat $OUT/smoke.txt | tail -3; tail -c 600 $OUT/bench_reference.json
python - "$OUT/bench.json" <<'PY' || tail -20 $OUT/bench.err
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("c5", d["value"], d["unit"], d["ms_per_step"], "frac", d["roofline"]["frac"], "e2e", d["e2e"]["value"],
      "cpu", d["cpu_baseline"]["value"], "parity", d.get("parity"), "clocks", d.get("clocks"))
for k, w in (d.get("workloads") or {}).items():
    print(k, w.get("value"), w.get("unit"), w.get("ms_per_step"), "frac", (w.get("roofline") or {}).get("frac"),
          "e2e", (w.get("e2e") or {}).get("value"), "parity", w.get("parity"))
PY
