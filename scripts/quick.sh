#!/bin/bash
# quick GPU check: selected tests + selected bench workloads
# usage: TESTS="tests/x.py" WORKLOADS="c1 c3" bash scripts/quick.sh tag
OUT=gpurun_out/${1:-quick}; mkdir -p $OUT
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest $TESTS -q -x > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
  tail -3 $OUT/pytest.txt
fi
for W in $WORKLOADS; do
  timeout 900 python bench.py --workload $W $BENCH_ARGS > $OUT/bench_$W.json 2> $OUT/bench_$W.err
  python - "$OUT/bench_$W.json" <<'PY' || tail -5 $OUT/bench_$W.err
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["config"]["workload"], d["value"], d["unit"], d["ms_per_step"], "frac", d["roofline"]["frac"],
      "e2e", d["e2e"]["value"], "cpu", d.get("cpu_baseline", {}).get("value"), "parity", d.get("parity"),
      d.get("exact_mode"), d.get("variants"), d["config"].get("l2"))
PY
done
