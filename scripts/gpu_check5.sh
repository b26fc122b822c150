#!/bin/bash
TAG=${1:-r2f}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_spmm_gpu.py tests/test_gcn_gpu.py tests/test_spmv_gpu.py tests/test_configs_gpu.py -m gpu -q -x > $OUT/pytest.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest.txt
tail -3 $OUT/pytest.txt
for W in c4 c3; do
  for V in 0 1; do
  LAPIS_B200_SPMM_V1=$V timeout 900 python bench.py --workload $W --extra none --no-cpu --e2e-steps 2 > $OUT/bench_${W}_v$V.json 2> $OUT/bench_${W}_v$V.err
  python - "$OUT/bench_${W}_v$V.json" $V <<'PY' || tail -5 $OUT/bench_${W}_v$V.err
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("v1" if sys.argv[2] == "1" else "v2", d["config"]["workload"][:40], d["value"], d["unit"], d["ms_per_step"], "frac", d["roofline"]["frac"])
for k, v in (d.get("kernels") or {}).items(): print("   ", k, v)
PY
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm_batch2" -s 3 -c 1 \
    -o $OUT/full_c4 python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --extra none > $OUT/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm_batch2" -s 3 -c 1 \
    -o $OUT/full_c3 python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --extra none > $OUT/ncu_c3.log 2>&1
tail -1 $OUT/ncu_c4.log $OUT/ncu_c3.log
