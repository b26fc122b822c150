#!/bin/bash
# exact-SpMV batch fold + GCN dense v2 + SpMM fp32 batch profile
TAG=${1:-r2e}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_spmv_gpu.py tests/test_gcn_gpu.py -m gpu -q -x > $OUT/pytest.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest.txt
tail -3 $OUT/pytest.txt
for W in c4 c1 c5; do
  timeout 900 python bench.py --workload $W --extra none --no-cpu --e2e-steps 2 > $OUT/bench_$W.json 2> $OUT/bench_$W.err
  python - "$OUT/bench_$W.json" <<'PY' || tail -5 $OUT/bench_$W.err
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["config"]["workload"], d["value"], d["unit"], d["ms_per_step"], "frac", d["roofline"]["frac"], "exact", d.get("exact_mode"))
print(" launches", d.get("gpu_launches"), d.get("gpu_launches_source"))
for k, v in (d.get("kernels") or {}).items(): print("   ", k, v)
PY
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c4.csv python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --extra none > /dev/null 2>&1
python scripts/launch_table.py $OUT/launches_c4.csv | tail -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm_batch_kernel|gcn_dense" -s 6 -c 2 \
    -o $OUT/full_c4 python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --extra none > $OUT/ncu_full.log 2>&1
tail -2 $OUT/ncu_full.log
