#!/bin/bash
TAG=${1:-r2g}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_spmm_gpu.py tests/test_capi_host.py -m "gpu or not gpu" -q -x > $OUT/pytest.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest.txt
tail -3 $OUT/pytest.txt
for P in 1 0; do for W in c3; do :; done
  LAPIS_BENCH_SPMM_PLAN=$P timeout 900 python bench.py --workload c3 --extra none --no-cpu --e2e-steps 2 > $OUT/bench_c3_p$P.json 2> $OUT/bench_c3_p$P.err
  python - "$OUT/bench_c3_p$P.json" $P <<'PY' || tail -5 $OUT/bench_c3_p$P.err
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("plan" if sys.argv[2] == "1" else "noplan", d["value"], d["unit"], d["ms_per_step"], "frac", d["roofline"]["frac"], d["workload_detail"].get("spmm_plan"))
for k, v in (d.get("kernels") or {}).items(): print("   ", k, v)
PY
done
timeout 900 python bench.py --workload c4 --extra none --no-cpu --e2e-steps 2 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
python -c "import json;d=json.loads(open('$OUT/bench_c4.json').read().strip().splitlines()[-1]);print('c4',d['value'],d['ms_per_step'],d.get('kernels'))" || tail -3 $OUT/bench_c4.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm_batch2" -s 3 -c 1 \
    -o $OUT/full_c3_plan python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --extra none > $OUT/ncu_c3.log 2>&1
tail -1 $OUT/ncu_c3.log
for T in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $T --log-file $OUT/sanitizer_$T.txt python scripts/sanitize.py > $OUT/sanitize_$T.out 2>&1
  echo "$T rc=$?"; tail -2 $OUT/sanitizer_$T.txt; tail -1 $OUT/sanitize_$T.out
done
