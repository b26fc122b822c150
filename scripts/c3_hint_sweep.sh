#!/bin/bash
# SpMM plan reuse hints: SpMM GPU tests, then config-3 lines over hint variants
OUT=gpurun_out/${1:-c3hint}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_spmm_gpu.py -q -x > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
tail -2 $OUT/pytest.txt
run() {
  local tag=$1; shift
  env "$@" timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 --extra none --no-cpu --e2e-steps 1 > $OUT/b_$tag.json 2> $OUT/b_$tag.err
  python - "$OUT/b_$tag.json" "$tag" <<'PY' || tail -5 $OUT/b_$tag.err
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], d["value"], d["ms_per_step"], d["roofline"]["frac"], d["workload_detail"].get("spmm_plan"))
PY
}
run nohint LAPIS_B200_SPMM_HINT=0
for F in 0 1 2; do for D in 8 4; do run F${F}_D$D LAPIS_B200_SPMM_FARPF=$F LAPIS_B200_SPMM_HINT_D=$D; done; done
run nohot_F0_D8 LAPIS_B200_SPMM_NOHOT=1 LAPIS_B200_SPMM_FARPF=0 LAPIS_B200_SPMM_HINT_D=8
run nohot_F1_D8 LAPIS_B200_SPMM_NOHOT=1 LAPIS_B200_SPMM_FARPF=1 LAPIS_B200_SPMM_HINT_D=8
