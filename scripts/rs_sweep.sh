#!/bin/bash
OUT=gpurun_out/${1:-rs_sweep}; mkdir -p $OUT
P="timeout 300 python scripts/spmv_variant.py"
for A in "300 27"; do
  $P tree $A
  for r in 1 2; do
  echo -n "v1 "; LAPIS_B200_RS_V1=1 $P exact $A; echo -n "dyn "; $P exact $A; echo -n "static "; LAPIS_B200_RS_STATIC=1 $P exact $A
  done
done 2>&1 | tee $OUT/sweep.txt
for K in "LAPIS_B200_SPMV_KERNEL=rs LAPIS_B200_RS_V1=1" "LAPIS_B200_SPMV_KERNEL=rs"; do
  env $K timeout 600 python bench.py --steps 10 --warmup 3 --extra none --no-cpu --e2e-steps 1 > $OUT/b.json 2> $OUT/b.err
  python - "$OUT/b.json" "$K" <<'PY' || tail -5 $OUT/b.err
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ex = d.get("exact_mode") or {}
print(sys.argv[2], d["value"], d["ms_per_step"], d["roofline"]["frac"], "| exact", ex.get("value"), ex.get("frac"), ex.get("kernel"))
PY
done
