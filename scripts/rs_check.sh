#!/bin/bash
# row-stream SpMV: SpMV / seam GPU tests, the C5 line (exact_mode) and the seam timing
OUT=gpurun_out/${1:-rs_check}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_rowstream_gpu.py tests/test_spmv_gpu.py tests/test_sparse_route.py tests/test_kokkos_b200.py tests/test_configs_gpu.py -q -x > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
tail -2 $OUT/pytest.txt
timeout 600 python bench.py --steps 10 --warmup 3 --extra none --no-cpu --e2e-steps 1 > $OUT/b.json 2> $OUT/b.err
python - "$OUT/b.json" <<'PY' || tail -5 $OUT/b.err
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ("value", "ms_per_step", "exact_mode", "variants", "seam")}, indent=0)[:1500])
print(d["roofline"])
PY
