#!/bin/bash
OUT=gpurun_out/${1:-tf32raw}; mkdir -p $OUT
timeout 300 python scripts/tf32_rawhi_check.py
timeout 900 python -m pytest tests/test_dense_gpu.py tests/test_configs_gpu.py tests/test_gcn_gpu.py -q -x > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
tail -n 2 $OUT/pytest.txt
for R in 1 0; do
  LAPIS_B200_TF32_RAW=$R timeout 600 python bench.py --workload c2f32 --steps 20 --warmup 3 --extra none --no-cpu --e2e-steps 1 > $OUT/b.json 2> $OUT/b.err
  python -c "import json;d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]);print('raw=$R', d['ms_per_step'], d['value'], d['roofline']['frac'])" || tail -3 $OUT/b.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"tf32|split" -c 24 python bench.py --workload c2f32 --steps 2 --warmup 3 --extra none --no-cpu --e2e-steps 1 2>/dev/null | grep -E "gpu__time" | awk -F'","' '{print $5, $NF}' | cut -c1-40,100- | sort | uniq -c | head
