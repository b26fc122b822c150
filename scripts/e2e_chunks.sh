#!/bin/bash
OUT=gpurun_out/${1:-e2e}; mkdir -p $OUT
for C in 16 64 128; do
  LAPIS_B200_STREAM_CHUNKS=$C timeout 900 python bench.py --steps 3 --warmup 3 --extra none --no-cpu --e2e-steps 5 > $OUT/b.json 2> $OUT/b.err
  python -c "import json;d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]);print('chunks=$C', d['ms_per_step'], d['e2e'])" || tail -3 $OUT/b.err
done
python scripts/link_probe.py 2>&1 | tail -5
