#!/bin/bash
# ncu full capture of the SpMV tile kernel (config 5) for one kernel shape + vector-kernel timings
TAG=${1:-prof}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for vl in 32 16 8; do
  timeout 300 python bench.py --steps 10 --no-cpu --e2e-steps 1 --vl $vl > $OUT/vl$vl.json 2>$OUT/vl$vl.err
  python -c "import json;d=json.load(open('$OUT/vl$vl.json'));print('vl',$vl,d['value'],d['roofline']['frac'])" || tail -3 $OUT/vl$vl.err
done
LAPIS_B200_SPMV_CFG=${CFG:-2} timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_tile -s 4 -c 1 \
    -o $OUT/spmv_tile_c5 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu_full.log 2>&1
tail -2 $OUT/ncu_full.log
