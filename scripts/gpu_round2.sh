#!/bin/bash
# benches of every workload + ncu of the two VL=4 SpMV kernels (tree vs exact)
TAG=${1:-r2}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for W in ${WORKLOADS:-c3 c2f32 c2f64}; do
  timeout 900 python bench.py --workload $W --steps 5 --e2e-steps 2 > $OUT/bench_$W.json 2> $OUT/bench_$W.err
  python -c "import json;d=json.load(open('$OUT/bench_$W.json'));print('$W',d['value'],d['unit'],d['roofline']['frac'],d.get('parity'),d.get('cpu_baseline',{}).get('value'))" || tail -5 $OUT/bench_$W.err
done
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_vector -s 3 -c 1 \
    -o $OUT/vec4_tree python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --vl 4 > $OUT/ncu_tree.log 2>&1
LAPIS_B200_SPMV_VL=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_vector -s 3 -c 1 \
    -o $OUT/vec4_exact python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu_exact.log 2>&1
tail -1 $OUT/ncu_tree.log $OUT/ncu_exact.log
fi
