#!/bin/bash
TAG=${1:-tx}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python -m pytest tests/test_spmv_gpu.py -q -x > $OUT/pytest_spmv.txt 2>&1; tail -2 $OUT/pytest_spmv.txt
for W in c5 c1; do for vl in auto 2 4 8; do
  if [ $vl = auto ]; then unset LAPIS_B200_SPMV_VL; else export LAPIS_B200_SPMV_VL=$vl; fi
  timeout 300 python bench.py --workload $W --steps 10 --no-cpu --e2e-steps 1 > $OUT/${W}_x$vl.json 2>$OUT/${W}_x$vl.err
  python -c "import json;d=json.load(open('$OUT/${W}_x$vl.json'));print('$W exact vl',"'"'$vl'"'",d['value'],d['roofline']['frac'],d['roofline']['kernel'])" || tail -3 $OUT/${W}_x$vl.err
done; unset LAPIS_B200_SPMV_VL
for vl in 2 4 8; do
  timeout 300 python bench.py --workload $W --steps 10 --no-cpu --e2e-steps 1 --vl $vl > $OUT/${W}_t$vl.json 2>$OUT/${W}_t$vl.err
  python -c "import json;d=json.load(open('$OUT/${W}_t$vl.json'));print('$W tree vl',$vl,d['value'],d['roofline']['frac'])" || tail -3 $OUT/${W}_t$vl.err
done; done
