#!/bin/bash
# A/B of prebuilt libraries in ablib/*.so (each copied over the in-tree lib) on
# the workloads in $WORKLOADS, alternating twice to cancel box drift
TAG=${1:-ab}; OUT=gpurun_out/$TAG; mkdir -p $OUT
LIB=paper_2509_25605_b200/lib/liblapis_b200.so
cp $LIB $OUT/.keep.so
for rep in 1 2; do
  for L in ablib/*.so; do
    cp $L $LIB
    n=$(basename $L .so)
    for W in ${WORKLOADS:-c2f64}; do
      env $ENVV timeout 300 python bench.py --workload $W --steps 20 --no-cpu ${BENCH_ARGS} > $OUT/$W.$n.$rep.json 2> $OUT/$W.$n.$rep.err
      python -c "import json;d=json.load(open('$OUT/$W.$n.$rep.json'));print('$W $n $rep',d['value'],d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'])" || tail -3 $OUT/$W.$n.$rep.err
    done
  done
done
cp $OUT/.keep.so $LIB; rm $OUT/.keep.so
