#!/bin/bash
# round-2 check: new parity tests, the default bench line (headline + workloads), reference arm
TAG=${1:-r2b}; OUT=gpurun_out/$TAG; mkdir -p $OUT
lscpu > $OUT/lscpu.txt 2>&1; free -g > $OUT/free.txt
timeout 1200 python -m pytest ${TESTS:-tests/test_configs_gpu.py tests/test_synth_inputs.py tests/test_spmv_gpu.py tests/test_spmm_gpu.py} -m gpu -q -x > $OUT/pytest.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest.txt
tail -5 $OUT/pytest.txt
timeout 1200 python bench.py ${BENCH_ARGS} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
tail -c 3000 $OUT/bench.json; tail -5 $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?"
tail -c 1500 $OUT/ref.json; tail -3 $OUT/ref.err
