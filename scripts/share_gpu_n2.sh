#!/bin/bash
# correctness run of bench.py's N = 2 path on ONE GPU (both ranks on cuda:0,
# gloo process group): the sharded SpMV / SpMM code paths end to end
OUT=gpurun_out/${1:-n2}; mkdir -p $OUT
for spec in "c5 --problem-size 120" "c1 --problem-size 400" "c3 --problem-size 200000" "c2f64 --problem-size 1024"; do
  set -- $spec; W=$1; shift
  LAPIS_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 2 --workload $W "$@" --steps 3 --warmup 3 \
    --e2e-steps 2 > $OUT/bench_$W.json 2> $OUT/bench_$W.err
  echo "$W rc=$?"; python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d[\"n_gpus\"], d[\"value\"], d[\"unit\"], d.get(\"sharded_parity\"), d[\"config\"].get(\"sharding\"))" $OUT/bench_$W.json; grep -i "error\|Traceback" $OUT/bench_$W.err | head -5
done
