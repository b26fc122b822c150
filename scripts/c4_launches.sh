#!/bin/bash
OUT=gpurun_out/${1:-c4l}; mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -c 60 \
  --log-file $OUT/launches_c4.csv python bench.py --workload c4 --steps 2 --warmup 3 --extra none --no-cpu --e2e-steps 1 > /dev/null 2>&1
python scripts/launch_table.py $OUT/launches_c4.csv
timeout 600 python bench.py --workload c4 --steps 20 --warmup 3 --extra none --no-cpu --e2e-steps 1 > $OUT/b.json 2>$OUT/b.err
python -c "import json;d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['value'], d['roofline'], d.get('kernels'))"
