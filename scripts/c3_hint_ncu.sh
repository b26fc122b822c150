#!/bin/bash
# DRAM bytes of the config-3 SpMM batch kernel with and without reuse hints
OUT=gpurun_out/${1:-c3hint_ncu}; mkdir -p $OUT
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum"
for V in "HINT=0" "NOHOT=1 LAPIS_B200_SPMM_HINT_D=8" "HINT_D=8" "NOHOT=1 LAPIS_B200_SPMM_HINT=0"; do
  tag=$(echo $V | tr ' =' '__')
  env LAPIS_B200_SPMM_$V timeout 900 ncu --metrics $M --clock-control none -k regex:spmm_batch2 -s 3 -c 1 --csv \
    python bench.py --workload c3 --steps 1 --warmup 3 --extra none --no-cpu --e2e-steps 1 > $OUT/$tag.csv 2> $OUT/$tag.err
  echo "== $V"; grep -E "dram__|gpu__time|lts__" $OUT/$tag.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
