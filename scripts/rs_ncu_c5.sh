#!/bin/bash
OUT=gpurun_out/${1:-rsc5}; mkdir -p $OUT
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active"
for n in 300 585; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:spmv_rowstream -s 3 -c 1 --csv python scripts/spmv_variant.py exact $n > $OUT/rs_$n.csv 2>&1
  echo "== rowstream n=$n"; grep -E "dram__|gpu__time|lts__|warps" $OUT/rs_$n.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
  timeout 900 ncu --metrics $M --clock-control none -k regex:spmv_vector -s 3 -c 1 --csv python scripts/spmv_variant.py tree $n > $OUT/vec_$n.csv 2>&1
  echo "== vector tree n=$n"; grep -E "dram__|gpu__time|lts__|warps" $OUT/vec_$n.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
