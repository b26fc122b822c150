#!/bin/bash
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_mio_throttle,smsp__pcsamp_warps_issue_stalled_short_scoreboard,smsp__pcsamp_warps_issue_stalled_lg_throttle
for P in 1 0; do
echo "policy=$P"
LAPIS_B200_SPMV_WB_POLICY=$P ncu --metrics $M --clock-control none -k regex:warpblock -s 3 -c 1 --csv python scripts/spmv_irregular_probe.py $P 2>/dev/null > /tmp/pl.csv
python - <<'PY'
import csv
rows = [r for r in csv.reader(open('/tmp/pl.csv')) if len(r) > 5]
h = rows[0]
for r in rows[1:]:
    print(r[h.index('Metric Name')], r[h.index('Metric Unit')], r[h.index('Metric Value')])
PY
done
