"""Per-kernel mean launch time from an ncu --metrics gpu__time_duration.sum CSV."""
import csv
import sys
from collections import defaultdict

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi and "lapis" in r[ki]:
            d[r[ki][:95]].append(float(r[vi].replace(",", "")))
    print(path)
    for k, v in d.items():
        print(f"  {len(v):4d} {sum(v) / len(v) / 1e3:10.1f} us  {k}")
