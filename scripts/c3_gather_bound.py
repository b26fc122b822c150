"""Cache-optimal DRAM traffic of config 3's X-row gathers.

Builds the config-3 power-law matrix (synth_inputs.PowerLawSpec(10M, seed 1),
the bench's matrix), writes its colind stream in CSR order and runs
scripts/cache_sim.c on it for caches of 32 / 64 / 96 / 126 MB of X rows
(512 B per row: K = 64 fp64): Belady's optimum, LRU, and pinning the most
referenced rows.  The minimum DRAM bytes per SpMM launch for a given cache
size is then  misses * 512 + structure (nnz * 12 + (N + 1) * 8) + Y (N * 512).
Output: profiles/c3_gather_bound.json.
    python scripts/c3_gather_bound.py
"""
import json
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import synth_inputs as S  # noqa: E402

N, K = 10_000_000, 64
ROW = K * 8
t0 = time.time()
spec = S.PowerLawSpec(N, seed=1)
rowptr, colind = S.powerlaw_structure_host(spec)
nnz = int(rowptr[-1])
colind.astype(np.int32).tofile("/tmp/c3_colind.bin")
sim = "/tmp/cache_sim"
subprocess.run(["gcc", "-O2", "-o", sim, str(ROOT / "scripts" / "cache_sim.c")], check=True)
caps = {"32MB": 32 << 20, "64MB": 64 << 20, "96MB": 96 << 20, "126MB": 126 << 20}
rows_of = {k: v // ROW for k, v in caps.items()}
out = subprocess.run([sim, "/tmp/c3_colind.bin", str(N), *map(str, rows_of.values())],
                     check=True, capture_output=True, text=True).stdout
res = json.loads(out)
structure = nnz * 12 + (N + 1) * 8
ybytes = N * ROW
table = {}
for (name, _), r in zip(caps.items(), res["results"]):
    table[name] = {k: {"misses": r[f"miss_{k}"],
                       "x_bytes": r[f"miss_{k}"] * ROW,
                       "dram_bytes_per_launch": r[f"miss_{k}"] * ROW + structure + ybytes}
                   for k in ("opt", "lru", "pin")}
    table[name]["cap_rows"] = r["cap_rows"]
doc = {"workload": "config 3 SpMM, K = 64 fp64, synth_inputs.PowerLawSpec(10M, seed 1)",
       "nnz": nnz, "gathers": res["accesses"], "distinct_columns": res["distinct"],
       "no_reuse_x_bytes": res["accesses"] * ROW, "compulsory_x_bytes": res["distinct"] * ROW,
       "structure_bytes": structure, "y_bytes": ybytes,
       "algorithmic_bytes": nnz * 12 + (N + 1) * 8 + N * ROW * 2,
       "order": "gathers in CSR order (rows ascending, columns ascending in a row)",
       "caches": table, "seconds": round(time.time() - t0, 1),
       "method": "scripts/cache_sim.c: Belady OPT (max-heap on next use), LRU, static pin of the "
                 "most referenced rows"}
(ROOT / "profiles" / "c3_gather_bound.json").write_text(json.dumps(doc, indent=1) + "\n")
print(json.dumps(doc, indent=1))
