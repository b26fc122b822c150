#!/usr/bin/env python
"""Summarise an ncu report (.ncu-rep) into the numbers the roofline needs.

    python scripts/ncu_summary.py <report.ncu-rep> [--algorithmic-bytes B] [--json out.json]

Prints duration, DRAM bytes read / written (the `traffic` of bench.py's
roofline object), achieved DRAM throughput, warps active, issue activity, the
tensor-pipe activity and the top warp-stall reasons, plus the SASS mnemonics
that prove which hardware path ran (UTC*MMA = tcgen05.mma, UTMALDG = TMA,
LDTM = tcgen05.ld, DMMA = fp64 tensor).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__warps_active.avg.per_cycle_active": "warps_active_per_sm",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1,
              "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def ncu(*args) -> str:
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--algorithmic-bytes", type=float, default=None)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    rows = list(csv.reader(io.StringIO(ncu("-i", a.report, "--page", "raw", "--csv"))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
    for k, name in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            v = vals[i].replace(",", "")
            try:
                x = float(v) * UNIT_SCALE.get(units[i], 1)
            except ValueError:
                continue
            out[name] = x
    stalls = {}
    for i, h in enumerate(hdr):
        m = re.fullmatch(r"smsp__pcsamp_warps_issue_stalled_([a-z_]+)", h)
        if m and not m.group(1).endswith("not_issued"):
            try:
                stalls[m.group(1)] = float(vals[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    out["top_stalls_pct"] = {k: round(100 * v / tot, 1)
                             for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
    if "duration" in out and "dram_read" in out:
        out["dram_bytes_per_launch"] = out["dram_read"] + out.get("dram_write", 0.0)
        out["dram_gbs"] = out["dram_bytes_per_launch"] / out["duration"] / 1e9
    if a.algorithmic_bytes:
        out["algorithmic_bytes"] = a.algorithmic_bytes
        out["traffic_over_algorithmic"] = out.get("dram_bytes_per_launch", 0) / a.algorithmic_bytes
    try:
        src = ncu("-i", a.report, "--page", "source", "--csv", "--print-source=sass")
        mnems = {}
        for m in re.finditer(r"\b(UTC[A-Z]*MMA|UTMALDG|UTMASTG|UBLKCP|LDTM|STTM|DMMA|HMMA|LDGSTS)\b", src):
            mnems[m.group(1)] = mnems.get(m.group(1), 0) + 1
        out["sass_evidence"] = mnems
    except subprocess.CalledProcessError:
        pass
    text = json.dumps(out, indent=1)
    print(text)
    if a.json:
        with open(a.json, "w") as f:
            f.write(text + "\n")


if __name__ == "__main__":
    sys.exit(main())
