#!/usr/bin/env python3
"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) as a
per-kernel table: launches, total ms, share.  usage: launch_table.py <csv> [cmd]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
tot = defaultdict(lambda: [0, 0.0])
for r in csv.DictReader(lines):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = r["Kernel Name"].split("(")[0][:44]
    v = float(r["Metric Value"].replace(",", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
             "nsecond": 1e-6}.get(r["Metric Unit"], 1e-6)
    tot[k][0] += 1
    tot[k][1] += v * scale
all_ms = sum(v[1] for v in tot.values())
print("# Launch list (ncu --metrics gpu__time_duration.sum --clock-control none)")
if len(sys.argv) > 2:
    print(f"# cmd: {sys.argv[2]}")
print("# cold-cache, serialised replays: compare SHARES, not absolute times")
print(f"{'kernel':44s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}")
for k, (n, ms) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:44s} {n:8d} {ms:10.2f} {100 * ms / all_ms:6.2f}%")
