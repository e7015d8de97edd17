#!/usr/bin/env python3
"""Per-CUDA-source-line hot spots of an ncu report (needs -lineinfo and
--import-source on): SASS instructions executed and warp-stall samples,
attributed to the source line they map to.
usage: tools/ncu_lines.py <report.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0, 0, ""])
f = ln = None
src = ""
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0]:
        ln, src = r[0], r[1]
        continue
    if len(r) > 7 and r[2].startswith("0x"):
        try:
            s, i = int(r[4] or 0), int(r[7] or 0)
        except ValueError:
            continue
        a = agg[(f, ln)]
        a[0] += s
        a[1] += i
        a[2] = src.strip()[:90]
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
rows = sorted(agg.items(), key=lambda kv: -kv[1][0])
print(f"{'samp%':>6} {'inst%':>6}  file:line  source")
for (fn, l), (s, i, sr) in rows[:top]:
    print(f"{100*s/ts:6.2f} {100*i/ti:6.2f}  {fn}:{l}  {sr}")
