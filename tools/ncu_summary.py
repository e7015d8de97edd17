#!/usr/bin/env python3
"""Key metrics of an ncu report (details page) as 'section | metric | value'."""
import csv
import io
import subprocess
import sys

KEEP = ("Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Cache Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Executed Instructions", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Achieved Occupancy", "Theoretical Occupancy", "Achieved Active Warps Per SM",
        "Block Limit Registers", "Block Limit Shared Mem", "Grid Size", "Block Size",
        "Branch Efficiency", "Waves Per SM", "L1/TEX Hit Rate", "L2 Hit Rate")
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in KEEP:
        print(f"{d['Kernel Name'][:28]:28s} | {d['Metric Name']:38s} | {d['Metric Value']} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hdr = rr[0]
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__pcsamp_sample_count"]
for row in rr[2:]:
    for w in want:
        if w in hdr:
            print(f"{'raw':28s} | {w:38s} | {row[hdr.index(w)]} {rr[1][hdr.index(w)]}")
