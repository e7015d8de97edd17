#!/usr/bin/env python3
"""Summarise paper_1711_04556_b200/_lib/ptxas.log: registers and spills per kernel."""
import re
import subprocess
import sys
from pathlib import Path

log = Path(sys.argv[1] if len(sys.argv) > 1 else
           Path(__file__).resolve().parent.parent / "paper_1711_04556_b200/_lib/ptxas.log")
text = log.read_text()
blocks = re.split(r"ptxas info\s+: Compiling entry function '([^']+)'", text)
for name, body in zip(blocks[1::2], blocks[2::2]):
    regs = re.search(r"Used (\d+) registers", body)
    spill = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", body)
    stack = re.search(r"(\d+) bytes stack frame", body)
    pretty = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    pretty = re.sub(r"\(.*", "", pretty)
    print(f"{pretty:40s} regs={regs.group(1) if regs else '?':>4} "
          f"stack={stack.group(1) if stack else '?':>4} "
          f"spill_st={spill.group(1) if spill else '?':>4} spill_ld={spill.group(2) if spill else '?':>4}")
