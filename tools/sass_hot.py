#!/usr/bin/env python3
"""Find the evaluation subroutine of a kernel in the library SASS and report
its size, spills (LDL/STL) and the scan-round instruction count.
usage: tools/sass_hot.py <mangled-kernel-substring>"""
import re
import subprocess
import sys
from pathlib import Path

lib = Path(__file__).resolve().parent.parent / "paper_1711_04556_b200/_lib/libb200tabu.so"
sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True).stdout
want = sys.argv[1] if len(sys.argv) > 1 else "k_solveILi1ELi32ELi1E"
funcs = re.split(r"\n\s*Function : ", sass)
body = next(f for f in funcs if f.startswith("_Z") and want in f.split("\n")[0])
ins = []
for line in body.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?)\s*;", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
# subroutine = [CALL target, first RET after it]
targets = sorted({int(t, 16) for _, x in ins for t in re.findall(r"CALL\.REL\.NOINC (0x[0-9a-f]+)", x)})
addr = [a for a, _ in ins]
for t in targets:
    i = addr.index(t) if t in addr else None
    if i is None:
        continue
    j = i
    while not ins[j][1].startswith("RET"):
        j += 1
    sub = ins[i:j + 1]
    votes = sum(1 for _, x in sub if x.startswith("VOTE.ANY R"))
    spills = sum(1 for _, x in sub if x.startswith(("LDL", "STL")))
    print(f"subroutine @{hex(t)}: {len(sub)} instr, ballots {votes}, LDL/STL {spills}")
spills = sum(1 for _, x in ins if x.startswith(("LDL", "STL")))
print(f"kernel total: {len(ins)} instr, LDL/STL {spills}")
