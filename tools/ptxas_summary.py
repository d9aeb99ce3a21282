"""Summarise a ptxas -v log: registers / spills per demangled kernel name.
   python tools/ptxas_summary.py paper_2602_11470_b200/build/ntt.ptxas.log [filter]"""
import re
import subprocess
import sys

log = open(sys.argv[1]).read().splitlines()
flt = sys.argv[2] if len(sys.argv) > 2 else ""
cur, rows = None, {}
for line in log:
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        rows.setdefault(cur, {})["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.setdefault(cur, {})["regs"] = int(m.group(1))
names = subprocess.run(["c++filt"], input="\n".join(rows), capture_output=True, text=True).stdout.splitlines()
for (k, v), nm in zip(rows.items(), names):
    nm = nm.replace("(anonymous namespace)::", "").replace("void ", "")
    nm = re.sub(r"\(sf::\w+, sf::\w+\)$", "", nm)
    if flt in nm:
        print(f"{nm:60s} regs {v.get('regs')}  spill st/ld {v.get('spill')}")
