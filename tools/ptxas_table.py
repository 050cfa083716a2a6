"""Registers / spills per kernel from a ptxas -v report (csrc/ptxas_report.txt), demangled.
usage: python tools/ptxas_table.py [report] [regex]"""
import re
import subprocess
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "paper_1811_01201_b200/csrc/ptxas_report.txt"
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
cur, rows = None, {}
for ln in open(path):
    m = re.search(r"Compiling entry function '(\S+)'", ln)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m and cur:
        rows.setdefault(cur, {})["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", ln)
    if m and cur:
        rows.setdefault(cur, {})["regs"] = int(m.group(1))
names = list(rows)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
for n, d in sorted(zip(names, dem), key=lambda x: x[1]):
    if pat and not pat.search(d):
        continue
    r = rows[n]
    print(f"{r.get('regs', '?'):>4} regs  spill {r.get('spill', (0, 0))}  {d}")
