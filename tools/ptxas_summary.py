"""Summarise `nvcc -Xptxas -v` logs: registers / spills per kernel (demangled names).
    python tools/ptxas_summary.py paper_2601_13994_b200/build/device.cu.o.log [filter]"""
import re
import subprocess
import sys

log = open(sys.argv[1]).read().splitlines()
flt = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
rows = []
for l in log:
    m = re.search(r"Compiling entry function '(\S+)'", l)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", l)
    if m:
        cur["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", l)
    if m:
        cur["regs"] = int(m.group(1))
names = subprocess.run(["c++filt"], input="\n".join(r["name"] for r in rows), capture_output=True,
                       text=True).stdout.splitlines()
for r, d in zip(rows, names):
    if flt in d:
        print(f"{r.get('regs', '?'):>4} regs  spill {r.get('spill', ('?', '?'))}  {d}")
