"""Registers / spills per K2 instantiation from the build's ptxas log (dev tool).

python scripts/ptxas_report.py [filter]   e.g. filter "float, 4"
"""
import os
import re
import subprocess
import sys

LOG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_0912_4506_b200", "csrc", "ptxas.log")
flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
rows = {}
for line in open(LOG):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur]["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
names = list(rows)
dem = subprocess.run(["cu++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
for n, d in zip(names, dem):
    d = d.replace("(int)", "").replace("(bool)", "")
    if ("tb_kernel" in d or "tb2_kernel" in d) and flt in d:
        r = rows[n]
        print(f"{r.get('regs', '?'):>4} regs  spill {r.get('spill', (0, 0))}  {d.split('(')[0]}")
