"""Instruction mix per cell-level of a K2 capture (dev tool).

python scripts/ncu_mix2.py REPORT.ncu-rep [N]
Reads the SASS source page (ncu --import-source), normalises executed
instruction counts by the executed DMUL/FMUL(2) count (one per cell-level;
FMUL2 counts two), prints the mix by opcode and the N hottest stall sites.
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
isrc, iex = h.index("Source"), h.index("Instructions Executed")
iss = h.index("Warp Stall Sampling (All Samples)")


def op(r):
    s = r[isrc].strip().split()
    if not s:
        return ""
    return s[1] if s[0].startswith("@") and len(s) > 1 else s[0]


mul = 0.0
for r in data:
    o = op(r)
    if o.startswith("DMUL") or o.startswith("FMUL2"):
        mul += int(r[iex] or 0) * (2 if o.startswith("FMUL2") else 1) * (1 if o.startswith("DMUL") else 1)
    elif o.startswith("FMUL") and not o.startswith("FMUL2"):
        mul += int(r[iex] or 0)
total = sum(int(r[iex] or 0) for r in data)
print(f"total {total / mul:.2f} instructions per warp-cell-level ({total} executed, {mul:.0f} multiplies)")
mix = collections.Counter()
for r in data:
    o = op(r)
    if o:
        mix[o] += int(r[iex] or 0) / mul
for o, n in mix.most_common(45):
    print(f"  {o:36s} {n:7.3f}")
tot_s = sum(float(r[iss] or 0) for r in data)
print("hottest stall sites:")
for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:top]:
    print(f"  {float(r[iss]) / tot_s * 100:5.1f}%  {r[isrc].strip()[:90]}")
