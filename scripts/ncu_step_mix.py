"""Per-z-step instruction mix of a K2 capture (dev tool).

python scripts/ncu_step_mix.py REPORT.ncu-rep [N]
Reads the SASS source page (ncu --import-source, -lineinfo), takes the most
common execution count of a DADD as "one z-step per warp", and prints the
executed instructions per step by opcode, plus the N hottest stall sites.
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, data = rows[1], rows[2:]
    isrc, iex = h.index("Source"), h.index("Instructions Executed")
    iss = h.index("Warp Stall Sampling (All Samples)")
    dadd = [int(r[iex] or 0) for r in data if "DADD" in r[isrc] or "FADD" in r[isrc]]
    ref = collections.Counter(dadd).most_common(1)[0][0]
    total = sum(int(r[iex] or 0) for r in data)
    print(f"one step = {ref} warp executions; {total / ref:.1f} instructions per warp-step")
    mix = collections.Counter()
    for r in data:
        s = r[isrc].strip().split()
        if s:
            mix[s[1] if s[0].startswith("@") else s[0]] += int(r[iex] or 0) / ref
    for op, n in mix.most_common(40):
        print(f"  {op:34s} {n:7.1f}")
    tot_s = sum(float(r[iss] or 0) for r in data)
    print("hottest stall sites:")
    for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:top]:
        print(f"  {float(r[iss]) / tot_s * 100:5.1f}%  x{int(r[iex] or 0) / ref:6.2f}  {r[isrc].strip()[:80]}")


if __name__ == "__main__":
    main()
