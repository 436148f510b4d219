"""Summarise scripts/ab_probe.sh output: best GLUP/s per (library, dtype, depth)."""
import collections
import re
import sys

best = collections.defaultdict(float)
lib = None
for line in open(sys.argv[1]):
    m = re.match(r"== (\S+) rep", line)
    if m:
        lib = m.group(1).split("/")[-1]
        continue
    m = re.match(r"(f32 )?\S+ (\d+)\s.*'glups': ([\d.]+)", line)
    if m and lib:
        key = (lib, "f32" if m.group(1) else "f64", int(m.group(2)))
        best[key] = max(best[key], float(m.group(3)))
libs = sorted({k[0] for k in best})
cols = sorted({(k[1], k[2]) for k in best})
print("lib".ljust(28) + "".join(f"{d}T{t}".rjust(9) for d, t in cols))
for l in libs:
    print(l.ljust(28) + "".join(f"{best[(l, d, t)]:9.1f}" for d, t in cols))
