"""Tabulate perf_probe output (shape x depth, GLUP/s per repetition) (dev)."""
import collections
import re
import sys

for f in sys.argv[1:]:
    d = collections.defaultdict(lambda: collections.defaultdict(list))
    for line in open(f):
        m = re.match(r"(\d+) (\d+)\s+\{'glups': ([\d.]+)", line)
        if m:
            d[int(m.group(1))][int(m.group(2))].append(float(m.group(3)))
    deps = sorted({k for v in d.values() for k in v})
    print(f)
    print("shape " + " ".join(f"T={t:<11d}" for t in deps))
    for sh in sorted(d):
        print(f"{sh:5d} " + " ".join(f"{'/'.join('%.0f' % x for x in d[sh].get(t, [])):13s}" for t in deps))
