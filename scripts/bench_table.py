"""One row per bench.py JSON line in a directory (dev tool): python scripts/bench_table.py DIR"""
import glob
import json
import os
import sys

for f in sorted(glob.glob(os.path.join(sys.argv[1], "bench_*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        print(os.path.basename(f), "ERR", exc)
        continue
    if d.get("impl") == "reference":
        rp = d.get("reference_package") or {}
        print(os.path.basename(f), d["value"], d["cpu_baseline"]["cores"],
              [(v["variant"], v["glups"]) for v in rp.get("variants", [])])
        continue
    c = d["clocks"] or {}
    print("%-30s T=%s %8.1f fracR=%.3f roof=%.3f e2e=%s clk=%s %s verify=%s launches=%s" % (
        os.path.basename(f), d["config"]["T"], d["value"], d["temporal_roofline"]["frac"], d["roofline"]["frac"],
        (d["e2e"] or {}).get("value"), c.get("sm_mhz"), c.get("reasons"), (d.get("verify") or {}).get("match"),
        d["gpu_launches"]))
