"""Summarise ncu output for profiles/ (dev tool, runs where `ncu` can import reports).

python scripts/summarize_ncu.py full REPORT.ncu-rep OUT_PREFIX   -> OUT_PREFIX_summary.txt + _raw.json
python scripts/summarize_ncu.py launches LAUNCHES.csv OUT.txt    -> per-kernel launch share table
"""
import collections
import csv
import io
import json
import subprocess
import sys

RAW_KEYS = [
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__block_size", "launch__grid_size",
    "launch__registers_per_thread", "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    # the LSU data pipe carries SHFL, LDS and STS: the busiest unit of the K2 kernels
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
]


def ncu_csv(report, page):
    out = subprocess.run(["ncu", "-i", report, "--page", page, "--csv"], capture_output=True, text=True,
                         check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full(report, prefix):
    rows = ncu_csv(report, "raw")
    names, units, vals = rows[0], rows[1], rows[2]
    raw = {}
    for k, u, v in zip(names, units, vals):
        if k in RAW_KEYS or (k.startswith("smsp__average_warps_issue_stalled_")
                             and k.endswith("_per_issue_active.ratio")):
            raw[k] = f"{v} {u}".strip()
    raw["kernel"] = vals[names.index("Kernel Name")] if "Kernel Name" in names else ""
    with open(prefix + "_raw.json", "w") as fh:
        json.dump(raw, fh, indent=1)
    det = ncu_csv(report, "details")
    hdr = det[0]
    sec, name, unit, val = (hdr.index(c) for c in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    keep = {"GPU Speed Of Light Throughput", "Compute Workload Analysis", "Scheduler Statistics",
            "Warp State Statistics", "Launch Statistics", "Occupancy", "Memory Workload Analysis"}
    lines = [f"kernel: {raw['kernel']}"]
    for r in det[1:]:
        if r[sec] in keep:
            lines.append(f"{r[sec][:28]:28s} {r[name]:40s} {r[unit]:14s} {r[val]}")
    with open(prefix + "_summary.txt", "w") as fh:
        fh.write("\n".join(lines) + "\n")


def launches(path, out):
    rows = list(csv.reader(line for line in open(path) if not line.startswith("==")))
    ix = {k: i for i, k in enumerate(rows[0])}
    per = collections.defaultdict(list)
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}
    for r in rows[1:]:
        if r[ix["Metric Name"]] == "gpu__time_duration.sum":
            per[r[ix["Kernel Name"]]].append(float(r[ix["Metric Value"]]) * scale[r[ix["Metric Unit"]]])
    tot = sum(sum(v) for v in per.values())
    with open(out, "w") as fh:
        fh.write(f"# {path}: gpu__time_duration.sum per launch (ncu, --clock-control none, serialised)\n")
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            fh.write(f"{k[:90]:90s} n={len(v):4d} avg={sum(v) / len(v):8.3f} ms "
                     f"total={sum(v):9.2f} ms share={100 * sum(v) / tot:5.1f}%\n")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
