"""Quick device timing of K2 at BASELINE sizes for every depth (dev tool).

python scripts/perf_probe.py [--n 1024] [--dtype f64] [--levels 24] [--depths 1,2,4]
Prints GLUP/s per depth (CUDA events, inputs >> L2) and the FP64 add probe.
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0912_4506_b200 as sp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--nz", type=int, default=0)
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--levels", type=int, default=24)
    ap.add_argument("--depths", default="1,2,3,4,5,6,8")
    ap.add_argument("--chunks", type=int, default=0)
    ap.add_argument("--shapes", default="0", help="comma list: 0=auto, k=shape k-1")
    ap.add_argument("--sched", default="", help="comma list of dynamic:strip (sp_set_schedule)")
    args = ap.parse_args()
    dt = np.float64 if args.dtype == "f64" else np.float32
    n = args.n
    nz = args.nz or n
    shape = (nz, n, n)
    pat = sp.FillPattern.dirichlet_box("random", shape, (1.0, 0, 0.5, 0, 0.25, 0))
    g = sp.TwoGrid(sp.GridDims(n, n, nz), pat, dtype=dt)
    out = {}
    rate = ctypes.c_double()
    ms = ctypes.c_double()
    sp._native.check(sp._native.lib().sp_probe_fp64(ctypes.byref(rate), ctypes.byref(ms)))
    out["fp64_dadd_per_s"] = rate.value
    combos = [(sh, sc) for sc in (args.sched.split(",") if args.sched else [""])
              for sh in [int(v) for v in args.shapes.split(",")]]
    for shape, sc in combos:
      sp._native.lib().sp_set_tuning(shape, args.chunks)
      if sc:
        dyn, strip = (int(v) for v in sc.split(":"))
        sp._native.lib().sp_set_schedule(dyn, strip)
      for depth in [int(d) for d in args.depths.split(",")]:
        levels = (args.levels // depth) * depth
        sp.sweeps(g, depth, depth=depth)   # warm-up (JIT attr, TMA descriptors)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        sp.sweeps(g, levels, depth=depth)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        glups = n * n * nz * levels / t / 1e9
        es = 8 if dt == np.float64 else 4
        key = f"S{shape}T{depth}" + (f"@{sc}" if sc else "")
        out[key] = {"glups": round(glups, 1), "ms_per_pass": round(t / (levels // depth) * 1e3, 3),
                            "hbm_equiv_gbs": round(glups * 2 * es / depth, 1)}
        print(shape, depth, sc, out[key], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
