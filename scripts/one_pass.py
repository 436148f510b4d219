"""Dev tool: run a few K2 passes of one configuration (for ncu captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0912_4506_b200 as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--nz", type=int, default=0)
ap.add_argument("--dtype", default="f64")
ap.add_argument("--depth", type=int, default=2)
ap.add_argument("--shape", type=int, default=0)
ap.add_argument("--passes", type=int, default=3)
ap.add_argument("--chunks", type=int, default=0)
ap.add_argument("--sched", default="", help="dynamic:strip")
args = ap.parse_args()
dt = np.float64 if args.dtype == "f64" else np.float32
n, nz = args.n, args.nz or args.n
pat = sp.FillPattern.dirichlet_box("random", (nz, n, n), (1.0, 0, 0.5, 0, 0.25, 0))
g = sp.TwoGrid(sp.GridDims(n, n, nz), pat, dtype=dt)
sp._native.lib().sp_set_tuning(args.shape, args.chunks)
if args.sched:
    sp._native.lib().sp_set_schedule(*(int(v) for v in args.sched.split(":")))
for _ in range(args.passes):
    sp.sweeps(g, args.depth, depth=args.depth)
torch.cuda.synchronize()
print("ok", g.digest())
