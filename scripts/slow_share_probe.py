"""How much do the boundary (SLOW-step) tiles cost?  Time a full T-level pass of C3 against a
pass over an interior sub-box made of whole tiles only (dev tool).

python scripts/slow_share_probe.py [--depth 4]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0912_4506_b200 as sp  # noqa: E402
from paper_0912_4506_b200.pipeline import run_pass  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--depth", type=int, default=4)
ap.add_argument("--reps", type=int, default=12)
args = ap.parse_args()
n, T = 1024, args.depth
pat = sp.FillPattern.dirichlet_box("random", (n, n, n), (1.0, 0, 0.5, 0, 0.25, 0))
g = sp.TwoGrid(sp.GridDims(n, n, n), pat)
lo, hi = (0, 0, 0), (n, n, n)


def timed(out_lo, out_hi):
    run_pass(g, T, lo, hi, out_lo=out_lo, out_hi=out_hi)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        run_pass(g, T, lo, hi, out_lo=out_lo, out_hi=out_hi)
    e1.record()
    torch.cuda.synchronize()
    cells = 1
    for a, b in zip(out_lo, out_hi):
        cells *= b - a
    return cells * T * args.reps / (e0.elapsed_time(e1) / 1e3) / 1e9


for rep in range(2):
    print("full pass          %.1f GLUP/s" % timed(lo, hi))
    # 16 x 17 whole tiles of the FQ 12x5 kernel (56 x 52 outputs), away from every x/y wall
    print("interior tiles     %.1f GLUP/s" % timed((0, 70, 64), (n, 70 + 17 * 52, 64 + 16 * 56)))
    print("x walls included   %.1f GLUP/s" % timed((0, 70, 0), (n, 70 + 17 * 52, n)))
    # four tile columns each: at the left wall, in the middle, at the right wall (all full-width tiles)
    for name, x0 in (("left wall", 0), ("middle", 448), ("right wall", n - 224)):
        print("4 columns, %-10s %.1f GLUP/s" % (name, timed((0, 70, x0), (n, 70 + 17 * 52, x0 + 224))))
    # four tile rows each (y): at the low wall, in the middle
    for name, y0 in (("low wall", 0), ("middle", 416)):
        print("4 rows, %-10s    %.1f GLUP/s" % (name, timed((0, y0, 64), (n, y0 + 208, 64 + 16 * 56))))
