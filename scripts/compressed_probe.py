"""Compressed (single-array, in-place) vs two-grid storage at BASELINE size (dev tool).

python scripts/compressed_probe.py [--n 1024] [--depths 2,3,4] [--levels 24] [--chunk 32]
Prints GLUP/s (CUDA events, inputs >> L2), HBM bytes of each storage and digest agreement.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0912_4506_b200 as sp  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--depths", default="2,3,4")
    ap.add_argument("--levels", type=int, default=24)
    ap.add_argument("--chunk", type=int, default=32)
    args = ap.parse_args()
    n = args.n
    shape = (n, n, n)
    pat = sp.FillPattern.dirichlet_box("random", shape, (1.0, 0, 0.5, 0, 0.25, 0))
    out = {}
    for depth in [int(d) for d in args.depths.split(",")]:
        levels = (args.levels // depth) * depth
        c = sp.CompressedGrid(sp.GridDims(n, n, n), pat, chunk=args.chunk)
        sp.sweeps(c, depth, depth=depth)                       # warm-up
        tc = timed(lambda: sp.sweeps(c, levels, depth=depth))
        dc = c.digest()
        import ctypes
        from paper_0912_4506_b200 import _native as N
        def scat():
            for _ in range(10):
                N.check(N.lib().sp_ghost_shell(c._box_ptr(), c.sp_dtype, ctypes.byref(c.layout),
                                               ctypes.c_void_p(c._shell.data_ptr()), 1, c.stream()))
        t_sc = timed(scat) / 10
        hb = c.hbm_bytes
        del c
        torch.cuda.empty_cache()
        g = sp.TwoGrid(sp.GridDims(n, n, n), pat)
        sp.sweeps(g, depth, depth=depth)
        tg = timed(lambda: sp.sweeps(g, levels, depth=depth))
        dg = g.digest()
        hg = sum(b.numel() * b.element_size() for b in g.buffers)
        del g
        torch.cuda.empty_cache()
        out[depth] = {"compressed_glups": round(n ** 3 * levels / tc / 1e9, 1),
                      "twogrid_glups": round(n ** 3 * levels / tg / 1e9, 1),
                      "compressed_GB": round(hb / 1e9, 2), "twogrid_GB": round(hg / 1e9, 2),
                      "same_digest": dc == dg, "ghost_scatter_ms": round(t_sc * 1e3, 3)}
        print(depth, out[depth], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
