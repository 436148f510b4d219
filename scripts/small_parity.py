"""Small K2 parity sweep (dev tool): every default depth, the level-split and cluster
variants, fp64 and fp32, on ragged boxes with walls -- bitwise against the C oracle.

python scripts/small_parity.py     (small enough for compute-sanitizer where the pool allows it;
                                    on this pool the sanitizer is closed)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_0912_4506_b200 as sp  # noqa: E402
from oracle import oracle as O  # noqa: E402


def run(shape, levels, depth, dtype, variant):
    lib = sp._native.lib()
    lib.sp_set_tuning(variant, 0)
    faces = (0.7, -0.25, 1.5, 0.0, -1.0, 0.5)
    g = sp.TwoGrid(sp.GridDims(shape[2], shape[1], shape[0]),
                   sp.FillPattern.dirichlet_box("random", shape, faces, seed=3), dtype=dtype)
    sp.sweeps(g, levels, depth=depth)
    ref = O.CGrid(shape, O.BoxPattern("random", seed=3, faces=faces, global_shape=shape), dtype=dtype)
    ref.sweeps(levels)
    ok = np.array_equal(g.interior().view(np.uint8), ref.interior().view(np.uint8))
    lib.sp_set_tuning(0, 0)
    print(f"variant {variant:2d} depth {depth} {np.dtype(dtype).name} {shape}: {'bitwise OK' if ok else 'MISMATCH'}",
          flush=True)
    return ok


def main():
    ok = True
    for dt in (np.float64, np.float32):
        for depth in (1, 2, 3, 4, 6, 8):
            ok &= run((11, 37, 70), depth * 2, depth, dt, 0)
        for v in (24, 25, 26, 27):        # level split (variants 23..26)
            for depth in (4, 8):
                ok &= run((10, 40, 66), depth, depth, dt, v)
    for v in (18, 19):                    # y-cooperative clusters (variants 17, 18)
        for depth in (2, 3):
            ok &= run((8, 70, 66), depth * 2, depth, np.float64, v)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
