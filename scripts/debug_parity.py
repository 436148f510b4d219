"""Dev tool: locate mismatching cells for a (shape, depth, dtype) combination."""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_0912_4506_b200 as sp  # noqa: E402
from oracle import oracle as O  # noqa: E402

lib = sp._native.lib()
faces = (0.3, -1.0, 2.0, 0.0, 1.0, -0.5)
for shape_id, depth, dt, grid in itertools.product(
        [int(v) for v in sys.argv[1].split(",")], [int(v) for v in sys.argv[2].split(",")],
        [np.float64, np.float32], [(9, 80, 70), (20, 70, 60), (40, 30, 64)]):
    lib.sp_set_tuning(shape_id, int(os.environ.get("CHUNKS", "0")))
    levels = depth
    seed = 3
    g = sp.TwoGrid(sp.GridDims(grid[2], grid[1], grid[0]),
                   sp.FillPattern.dirichlet_box("random", grid, faces, seed=seed), dtype=dt)
    sp.sweeps(g, levels, depth=depth)
    got = g.interior()
    ref = O.CGrid(grid, O.BoxPattern("random", seed=seed, faces=faces, global_shape=grid), dtype=dt)
    ref.sweeps(levels)
    r = ref.interior()
    bad = np.argwhere(got.view(np.uint8).reshape(got.shape + (-1,)).any(-1) !=
                      False) if False else np.argwhere(got != r)
    tag = "OK " if len(bad) == 0 else "BAD"
    info = ""
    if len(bad):
        zs = np.unique(bad[:, 0])
        ys = np.unique(bad[:, 1])
        xs = np.unique(bad[:, 2])
        info = f"n={len(bad)} z={zs[:10]} y={ys[:12]} x={xs[:12]}"
    print(tag, shape_id, depth, np.dtype(dt).name, grid, info, flush=True)
lib.sp_set_tuning(0, 0)
