"""Full-size golden digests for the BASELINE configs, computed by the C oracle.

The C oracle (oracle/jacobi_oracle.c) is pinned bit-for-bit to the reference
package by tests/test_oracle.py on the fixtures make_golden.py produced from
the reference itself; running the reference's numpy code at 1024^3 x 100
sweeps is impractical ("Scale of goldens"), so the full-size
goldens are the pinned oracle's digests.  Run here (needs ~35 GB of RAM):

    python tests/golden/make_big_digests.py [--only c1,c2,...]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402

Z1 = (1.0, 0.0, 0.0, 0.0, 0.0, 0.0)
C3F = (1.0, 0.0, 0.5, 0.0, 0.25, 0.0)

# name -> (shape (nz, ny, nx), kind, faces, dtype, checkpoints in levels)
CASES = {
    "c1": ((128, 128, 128), "random", Z1, np.float64, [0, 100]),
    "c2": ((512, 512, 512), "random", Z1, np.float64, [0, 200]),
    "c3": ((1024, 1024, 1024), "random", C3F, np.float64, [0, 100]),
    "c4": ((2048, 1024, 1024), "random_pm1", (0.0,) * 6, np.float32, [0, 200]),
    "c5w": ((512, 1024, 1024), "random", Z1, np.float64, [0, 100]),
    "c5s": ((2048, 1024, 1024), "random", Z1, np.float64, [0, 100]),
}


def run(name):
    shape, kind, faces, dtype, cps = CASES[name]
    t0 = time.time()
    g = O.CGrid(shape, O.BoxPattern(kind, seed=0, faces=faces, global_shape=shape), dtype=dtype)
    out = {"shape": list(shape), "kind": kind, "faces": list(faces),
           "dtype": np.dtype(dtype).name, "digests": {}}
    done = 0
    for lv in cps:
        g.sweeps(lv - done)
        done = lv
        out["digests"][str(lv)] = str(g.digest())
    out["oracle_seconds"] = round(time.time() - t0, 1)
    out["oracle_threads"] = O.num_threads()
    del g
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=",".join(CASES))
    args = ap.parse_args()
    path = os.path.join(HERE, "big_digests.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    for name in args.only.split(","):
        data[name] = run(name)
        print(name, data[name], flush=True)
        with open(path, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
