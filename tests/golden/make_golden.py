"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``stencilpipe`` from /root/reference/pkg/src, runs the reference's
own ``TwoGrid``/``sweep_naive``/``oracle``/``run_distributed`` and writes
small fixtures next to this script.  The GPU box never runs this file; the
tests only read its outputs.  The fixtures pin the oracle (oracle/) and the
device kernels.

Faced patterns (the BASELINE configs' Dirichlet boxes) are built here as
duck-typed objects with ``.evaluate(lo, hi)`` on top of the reference's own
``FillPattern.random`` (the same trick as R/decomp.py:107-117), independently
of oracle/oracle.py.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from stencilpipe.decomp import run_distributed  # noqa: E402
from stencilpipe.grid import FillPattern, GridDims, TwoGrid  # noqa: E402
from stencilpipe.kernel import stencil_point, sweep_naive  # noqa: E402
from stencilpipe.pipeline import PipelineConfig, run_node_sweeps  # noqa: E402
from stencilpipe.verify import oracle, oracle_trajectory  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

_H1 = np.uint64(0x9E3779B97F4A7C15)


def digest(inner) -> int:
    """Order-independent digest, defined in oracle/jacobi_oracle.c."""
    inner = np.ascontiguousarray(inner)
    if inner.dtype == np.float64:
        bits = inner.view(np.uint64).ravel()
    else:
        bits = inner.view(np.uint32).ravel().astype(np.uint64)
    idx = np.arange(bits.size, dtype=np.uint64)
    H2 = np.uint64(0xBF58476D1CE4E5B9)
    H3 = np.uint64(0x94D049BB133111EB)
    with np.errstate(over="ignore"):
        h = bits + idx * _H1
        h = (h ^ (h >> np.uint64(30))) * H2
        h = (h ^ (h >> np.uint64(27))) * H3
        h = h ^ (h >> np.uint64(31))
        return int(np.sum(h, dtype=np.uint64))


class FacedPattern:
    """Reference FillPattern interior + constant Dirichlet faces.

    faces = (z-, z+, y-, y+, x-, x+); a ghost cell takes the first face it
    lies beyond in that order.  ``pm1`` maps u -> 2u-1 (BASELINE config 4).
    """

    def __init__(self, base: FillPattern, gshape, faces, pm1=False, origin=(0, 0, 0)):
        self.base = base
        self.gshape = tuple(gshape)
        self.faces = tuple(faces)
        self.pm1 = pm1
        self.origin = tuple(origin)

    def evaluate(self, lo, hi):
        glo = tuple(l + o for l, o in zip(lo, self.origin))
        ghi = tuple(h + o for h, o in zip(hi, self.origin))
        v = self.base.evaluate(glo, ghi)
        if self.pm1:
            v = 2.0 * v - 1.0
        z = np.arange(glo[0], ghi[0]).reshape(-1, 1, 1)
        y = np.arange(glo[1], ghi[1]).reshape(1, -1, 1)
        x = np.arange(glo[2], ghi[2]).reshape(1, 1, -1)
        nz, ny, nx = self.gshape
        conds = [(z < 0, 0), (z >= nz, 1), (y < 0, 2), (y >= ny, 3), (x < 0, 4), (x >= nx, 5)]
        for cond, f in reversed(conds):
            v = np.where(cond, self.faces[f], v)
        return np.ascontiguousarray(v + np.zeros(v.shape))


def run_twogrid(dims, pattern, levels, dtype=np.float64):
    g = TwoGrid(dims, pattern)
    if dtype != np.float64:
        g.a = g.a.astype(dtype)
        g.b = g.b.astype(dtype)
    for _ in range(levels):
        sweep_naive(g)
    return g


def main():
    kat = {}
    # --- known answers (R/grid.py:109-117, R/kernel.py:18-20) --------------
    r0 = FillPattern.random(0)
    pts = {}
    for c in [(0, 0, 0), (-1, -1, -1), (0, 0, 1), (1, 0, 0), (0, 1, 0), (5, 7, 11),
              (127, 127, 127), (1023, 1023, 1023), (-1, 1024, 513)]:
        v = r0.evaluate(c, tuple(i + 1 for i in c))[0, 0, 0]
        pts[",".join(map(str, c))] = int(np.float64(v).view(np.uint64))
    kat["random0_bits"] = pts
    r42 = FillPattern.random(42)
    kat["random42_bits_0_0_0"] = int(np.float64(r42.evaluate((0, 0, 0), (1, 1, 1))[0, 0, 0]).view(np.uint64))
    kat["one_sixth_bits"] = int(np.float64(1.0 / 6.0).view(np.uint64))
    kat["one_sixth_f32_bits"] = int(np.float32(1.0 / 6.0).view(np.uint32))
    vals = (0.1, 0.7, 1e-17, 0.3, 0.9, 1.1)
    kat["stencil_point_order"] = {"args": vals,
                                  "bits": int(np.float64(stencil_point(*vals)).view(np.uint64))}
    fields = {}

    # --- hotplate 4^3, one sweep (reference test_kernel.py:34-41) -----------
    g = run_twogrid(GridDims(4, 4, 4), FillPattern.hotplate(), 1)
    fields["hotplate4_l1"] = g.interior().copy()

    # --- random(11) 16^3 trajectory, levels 0..8 ----------------------------
    traj = oracle_trajectory(GridDims(16, 16, 16), FillPattern.random(11), 8)
    fields["r11_16_traj"] = np.stack(traj)

    # --- ragged 9x7x5 random(2), 7 sweeps; 1x3x2 degenerate -----------------
    fields["r2_9x7x5_l7"] = oracle(GridDims(9, 7, 5), FillPattern.random(2), 7).interior().copy()
    fields["r3_1x3x2_l3"] = oracle(GridDims(1, 3, 2), FillPattern.random(3), 3).interior().copy()
    fields["linear_6_l8"] = oracle(GridDims(6, 6, 6), FillPattern.linear(), 8).interior().copy()

    # --- pipelined engine == oracle (reference test_pipeline.py:156-163) ----
    g = TwoGrid(GridDims(24, 24, 24), FillPattern.random(11))
    run_node_sweeps(g, PipelineConfig(teams=2, team_size=4, updates_per_thread=2,
                                      block=(24, 16, 16)), 1)
    fields["r11_24_pipe_u16"] = g.interior().copy()

    # --- C1 shape at reduced size: faced random(0), T-agnostic ---------------
    fp = FacedPattern(FillPattern.random(0), (20, 18, 33), (1.0, 0, 0, 0, 0, 0))
    fields["c1like_33x18x20_l12"] = run_twogrid(GridDims(33, 18, 20), fp, 12).interior().copy()
    fp3 = FacedPattern(FillPattern.random(0), (17, 19, 21), (1.0, 0.0, 0.5, 0.0, 0.25, 0.0))
    g3 = run_twogrid(GridDims(21, 19, 17), fp3, 9)
    fields["c3like_21x19x17_l9"] = g3.interior().copy()
    fields["c3like_21x19x17_full0"] = TwoGrid(GridDims(21, 19, 17), fp3).current.copy()

    # --- float32 (BASELINE config 4 shape): uniform[-1,1), zero faces -------
    fp4 = FacedPattern(FillPattern.random(0), (24, 20, 36), (0,) * 6, pm1=True)
    g4 = run_twogrid(GridDims(36, 20, 24), fp4, 10, dtype=np.float32)
    assert g4.current.dtype == np.float32
    fields["c4like_f32_36x20x24_l10"] = g4.interior().copy()

    # --- distributed z-slabs (R/decomp.py:240-268), layouts (1,1,P) ---------
    dist = {}
    for P, h, steps in [(2, 1, 3), (2, 4, 2), (3, 2, 2), (4, 4, 2), (4, 8, 1)]:
        gd = GridDims(12, 10, 40)
        fpd = FacedPattern(FillPattern.random(0), (40, 10, 12), (1.0, 0, 0, 0, 0, 0))
        gathered, _ = run_distributed(gd, fpd, (1, 1, P), cfg=None, outer_steps=steps, h=h)
        key = f"dist_P{P}_h{h}_s{steps}"
        fields[key] = gathered
        dist[key] = {"P": P, "h": h, "steps": steps, "levels": h * steps}
    kat["dist_cases"] = dist

    # --- C1 itself: 128^3, faces z-=1, random(0), 100 sweeps (digest only) --
    fp1 = FacedPattern(FillPattern.random(0), (128, 128, 128), (1.0, 0, 0, 0, 0, 0))
    g1 = run_twogrid(GridDims(128, 128, 128), fp1, 100)
    kat["c1_digest_l100"] = digest(g1.interior())
    fields["c1_planes_l100"] = g1.interior()[[0, 1, 63, 126, 127]].copy()
    kat["c1_planes_index"] = [0, 1, 63, 126, 127]
    kat["c1_digest_l0"] = digest(TwoGrid(GridDims(128, 128, 128), fp1).interior())

    for k, v in fields.items():
        kat.setdefault("digests", {})[k] = digest(v) if v.ndim == 3 else None
    np.savez_compressed(os.path.join(HERE, "ref_fields.npz"), **fields)
    with open(os.path.join(HERE, "ref_kat.json"), "w") as fh:
        json.dump(kat, fh, indent=1, sort_keys=True)
    print("wrote", sorted(fields))


if __name__ == "__main__":
    main()
