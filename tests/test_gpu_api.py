"""Device forms of the reference API calls the round-1 suite did not exercise
(VERDICT r01 missing #2 / weak #1): sweep_spatial_blocked, check_maximum_principle,
value_at.  Each mirrors the reference test it is named after
(R = /root/reference/pkg; R/tests/test_kernel.py:55-161, R/tests/test_grid.py:29-66)
and checks the device result bit for bit against the oracle.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bitwise(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def _oracle(O, shape, seed, levels):
    g = O.CGrid(shape, O.BoxPattern("random", seed=seed, faces=None, global_shape=None))
    g.sweeps(levels)
    return g.interior()


@pytest.mark.parametrize("dims,bs,sweeps,seed", [
    ((32, 32, 32), (32, 8, 8), 4, 7),      # R/tests/test_kernel.py:63-72
    ((8, 8, 8), (1, 1, 1), 2, 5),          # unit blocks, :75-83
    ((9, 7, 5), (9, 7, 5), 1, 2),          # one block = the domain, :86-93
    ((40, 24, 33), (16, 5, 7), 3, 11),     # ragged last blocks in every axis
])
def test_blocked_matches_naive_and_oracle(sp, O, dims, bs, sweeps, seed):
    d = sp.GridDims(*dims)
    pat = sp.FillPattern.random(seed)
    ref = sp.allocate(d, "twogrid", pat)
    blk = sp.allocate(d, "twogrid", pat)
    for _ in range(sweeps):
        sp.sweep_naive(ref)
        sp.sweep_spatial_blocked(blk, bs)
    assert sp.compare(ref, blk).bitwise
    assert _bitwise(blk.interior(), _oracle(O, d.shape, seed, sweeps))


def test_blocked_launches_one_pass_per_z_block(sp):
    g = sp.allocate(sp.GridDims(8, 8, 10), "twogrid", sp.FillPattern.random(1))
    n0 = sp.launch_count()
    sp.sweep_spatial_blocked(g, (8, 8, 3))           # z blocks [0,3) [3,6) [6,9) [9,10)
    assert sp.launch_count() - n0 == 4


@pytest.mark.parametrize("bs", [(5, 4, 4), (4, 5, 4), (4, 4, 5), (0, 4, 4), (4, 4, 0)])
def test_blocked_rejects_bad_blocks(sp, bs):
    g = sp.allocate(sp.GridDims(4, 4, 4), "twogrid", sp.FillPattern.constant(0.0))
    with pytest.raises(sp.GridError):
        sp.sweep_spatial_blocked(g, bs)          # R/tests/test_kernel.py:95-98


@pytest.mark.parametrize("seed", [0, 1, 17, 256, 9999])
def test_maximum_principle_random(sp, seed):
    g = sp.allocate(sp.GridDims(6, 6, 6), "twogrid", sp.FillPattern.random(seed))
    before = g.full_view().copy()
    sp.sweep_naive(g)
    assert sp.check_maximum_principle(before, g.interior())      # R/tests/test_kernel.py:155-161


def test_maximum_principle_faced_box_deep_passes(sp):
    shape = (24, 20, 36)
    faces = (1.0, 0.0, 0.5, 0.0, 0.25, 0.0)
    g = sp.TwoGrid(sp.GridDims(36, 20, 24), sp.FillPattern.dirichlet_box("random", shape, faces, seed=0))
    before = g.full_view().copy()
    interior0 = g.interior().copy()
    for T in (2, 4, 8):
        sp.sweeps(g, T, depth=T)
        after = g.interior()
        assert sp.check_maximum_principle(before, after)
        # with the shell passed separately (R/verify.py:74-83 ghost_shell argument)
        assert sp.check_maximum_principle(interior0, after, ghost_shell=before)
        before = g.full_view().copy()


def test_maximum_principle_detects_violation(sp):
    before = np.zeros((3, 3, 3))
    after = np.full((1, 1, 1), 1e-300)
    assert not sp.check_maximum_principle(before, after)
    assert sp.check_maximum_principle(before, after, ghost_shell=np.array([1.0]))


def test_value_at_linear_fill(sp):
    g = sp.allocate(sp.GridDims(2, 2, 2), "twogrid", sp.FillPattern.linear())   # R/tests/test_grid.py:29-34
    assert g.value_at(1, 1, 1) == 3.0
    assert g.value_at(0, 0, 0) == 0.0
    assert g.value_at(-1, 0, 0) == -1.0


def test_value_at_constant_everywhere_and_bounds(sp):
    g = sp.allocate(sp.GridDims(3, 3, 3), "twogrid", sp.FillPattern.constant(5.0))
    for idx in [(-1, -1, -1), (0, 0, 0), (2, 1, 0), (3, 3, 3)]:
        assert g.value_at(*idx) == 5.0                                     # R/tests/test_grid.py:54-57
    with pytest.raises(IndexError):
        g.value_at(4, 0, 0)                                                # :60-65
    with pytest.raises(IndexError):
        g.value_at(0, 0, -2)


def test_value_at_tracks_current_after_sweeps(sp, O):
    d = sp.GridDims(10, 9, 8)
    g = sp.allocate(d, "twogrid", sp.FillPattern.random(3))
    sp.sweeps(g, 5, depth=2)
    ref = _oracle(O, d.shape, 3, 5)
    for (i, j, k) in [(0, 0, 0), (9, 8, 7), (4, 3, 2)]:
        assert g.value_at(i, j, k) == ref[k, j, i]
