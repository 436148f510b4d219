"""Compressed single-array storage (R/grid.py:164-208, R/kernel.py:83-121) on the device:
in-place passes whose box moves by whole planes, checked bit-for-bit against the oracle
(which runs the plain A/B sweeps: the storage must not change a single bit) and against the
reference's own trajectory goldens."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FACES = (0.7, -0.25, 1.5, 0.0, -1.0, 0.5)


def _bitwise(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def _oracle(O, shape, kind, seed, faces, levels, dtype=np.float64):
    g = O.CGrid(shape, O.BoxPattern(kind, seed=seed, faces=faces,
                                    global_shape=shape if faces else None), dtype=dtype)
    g.sweeps(levels)
    return g


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("shape,levels,depth,chunk", [
    ((40, 37, 70), 12, 2, 16),      # several chunks: the chunk-order hazards are live
    ((70, 20, 66), 12, 4, 16),
    ((33, 31, 29), 9, 3, 16),
    ((100, 12, 40), 16, 8, 16),     # deepest pass, chunk = 2T
    ((9, 7, 5), 7, 3, 32),          # one chunk shorter than the shift
    ((64, 64, 64), 10, 1, 16),      # single-level passes, alternating direction
    ((50, 24, 40), 10, 2, 16),      # a 2-plane last chunk: the producer runs units ahead
])
def test_compressed_matches_oracle(sp, O, dtype, shape, levels, depth, chunk):
    nz, ny, nx = shape
    pat = sp.FillPattern.dirichlet_box("random", shape, FACES, seed=sum(shape))
    g = sp.CompressedGrid(sp.GridDims(nx, ny, nz), pat, dtype=dtype, chunk=chunk)
    sp.sweeps(g, levels, depth=depth)
    ref = _oracle(O, shape, "random", sum(shape), FACES, levels, dtype=dtype)
    assert _bitwise(g.interior(), ref.interior()), (shape, depth)
    # the ghost shell travelled with the box
    full = g.full_view()
    assert _bitwise(full, ref.current)


def test_compressed_random_ghosts_and_trajectory(sp, ref_fields):
    """random(11) on 16^3 has per-cell random ghosts (the shell must be re-scattered
    exactly); every level against the reference's own trajectory."""
    g = sp.allocate(sp.GridDims(16, 16, 16), "compressed", sp.FillPattern.random(11), slack=4)
    assert g.storage == "compressed"
    for lv in range(1, 9):
        sp.sweeps(g, 1, depth=1)
        assert _bitwise(g.interior(), ref_fields["r11_16_traj"][lv]), lv
    h = sp.CompressedGrid(sp.GridDims(16, 16, 16), sp.FillPattern.random(11))
    cfg = sp.PipelineConfig(teams=1, team_size=2, updates_per_thread=2, storage="compressed", depth=4)
    sp.run_node_sweeps(h, cfg, 2)        # 2 node sweeps of U=4
    assert _bitwise(h.interior(), ref_fields["r11_16_traj"][8])
    assert h.digest() == g.digest()


def test_compressed_footprint_and_errors(sp):
    d = sp.GridDims(64, 64, 1024)
    g = sp.CompressedGrid(d, sp.FillPattern.constant(0.5), chunk=32)
    two = 2 * 8 * (d.nz + 2) * g.layout.pz     # A/B in the same padded layout
    assert g.hbm_bytes < 0.6 * two
    cfg = sp.PipelineConfig(storage="twogrid")
    with pytest.raises(ValueError):
        sp.run_node_sweeps(g, cfg, 1)
    with pytest.raises(sp.GridError):
        sp.CompressedGrid(sp.GridDims(8, 8, 8, ghost=2), sp.FillPattern.constant(0.0))


def test_compressed_upload_download_matches_twogrid(sp):
    """The host-transfer API of the compressed grid (the bench's e2e path) against TwoGrid."""
    import torch
    d = sp.GridDims(40, 24, 50)
    pat = sp.FillPattern.dirichlet_box("random", d.shape, FACES, seed=9)
    src = sp.TwoGrid(d, pat)
    field = torch.from_numpy(src.full_view()).pin_memory()
    c = sp.CompressedGrid(d, sp.FillPattern.constant(0.0), chunk=16)
    sp.sweeps(c, 3, depth=3)                 # move the box first: upload must land at the offset
    c.upload(field)
    sp.sweeps(c, 10, depth=2)
    sp.sweeps(src, 10, depth=2)
    assert _bitwise(c.download().numpy(), src.interior())


# --- the reference's compressed-grid API (slack honoured as given) -------------------
# R = /root/reference/pkg; mirrors R/tests/test_kernel.py:126-145, R/tests/test_grid.py:68-90,
# R/tests/test_pipeline.py:179-202 on the device, checked against the oracle.

def _ref_oracle(O, shape, seed, levels):
    g = O.CGrid(shape, O.BoxPattern("random", seed=seed))
    g.sweeps(levels)
    return g.interior()


def test_update_block_compressed_one_level(sp, O):
    d = sp.GridDims(8, 8, 8)
    g = sp.allocate(d, "compressed", sp.FillPattern.random(3), slack=1)
    assert g.offset == 1 and g.slack == 1
    sp.update_block(g, (0, 0, 0), d.shape, level=1, direction=-1)
    g.shift_origin(-1)
    assert _bitwise(g.interior(), _ref_oracle(O, d.shape, 3, 1))


def test_update_block_compressed_round_trip(sp, O):
    d = sp.GridDims(8, 8, 8)
    g = sp.allocate(d, "compressed", sp.FillPattern.random(29), slack=1)
    sp.update_block(g, (0, 0, 0), d.shape, level=1, direction=-1)
    g.shift_origin(-1)
    sp.update_block(g, (0, 0, 0), d.shape, level=1, direction=+1)
    g.shift_origin(+1)
    assert _bitwise(g.interior(), _ref_oracle(O, d.shape, 29, 2))


def test_update_block_compressed_blocked_levels(sp, O):
    """Two levels of a forward blocked traversal (z, y, x block order, shift -1),
    each block refreshing only the ghost faces it touches; level 2 reads at
    offset - 1 (R/kernel.py:141-147)."""
    from paper_0912_4506_b200.kernel import block_edges
    d = sp.GridDims(13, 11, 9)
    g = sp.allocate(d, "compressed", sp.FillPattern.random(5), slack=3)
    ez, ey, ex = block_edges(9, 4), block_edges(11, 5), block_edges(13, 6)
    for level in (1, 2):
        for z0, z1 in zip(ez[:-1], ez[1:]):
            for y0, y1 in zip(ey[:-1], ey[1:]):
                for x0, x1 in zip(ex[:-1], ex[1:]):
                    sp.update_block(g, (z0, y0, x0), (z1, y1, x1), level=level, direction=-1)
    g.shift_origin(-2)
    assert _bitwise(g.interior(), _ref_oracle(O, d.shape, 5, 2))


def test_compressed_offset_identity_and_room(sp):
    g = sp.allocate(sp.GridDims(5, 5, 5), "compressed", sp.FillPattern.random(9), slack=2)
    before = g.value_at(2, 3, 4)
    g.shift_origin(-1)
    g.shift_origin(+1)
    assert g.value_at(2, 3, 4) == before
    h = sp.allocate(sp.GridDims(4, 4, 4), "compressed", sp.FillPattern.constant(0.0), slack=1)
    with pytest.raises(sp.GridError):
        h.shift_origin(-2)
    with pytest.raises(sp.GridError):
        sp.CompressedGrid(sp.GridDims(4, 4, 4), sp.FillPattern.constant(0.0), slack=-1)
    with pytest.raises(sp.GridError):
        sp.CompressedGrid(sp.GridDims(2, 2, 2), sp.FillPattern.constant(0.0), slack=2 ** 22)
    with pytest.raises(sp.GridError):       # level 3 backwards from offset 1 reads at -1
        sp.update_block(h, (0, 0, 0), (4, 4, 4), level=3, direction=-1)
    with pytest.raises(sp.GridError):       # the write at offset 2 escapes slack 1
        sp.update_block(h, (0, 0, 0), (4, 4, 4), level=1, direction=+1)


@pytest.mark.parametrize("depth", [1, 2, 4])
def test_compressed_pipeline_matches_oracle(sp, O, depth):
    d = sp.GridDims(16, 16, 16)
    cfg = sp.PipelineConfig(teams=1, team_size=2, updates_per_thread=2, block=(16, 8, 8),
                            storage="compressed", depth=depth)
    g = sp.allocate(d, "compressed", sp.FillPattern.random(41), slack=cfg.levels_per_sweep)
    sp.run_node_sweeps(g, cfg, 3)            # odd sweep count exercises both directions
    assert g.offset == 0                     # -U, +U, -U from slack = U
    assert _bitwise(g.interior(), _ref_oracle(O, d.shape, 41, 12))


def test_compressed_needs_slack(sp):
    cfg = sp.PipelineConfig(teams=1, team_size=2, updates_per_thread=2, storage="compressed")
    g = sp.allocate(sp.GridDims(8, 8, 8), "compressed", sp.FillPattern.constant(0.0), slack=2)
    with pytest.raises(sp.ScheduleError):
        sp.run_node_sweeps(g, cfg, 1)


def test_dump_compressed_logical_view(sp):
    import io
    g = sp.allocate(sp.GridDims(3, 3, 3), "compressed", sp.FillPattern.linear(), slack=2)
    buf = io.StringIO()
    sp.dump_field(g, buf)
    buf.seek(0)
    dims, arr = sp.load_field(buf)
    assert dims.ghost == 1
    assert arr[1, 1, 1] == 0.0 and arr[3, 3, 3] == 6.0


def test_native_compressed_shift_origin_then_sweep(sp, O):
    """Device-native slack: an origin move without data movement is legal; the
    next pass reads at the moved origin (as the reference would)."""
    d = sp.GridDims(20, 12, 40)
    g = sp.CompressedGrid(d, sp.FillPattern.random(4), chunk=16)
    sp.sweeps(g, 4, depth=2)
    ref = _ref_oracle(O, d.shape, 4, 4)
    assert _bitwise(g.interior(), ref)
    g.shift_origin(-1)
    g.shift_origin(+1)
    sp.sweeps(g, 3, depth=3)
    assert _bitwise(g.interior(), _ref_oracle(O, d.shape, 4, 7))
