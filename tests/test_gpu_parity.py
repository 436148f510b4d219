"""Device parity: every result compared bit-for-bit with the reference goldens
(tests/golden, produced by the reference package itself) or with the pinned
C oracle on identical seeded inputs.

fp64 tolerance: bitwise (north_star: <=1e-13 relative, bit-exact when the
reference's summation order is kept -- it is).  fp32 tolerance: <=1e-5
relative per north_star, and we additionally assert bitwise.
"""

import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

Z1 = (1.0, 0.0, 0.0, 0.0, 0.0, 0.0)
C3F = (1.0, 0.0, 0.5, 0.0, 0.25, 0.0)


def dims_of(sp, shape, ghost=1):
    return sp.GridDims(shape[2], shape[1], shape[0], ghost)


def oracle_run(O, shape, kind, seed, faces, levels, dtype=np.float64):
    g = O.CGrid(shape, O.BoxPattern(kind, seed=seed, faces=faces,
                                    global_shape=shape if faces else None), dtype=dtype)
    g.sweeps(levels)
    return g


def bitwise(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))


# ---- K3 fill ------------------------------------------------------------------

def test_fill_matches_reference_hash(sp, kat):
    pat = sp.FillPattern.random(0)
    for key, bits in kat["random0_bits"].items():
        c = tuple(int(v) for v in key.split(","))
        v = pat.evaluate(c, tuple(i + 1 for i in c))[0, 0, 0]
        assert np.float64(v).view(np.uint64) == bits, key


def test_fill_faced_box_matches_reference(sp, ref_fields):
    shape = (17, 19, 21)
    g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.dirichlet_box("random", shape, C3F))
    assert bitwise(g.full_view(), ref_fields["c3like_21x19x17_full0"])
    # B is a copy of A including the ghost shell (R/grid.py:132-133)
    assert bitwise(g.other.cpu().numpy(), g.full_view())


def test_c1_initial_digest(sp, kat):
    shape = (128, 128, 128)
    g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.dirichlet_box("random", shape, Z1))
    assert g.digest() == kat["c1_digest_l0"]


# ---- reference known answers ------------------------------------------------------

def test_hotplate_first_sweep_golden(sp, ref_fields):
    g = sp.TwoGrid(sp.GridDims(4, 4, 4), sp.FillPattern.hotplate())
    sp.sweep_naive(g)
    expected = np.zeros((4, 4, 4))
    expected[:, :, 0] = 1.0 / 6.0
    assert bitwise(g.interior(), expected)
    assert bitwise(g.interior(), ref_fields["hotplate4_l1"])


@pytest.mark.parametrize("kind", ["constant", "linear"])
def test_fixed_points(sp, kind):
    pat = sp.FillPattern.constant(3.5) if kind == "constant" else sp.FillPattern.linear()
    g = sp.TwoGrid(sp.GridDims(16, 16, 16), pat)
    start = g.interior().copy()
    sp.sweeps(g, 64, depth=4)
    assert bitwise(g.interior(), start)


def test_trajectory_every_level(sp, ref_fields):
    traj = ref_fields["r11_16_traj"]
    g = sp.TwoGrid(sp.GridDims(16, 16, 16), sp.FillPattern.random(11))
    assert bitwise(g.interior(), traj[0])
    for lv in range(1, 9):
        sp.sweep_naive(g)
        assert bitwise(g.interior(), traj[lv]), lv


@pytest.mark.parametrize("depth", range(1, 9))
def test_trajectory_temporal_blocking(sp, ref_fields, depth):
    traj = ref_fields["r11_16_traj"]
    for levels in (depth, 8):
        g = sp.TwoGrid(sp.GridDims(16, 16, 16), sp.FillPattern.random(11))
        sp.sweeps(g, levels, depth=depth)
        assert bitwise(g.interior(), traj[levels]), (depth, levels)


@pytest.mark.parametrize("depth", [1, 2, 3, 4, 5, 8])
def test_ragged_and_degenerate(sp, ref_fields, depth):
    g = sp.TwoGrid(sp.GridDims(9, 7, 5), sp.FillPattern.random(2))
    sp.sweeps(g, 7, depth=depth)
    assert bitwise(g.interior(), ref_fields["r2_9x7x5_l7"])
    g = sp.TwoGrid(sp.GridDims(1, 3, 2), sp.FillPattern.random(3))
    sp.sweeps(g, 3, depth=depth)
    assert bitwise(g.interior(), ref_fields["r3_1x3x2_l3"])


def test_pipeline_config_u16(sp, ref_fields):
    g = sp.TwoGrid(sp.GridDims(24, 24, 24), sp.FillPattern.random(11))
    cfg = sp.PipelineConfig(teams=2, team_size=4, updates_per_thread=2, block=(24, 16, 16))
    sp.run_node_sweeps(g, cfg, 1)
    assert bitwise(g.interior(), ref_fields["r11_24_pipe_u16"])


@pytest.mark.parametrize("depth", range(1, 9))
def test_faced_boxes(sp, ref_fields, depth):
    shape = (20, 18, 33)
    g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.dirichlet_box("random", shape, Z1))
    sp.sweeps(g, 12, depth=depth)
    assert bitwise(g.interior(), ref_fields["c1like_33x18x20_l12"])
    shape = (17, 19, 21)
    g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.dirichlet_box("random", shape, C3F))
    sp.sweeps(g, 9, depth=depth)
    assert bitwise(g.interior(), ref_fields["c3like_21x19x17_l9"])


@pytest.mark.parametrize("depth", range(1, 9))
def test_float32(sp, ref_fields, depth):
    shape = (24, 20, 36)
    pat = sp.FillPattern.dirichlet_box("random_pm1", shape, (0.0,) * 6)
    g = sp.TwoGrid(dims_of(sp, shape), pat, dtype=np.float32)
    sp.sweeps(g, 10, depth=depth)
    got, ref = g.interior(), ref_fields["c4like_f32_36x20x24_l10"]
    assert got.dtype == np.float32
    cmp = sp.compare(ref, got, tol=sp.F32_REL_TOL)   # north_star fp32 tolerance 1e-5
    assert cmp.passed, str(cmp)
    assert cmp.bitwise, str(cmp)


def test_ghost_shell_never_written(sp):
    shape = (13, 11, 19)
    g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.dirichlet_box("random", shape, C3F))
    a0 = g.current.cpu().numpy().copy()
    sp.sweeps(g, 11, depth=4)
    for arr in (g.current.cpu().numpy(), g.other.cpu().numpy()):
        shell = np.ones(arr.shape, bool)
        shell[1:-1, 1:-1, 1:-1] = False
        assert bitwise(arr[shell], a0[shell])


def test_update_block_level_parity(sp, O):
    shape = (6, 6, 6)
    g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.random(13))
    sp.update_block(g, (0, 0, 0), shape, level=1)
    sp.update_block(g, (0, 0, 0), shape, level=2)
    ref = oracle_run(O, shape, "random", 13, None, 2)
    assert bitwise(g.interior(), ref.interior())


def test_update_block_subbox_matches_oracle(sp, O):
    shape = (9, 10, 11)
    g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.random(5))
    ref = O.CGrid(shape, O.BoxPattern("random", seed=5))
    for lo, hi in [((0, 0, 0), (4, 10, 11)), ((2, 3, 1), (7, 9, 5)), ((0, 0, 0), (1, 1, 1))]:
        sp.update_block(g, lo, hi, level=1)
        ref.update_region(lo, hi, level=1)
        assert bitwise(g.other.cpu().numpy(), ref.b if ref.active == 0 else ref.a)


def test_update_block_bounds(sp):
    g = sp.TwoGrid(sp.GridDims(4, 4, 4), sp.FillPattern.constant(0.0))
    with pytest.raises(sp.GridError):
        sp.update_block(g, (0, 0, 0), (5, 4, 4))
    with pytest.raises(sp.GridError):
        sp.update_block(g, (2, 0, 0), (1, 4, 4))


def test_schedule_errors(sp):
    g = sp.TwoGrid(sp.GridDims(4, 4, 4), sp.FillPattern.constant(0.0))
    with pytest.raises(sp.ScheduleError):
        sp.run_node_sweeps(g, sp.PipelineConfig(teams=1, team_size=1, updates_per_thread=5), 1)


# ---- randomised parity vs the pinned C oracle ----------------------------------------

CASES = [((1, 1, 1), 3, 1), ((2, 3, 5), 5, 2), ((17, 32, 64), 9, 4), ((40, 70, 130), 8, 8),
         ((33, 31, 29), 7, 3), ((64, 24, 56), 8, 4), ((5, 100, 9), 6, 6), ((70, 65, 190), 10, 5)]


@pytest.mark.parametrize("shape,levels,depth", CASES)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_random_shapes_vs_oracle(sp, O, shape, levels, depth, dtype):
    seed = sum(shape) * 7 + levels
    faces = (0.3, -1.0, 2.0, 0.0, 1.0, -0.5)
    g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.dirichlet_box("random", shape, faces, seed=seed),
                   dtype=dtype)
    sp.sweeps(g, levels, depth=depth)
    ref = oracle_run(O, shape, "random", seed, faces, levels, dtype=dtype)
    assert bitwise(g.interior(), ref.interior()), (shape, levels, depth)


# ---- sub-box passes (the overlap split) --------------------------------------------

@pytest.mark.parametrize("T", [1, 3, 4, 8])
def test_partial_boxes_compose(sp, T):
    shape = (40, 30, 50)
    pat = sp.FillPattern.dirichlet_box("random", shape, C3F)
    full = sp.TwoGrid(dims_of(sp, shape), pat)
    sp.pipeline.run_pass(full, T, (0, 0, 0), shape)
    split = sp.TwoGrid(dims_of(sp, shape), pat)
    nz = shape[0]
    for olo, ohi in [((0, 0, 0), (T, 30, 50)), ((nz - T, 0, 0), (nz, 30, 50)),
                     ((T, 0, 0), (nz - T, 30, 50))]:
        sp.pipeline.run_pass(split, T, (0, 0, 0), shape, out_lo=olo, out_hi=ohi)
    assert bitwise(full.other.cpu().numpy(), split.other.cpu().numpy())


# ---- distributed z-slabs (single process, ranks share the GPU) -----------------------

@pytest.mark.parametrize("case", ["dist_P2_h1_s3", "dist_P2_h4_s2", "dist_P3_h2_s2",
                                  "dist_P4_h4_s2", "dist_P4_h8_s1"])
def test_distributed_matches_reference(sp, kat, ref_fields, case):
    c = kat["dist_cases"][case]
    gd = sp.GridDims(12, 10, 40)
    pat = sp.FillPattern.dirichlet_box("random", (40, 10, 12), Z1)
    gathered, fields = sp.run_distributed(gd, pat, (1, 1, c["P"]), cfg=None,
                                          outer_steps=c["steps"], h=c["h"])
    assert bitwise(gathered, ref_fields[case])


def test_distributed_pipelined_depth_split(sp, ref_fields):
    # h=8 with depth 3: three passes per outer step over extended domains
    gd = sp.GridDims(12, 10, 40)
    pat = sp.FillPattern.dirichlet_box("random", (40, 10, 12), Z1)
    cfg = sp.PipelineConfig(teams=1, team_size=4, updates_per_thread=2, depth=3)
    gathered, _ = sp.run_distributed(gd, pat, (1, 1, 4), cfg, outer_steps=1)
    assert bitwise(gathered, ref_fields["dist_P4_h8_s1"])


# Multi-axis layouts with the x -> y -> z extended-slab exchange;
# the cases restate the reference's own tests (test_decomp.py:169-204).

def _oracle_interior(O, shape, kind, seed, levels):
    g = O.CGrid(shape, O.BoxPattern(kind, seed=seed))
    g.sweeps(levels)
    return g.interior()


def test_multi_axis_serial_matches_oracle(sp, O):
    gathered, _ = sp.run_distributed(sp.GridDims(16, 16, 16), sp.FillPattern.random(37), (2, 2, 1),
                                     cfg=None, outer_steps=3, h=2)
    assert bitwise(gathered, _oracle_interior(O, (16, 16, 16), "random", 37, 6))


def test_multi_axis_pipelined_matches_oracle(sp, O):
    cfg = sp.PipelineConfig(teams=1, team_size=2, updates_per_thread=2, block=(24, 8, 8))
    gathered, _ = sp.run_distributed(sp.GridDims(24, 24, 24), sp.FillPattern.random(43), (2, 1, 2),
                                     cfg, outer_steps=2)
    assert bitwise(gathered, _oracle_interior(O, (24, 24, 24), "random", 43, 8))


def test_multi_axis_hotplate_walls(sp, O):
    gathered, _ = sp.run_distributed(sp.GridDims(16, 16, 16), sp.FillPattern.hotplate(), (2, 1, 1),
                                     cfg=None, outer_steps=2, h=4)
    assert bitwise(gathered, _oracle_interior(O, (16, 16, 16), "hotplate", 0, 8))


def test_multi_axis_all_three_axes(sp, O):
    shape = (16, 18, 20)
    faces = (1.0, 0.0, 0.5, 0.0, 0.25, 0.0)
    pat = sp.FillPattern.dirichlet_box("random", shape, faces, seed=0)
    gathered, _ = sp.run_distributed(sp.GridDims(20, 18, 16), pat, (2, 3, 2), cfg=None,
                                     outer_steps=2, h=3)
    ref = O.CGrid(shape, O.BoxPattern("random", seed=0, faces=faces, global_shape=shape))
    ref.sweeps(6)
    assert bitwise(gathered, ref.interior())


def test_shuffled_phase_order_breaks_corners(sp, O):
    gd, pat = sp.GridDims(16, 16, 16), sp.FillPattern.random(47)
    good, _ = sp.run_distributed(gd, pat, (2, 2, 1), cfg=None, outer_steps=2, h=2, order=("x", "y", "z"))
    bad, _ = sp.run_distributed(gd, pat, (2, 2, 1), cfg=None, outer_steps=2, h=2, order=("y", "x", "z"))
    ref = _oracle_interior(O, (16, 16, 16), "random", 47, 4)
    assert bitwise(good, ref)
    assert not sp.compare(ref, bad).passed


# ---- C1: the BASELINE parity config ----------------------------------------------------

def test_c1_full_grid_vs_reference(sp, kat, ref_fields):
    shape = (128, 128, 128)
    g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.dirichlet_box("random", shape, Z1))
    cfg = sp.PipelineConfig(teams=1, team_size=1, updates_per_thread=4, depth=4)   # T=4
    sp.run_node_sweeps(g, cfg, 25)                                                 # 100 sweeps
    assert g.digest() == kat["c1_digest_l100"]
    inner = g.interior()
    assert bitwise(inner[kat["c1_planes_index"]], ref_fields["c1_planes_l100"])


@pytest.mark.parametrize("shape_id", list(range(1, 133)))
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_every_cta_shape(sp, O, shape_id, dtype):
    lib = sp._native.lib()
    lib.sp_set_tuning(shape_id, 0)
    try:
        for shape, levels, depth in [((40, 70, 130), 8, 4), ((33, 31, 29), 7, 3), ((70, 65, 190), 10, 2),
                                     ((20, 18, 33), 8, 8), ((9, 80, 70), 5, 5)]:
            seed = sum(shape) + levels
            faces = (0.3, -1.0, 2.0, 0.0, 1.0, -0.5)
            g = sp.TwoGrid(dims_of(sp, shape),
                           sp.FillPattern.dirichlet_box("random", shape, faces, seed=seed), dtype=dtype)
            sp.sweeps(g, levels, depth=depth)
            ref = oracle_run(O, shape, "random", seed, faces, levels, dtype=dtype)
            assert bitwise(g.interior(), ref.interior()), (shape_id, shape, depth)
    finally:
        lib.sp_set_tuning(0, 0)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_k1_streaming_kernel(sp, O, dtype):
    """K1 (L1-streaming, no shared memory) for single-level sweeps and sub-boxes."""
    lib = sp._native.lib()
    lib.sp_set_tuning(-1, 0)
    try:
        for shape, levels in [((9, 7, 5), 4), ((33, 70, 129), 3), ((1, 1, 1), 2), ((64, 24, 56), 5)]:
            faces = (0.3, -1.0, 2.0, 0.0, 1.0, -0.5)
            g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.dirichlet_box("random", shape, faces, seed=3),
                           dtype=dtype)
            sp.sweeps(g, levels, depth=1)
            ref = oracle_run(O, shape, "random", 3, faces, levels, dtype=dtype)
            assert bitwise(g.interior(), ref.interior()), shape
        shape = (9, 10, 11)
        g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.random(5), dtype=dtype)
        ref = O.CGrid(shape, O.BoxPattern("random", seed=5), dtype=dtype)
        for lo, hi in [((2, 3, 1), (7, 9, 5)), ((0, 0, 3), (9, 10, 11))]:
            sp.update_block(g, lo, hi, level=1)
            ref.update_region(lo, hi, level=1)
            assert bitwise(g.other.cpu().numpy(), ref.b if ref.active == 0 else ref.a)
    finally:
        lib.sp_set_tuning(0, 0)


def test_dump_load_round_trip(sp, O):
    import io
    shape = (5, 6, 7)
    g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.random(21))
    sp.sweeps(g, 3, depth=3)
    buf = io.StringIO()
    sp.dump_field(g, buf)
    buf.seek(0)
    dims, field = sp.load_field(buf)
    h = sp.TwoGrid(dims, sp.ArrayPattern(field, dims.ghost))
    assert bitwise(h.full_view(), g.full_view())
    sp.sweeps(g, 2, depth=2)
    sp.sweeps(h, 2, depth=1)
    ref = oracle_run(O, shape, "random", 21, None, 5)
    assert bitwise(g.interior(), ref.interior()) and bitwise(h.interior(), ref.interior())


def test_device_oracle_api(sp, ref_fields):
    """verify.oracle / oracle_trajectory keep the reference's names and results."""
    traj = sp.oracle_trajectory(sp.GridDims(16, 16, 16), sp.FillPattern.random(11), 8)
    for lv, st in enumerate(traj):
        assert bitwise(st, ref_fields["r11_16_traj"][lv]), lv
    g = sp.oracle(sp.GridDims(4, 4, 4), sp.FillPattern.hotplate(), 1)
    assert bitwise(g.interior(), ref_fields["hotplate4_l1"])
    # the temporally blocked engine agrees with the one-level engine
    blocked = sp.TwoGrid(sp.GridDims(16, 16, 16), sp.FillPattern.random(11))
    sp.sweeps(blocked, 8, depth=4)
    assert sp.compare(sp.oracle(sp.GridDims(16, 16, 16), sp.FillPattern.random(11), 8), blocked).bitwise


@pytest.mark.parametrize("sched", [(0, 0), (1, 0), (1, 3), (0, 5)])
def test_unit_schedules(sp, O, sched):
    """Static/dynamic unit claiming and strip orders give identical fields."""
    lib = sp._native.lib()
    prev = lib.sp_set_schedule(*sched)
    try:
        for shape, levels, depth, chunks in [((40, 70, 130), 8, 4, 0), ((70, 65, 190), 10, 2, 7),
                                             ((33, 31, 29), 6, 3, 29), ((5, 200, 300), 4, 2, 1)]:
            lib.sp_set_tuning(0, chunks)
            faces = (0.3, -1.0, 2.0, 0.0, 1.0, -0.5)
            g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.dirichlet_box("random", shape, faces, seed=5))
            sp.sweeps(g, levels, depth=depth)
            ref = oracle_run(O, shape, "random", 5, faces, levels)
            assert bitwise(g.interior(), ref.interior()), (sched, shape, chunks)
    finally:
        lib.sp_set_tuning(0, 0)
        lib.sp_set_schedule(prev // 1000, prev % 1000)


def test_dynamic_counter_rearms(sp, O):
    """More launches than unit counters: every counter must be back at zero for reuse."""
    shape = (6, 20, 70)
    faces = (1.0, 0.0, 0.5, 0.0, 0.25, 0.0)
    g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.dirichlet_box("random", shape, faces, seed=9))
    levels = 2 * 1100
    sp.sweeps(g, levels, depth=2)
    ref = oracle_run(O, shape, "random", 9, faces, levels)
    assert bitwise(g.interior(), ref.interior())


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_upload_download_round_trip(sp, O, dtype):
    """TwoGrid.upload / download (one pitched DMA each) against the oracle."""
    import torch
    shape = (19, 23, 37)
    faces = (0.3, -1.0, 2.0, 0.0, 1.0, -0.5)
    src = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.dirichlet_box("random", shape, faces, seed=4),
                     dtype=dtype)
    field = src.full_view()                                  # dense ghosted host field
    g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.constant(7.0), dtype=dtype)
    pinned = torch.from_numpy(field.copy()).pin_memory()
    g.upload(pinned)
    assert bitwise(g.full_view(), field)
    assert bitwise(g.other.cpu().numpy(), field)              # B = copy of A
    sp.sweeps(g, 6, depth=3)
    out = torch.empty(shape, dtype=g.torch_dtype).pin_memory()
    g.download(out)
    torch.cuda.synchronize()
    ref = oracle_run(O, shape, "random", 4, faces, 6, dtype=dtype)
    assert bitwise(out.numpy(), ref.interior())
    assert bitwise(g.download().numpy(), ref.interior())     # fresh pinned tensor, synchronised
    with pytest.raises(sp.GridError):
        g.upload(np.zeros((3, 3, 3), dtype=dtype))


@pytest.mark.parametrize("shape_id", [24, 25, 26, 27])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_level_split_pipeline(sp, O, shape_id, dtype):
    """Level-split K2 (levels 1..T/2 on one CTA, T/2+1..T on its cluster peer, planes handed
    over by st.async): ragged boxes with walls, depths 4/6/8, and sub-box output passes."""
    lib = sp._native.lib()
    lib.sp_set_tuning(shape_id, 0)
    try:
        for shape, levels, depth in [((37, 45, 70), 16, 8), ((23, 40, 66), 12, 6), ((30, 33, 129), 8, 4),
                                     ((9, 17, 20), 8, 8)]:
            faces = (0.7, -0.25, 1.5, 0.0, -1.0, 0.5)
            seed = sum(shape) + depth
            g = sp.TwoGrid(dims_of(sp, shape), sp.FillPattern.dirichlet_box("random", shape, faces, seed=seed),
                           dtype=dtype)
            sp.sweeps(g, levels, depth=depth)
            ref = oracle_run(O, shape, "random", seed, faces, levels, dtype=dtype)
            assert bitwise(g.interior(), ref.interior()), (shape_id, shape, depth)
    finally:
        lib.sp_set_tuning(0, 0)


def test_dynamic_counters_per_stream(sp, O):
    """Many K2 launches in flight on several streams at once (VERDICT r01 weak #8:
    the counter pool was round-robin per device); every stream's result is exact."""
    import torch
    shape = (40, 30, 70)
    pat = sp.FillPattern.random(21)
    streams = [torch.cuda.Stream() for _ in range(6)]
    grids = [sp.TwoGrid(sp.GridDims(70, 30, 40), pat) for _ in streams]
    torch.cuda.synchronize()
    for _ in range(3):
        for s, g in zip(streams, grids):
            with torch.cuda.stream(s):
                sp.sweeps(g, 8, depth=2)
    torch.cuda.synchronize()
    ref = O.CGrid(shape, O.BoxPattern("random", seed=21))
    ref.sweeps(24)
    for g in grids:
        assert np.array_equal(g.interior().view(np.uint64), ref.interior().view(np.uint64))


def test_tuning_override_is_thread_local(sp):
    import threading
    lib = sp._native.lib()
    lib.sp_set_tuning(0, 0)
    seen = {}

    def other():
        seen["prev"] = lib.sp_set_tuning(3, 7)     # another thread: starts from the defaults
        lib.sp_set_tuning(0, 0)
    lib.sp_set_tuning(5, 2)
    t = threading.Thread(target=other)
    t.start()
    t.join()
    assert seen["prev"] == 0                        # (0+0)*1000 + 0: untouched by this thread's 5/2
    assert lib.sp_set_tuning(0, 0) == 5 * 1000 + 2
