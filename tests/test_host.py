"""Host-side logic (no GPU): API mirrors, schedules, decomposition geometry,
and the C ABI library's exported surface."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol(sp):
    hdr = open(os.path.join(ROOT, "include", "stencilpipe_b200.h")).read()
    declared = set(re.findall(r"^\w[\w\s\*]*?\b(sp_\w+)\(", hdr, flags=re.M))
    assert declared == set(sp._native.EXPORTS)
    L = sp._native.load_library()
    for name in declared:
        assert hasattr(L, name), name
    assert L.sp_version() == 1


def test_layout_policy(sp):
    L = sp._native.load_library()
    lay = sp._native.Layout()
    n = ctypes.c_int64()
    assert L.sp_layout_make(1024, 1024, 1024, 1, 1, 1, 0, ctypes.byref(lay), ctypes.byref(n)) == 0
    x_off = lay.origin - lay.gz * lay.pz - lay.gy * lay.py
    assert (lay.origin * 8) % 128 == 0 and (lay.py * 8) % 128 == 0
    assert x_off >= lay.gx and x_off + lay.nx + lay.gx <= lay.py
    assert n.value == lay.pz * (1024 + 2)
    # fp32: 128-byte aligned rows as well
    assert L.sp_layout_make(33, 18, 20, 1, 1, 4, 1, ctypes.byref(lay), ctypes.byref(n)) == 0
    assert (lay.origin * 4) % 128 == 0 and (lay.py * 4) % 16 == 0
    # GridError on bad extents (R/grid.py:36-41)
    assert L.sp_layout_make(0, 4, 4, 1, 1, 1, 0, ctypes.byref(lay), ctypes.byref(n)) == 1
    assert b"interior extents" in L.sp_last_error()


def test_griddims_mirror(sp):
    d = sp.GridDims(4, 5, 6, ghost=2)
    assert d.shape == (6, 5, 4) and d.alloc_shape == (10, 9, 8)
    with pytest.raises(sp.GridError):
        sp.GridDims(0, 4, 4)
    with pytest.raises(sp.GridError):
        sp.GridDims(4, 4, 4, ghost=0)
    with pytest.raises(sp.GridError):
        sp.FillPattern("nope")


def test_pipeline_config_mirror(sp):
    cfg = sp.PipelineConfig(teams=2, team_size=4, updates_per_thread=2)
    assert cfg.levels_per_sweep == 16 and cfg.n_threads == 8
    for bad in [dict(teams=0), dict(min_dist=0), dict(max_dist=0), dict(sync="x"),
                dict(storage="x"), dict(depth=9)]:
        with pytest.raises(ValueError):
            sp.PipelineConfig(**bad)
    assert sp.default_block_size(sp.GridDims(48, 48, 48), sp.PipelineConfig()) == (48, 16, 16)


def test_domains_to_passes(sp):
    from paper_0912_4506_b200.pipeline import domains_to_passes
    # rank 1 of 4, h=4, z-slab: z ranges (-3,19),(-2,18),(-1,17),(0,16)
    doms = [((-3, 0, 0), (19, 8, 8)), ((-2, 0, 0), (18, 8, 8)), ((-1, 0, 0), (17, 8, 8)),
            ((0, 0, 0), (16, 8, 8))]
    assert domains_to_passes(doms, 4, 4) == [(4, (0, 0, 0), (16, 8, 8), (1, 0, 0), (1, 0, 0))]
    assert domains_to_passes(doms, 4, 3) == [(3, (-1, 0, 0), (17, 8, 8), (1, 0, 0), (1, 0, 0)),
                                             (1, (0, 0, 0), (16, 8, 8), (1, 0, 0), (1, 0, 0))]
    plain = [((0, 0, 0), (8, 8, 8))] * 5
    assert domains_to_passes(plain, 5, 2) == [(2, (0, 0, 0), (8, 8, 8), (0, 0, 0), (0, 0, 0))] * 2 + \
        [(1, (0, 0, 0), (8, 8, 8), (0, 0, 0), (0, 0, 0))]
    with pytest.raises(sp.ScheduleError):
        domains_to_passes([((0, 0, 0), (8, 8, 8)), ((-1, 0, 0), (8, 8, 8))], 2, 2)


def test_decomposition_geometry(sp):
    from paper_0912_4506_b200.decomp import _split, face_flags, level_domains_for_rank
    assert _split(10, 3) == [(0, 4), (4, 7), (7, 10)]
    d = sp.decompose(sp.GridDims(16, 16, 64), 4, (1, 1, 4), 4)
    assert d.ranges(1) == ((16, 32), (0, 16), (0, 16))
    assert level_domains_for_rank(d, 1, 4) == [((-3, 0, 0), (19, 16, 16)), ((-2, 0, 0), (18, 16, 16)),
                                               ((-1, 0, 0), (17, 16, 16)), ((0, 0, 0), (16, 16, 16))]
    assert face_flags(d, 0) == ((0, 0, 0), (1, 0, 0))
    assert face_flags(d, 3) == ((1, 0, 0), (0, 0, 0))
    with pytest.raises(sp.DecompositionError):
        sp.decompose(sp.GridDims(16, 16, 16), 3, (1, 1, 2), 1)
    with pytest.raises(sp.DecompositionError):
        sp.decompose(sp.GridDims(16, 16, 6), 2, (1, 1, 2), 4)   # 3 cells per rank < h


def test_plane_spans_are_contiguous_planes(sp):
    import torch
    from paper_0912_4506_b200.decomp import plane_spans
    L = sp._native.load_library()
    lay = sp._native.Layout()
    n = ctypes.c_int64()
    L.sp_layout_make(5, 4, 10, 1, 1, 3, 0, ctypes.byref(lay), ctypes.byref(n))
    buf = torch.arange(n.value, dtype=torch.float64)
    s_lo, s_hi, r_lo, r_hi = plane_spans(buf, lay, 3)
    assert s_lo.numel() == 3 * lay.pz
    assert int(s_lo[0]) == 3 * lay.pz                 # plane z=0 follows 3 ghost planes
    assert int(r_lo[0]) == 0                          # planes -3..-1
    assert int(s_hi[0]) == (3 + 10 - 3) * lay.pz
    assert int(r_hi[0]) == (3 + 10) * lay.pz


def test_stencil_point_and_compare(sp):
    assert sp.stencil_point(1.0, 2.0, 3.0, 4.0, 0.0, 5.0) == 15.0 / 6.0
    a = np.random.default_rng(0).random((4, 4, 4))
    assert sp.compare(a, a.copy()).bitwise
    assert sp.REL_TOL == 1e-13


def test_no_cpu_fallback(sp, monkeypatch):
    import torch
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(sp.NativeUnavailable):
        sp.TwoGrid(sp.GridDims(4, 4, 4), sp.FillPattern.random(0))


def test_product_never_imports_oracle():
    """The checker stays test infrastructure: no product file imports or loads it."""
    pkg = os.path.join(ROOT, "paper_0912_4506_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, flags=re.M), f
                assert "libjacobi_oracle" not in txt, f


def test_load_field_reads_reference_dump(sp):
    """A dump written by the reference itself (R/grid.py:280-289) parses here."""
    import io
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        from stencilpipe.grid import FillPattern, GridDims, TwoGrid, dump_field
    except ImportError:
        pytest.skip("reference package not present")
    g = TwoGrid(GridDims(3, 4, 5), FillPattern.random(9))
    buf = io.StringIO()
    dump_field(g, buf)
    buf.seek(0)
    dims, field = sp.load_field(buf)
    assert (dims.nx, dims.ny, dims.nz, dims.ghost) == (3, 4, 5, 1)
    assert np.array_equal(field.view(np.uint64), g.current.view(np.uint64))
    pat = sp.ArrayPattern(field, 1)
    assert np.array_equal(pat.evaluate((0, 0, 0), (5, 4, 3)), g.interior())


def test_schedule_validation_matches_reference(sp):
    """check_schedule raises exactly where the reference's build_schedule does."""
    import sys
    from paper_0912_4506_b200.pipeline import check_schedule
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        from stencilpipe import pipeline as rp
        from stencilpipe.grid import GridDims as RDims
    except ImportError:
        pytest.skip("reference package not present")
    cases = [((8, 8, 8), dict(teams=1, team_size=1, updates_per_thread=4, block=(8, 2, 2))),
             ((8, 8, 8), dict(teams=1, team_size=2, updates_per_thread=2, block=(8, 4, 4))),
             ((24, 24, 24), dict(teams=2, team_size=4, updates_per_thread=2, block=(24, 16, 16))),
             ((12, 10, 9), dict(teams=1, team_size=1, updates_per_thread=5, block=(12, 3, 3))),
             ((4, 4, 4), dict(teams=1, team_size=1, updates_per_thread=5)),
             ((16, 16, 16), dict(teams=1, team_size=2, updates_per_thread=1, block=(16, 1, 1)))]
    for (nx, ny, nz), kw in cases:
        ref_err = ours_err = None
        try:
            rp.build_schedule(RDims(nx, ny, nz), rp.PipelineConfig(**kw))
        except rp.ScheduleError:
            ref_err = True
        try:
            check_schedule(sp.GridDims(nx, ny, nz), sp.PipelineConfig(**kw))
        except sp.ScheduleError:
            ours_err = True
        assert ref_err == ours_err, ((nx, ny, nz), kw)


def test_describe_variant_defaults(sp):
    """The variant table's defaults (host-only introspection, no device needed)."""
    N = sp._native
    d = {(dt, T): N.describe_variant(dt, T) for dt in (N.SP_F64, N.SP_F32) for T in range(1, 9)}
    assert "2 CTA/SM" in d[(N.SP_F64, 2)] and "8 warps x 4 rows" in d[(N.SP_F64, 2)]
    assert "16 warps x 3 rows" in d[(N.SP_F64, 3)] and "tensor memory" in d[(N.SP_F64, 3)]
    assert "12 warps x 5 rows" in d[(N.SP_F64, 4)] and "z-queue (v[p-1], v[p])" in d[(N.SP_F64, 4)]
    assert "12 warps x 6 rows" in d[(N.SP_F32, 4)] and "tensor memory" in d[(N.SP_F32, 4)]
    for T in range(5, 9):
        assert "tensor memory" in d[(N.SP_F64, T)] and "tensor memory" in d[(N.SP_F32, T)]
    assert "64x64 footprint" in d[(N.SP_F32, 8)]
    with pytest.raises(ValueError):
        N.describe_variant(N.SP_F64, 9)


def test_cuda_engine_default_depth():
    """SlabRunner(depth=None) asks the engine (the method sat on PeerBuffer)."""
    from paper_0912_4506_b200.dist import CudaEngine
    from paper_0912_4506_b200.pipeline import DEFAULT_DEPTH
    from paper_0912_4506_b200 import _native as N

    class G:
        sp_dtype = N.SP_F64
    assert CudaEngine().default_depth(G()) == DEFAULT_DEPTH[N.SP_F64]
    G.sp_dtype = N.SP_F32
    assert CudaEngine().default_depth(G()) == DEFAULT_DEPTH[N.SP_F32]


def test_k2_sass_uses_tma_and_tensor_memory_and_no_fma():
    """The fp64 T=4 K2 unit as built: TMA loads, tensor-memory ld/st (tq_kernel's z-queue) and
    not one DFMA (bit-exactness with the reference's add/multiply order forbids contraction).
    Reads the object the build left in-tree; skips where it or cuobjdump is absent."""
    import shutil
    import subprocess
    obj = os.path.join(ROOT, "paper_0912_4506_b200", "build", "obj", "tb_double_4.o")
    if not os.path.exists(obj) or not shutil.which("cuobjdump"):
        pytest.skip("no build objects / cuobjdump here")
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True, check=True).stdout
    count = {m: len(re.findall(r"\b%s\b" % m, sass)) for m in ("UTMALDG", "LDTM", "STTM", "DADD", "DMUL", "DFMA")}
    assert count["UTMALDG"] > 0 and count["LDTM"] > 0 and count["STTM"] > 0, count
    assert count["DADD"] > 0 and count["DMUL"] > 0 and count["DFMA"] == 0, count
