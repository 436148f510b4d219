"""Temporally blocked node sweeps on the device (drop-in for R/pipeline.py).

The reference's engine runs U = n*t*T levels per node sweep with CPU thread
teams trailing each other over shifted blocks (R/pipeline.py:283-462).  On a
B200 the same schedule is the z-wavefront inside K2: each CTA applies up to 8
levels per pass over HBM, level t lagging level t-1 by one plane.  The
thread/team/sync fields of ``PipelineConfig`` are validated exactly like the
reference (R/pipeline.py:38-68) but have no device meaning; only
``levels_per_sweep`` (U) matters, split into passes of ``depth`` levels.
(R = /root/reference/pkg/src/stencilpipe)
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _native as N
from .grid import GridDims, TwoGrid, _on

# Levels fused per HBM pass when the config does not say: the depth with the
# highest SUSTAINED throughput on B200 (C3 1024^3 fp64, 100 sweeps, tensor-memory
# kernels: T=3 744, T=4 840, T=5 821 GLUP/s -- T <= 3 saturates HBM and runs into the
# board power cap at ~1700 MHz).
DEFAULT_DEPTH = {N.SP_F64: 4, N.SP_F32: 4}
# In-place passes (compressed storage), C3 1024^3 at chunk 64: T=3 662, T=4 791, T=5 728 GLUP/s.
DEFAULT_DEPTH_INPLACE = {N.SP_F64: 4, N.SP_F32: 4}
MAX_DEPTH = 8


class ScheduleError(ValueError):
    """Block/shift geometry cannot tile the domain at every level (R/pipeline.py:30)."""


class PipelineTimeout(RuntimeError):
    """Kept for API parity (R/pipeline.py:34); device runs never spin on the host."""


@dataclass(frozen=True)
class PipelineConfig:
    """Node-sweep configuration (R/pipeline.py:38-68) plus the device pass depth."""
    teams: int = 1
    team_size: int = 1
    updates_per_thread: int = 2
    min_dist: int = 1
    max_dist: int = 4
    team_delay: int = 0
    sync: str = "relaxed"
    block: tuple | None = None
    storage: str = "twogrid"
    spin_timeout: float = 30.0
    depth: int | None = None   # levels fused per HBM pass on the device (1..8)

    def __post_init__(self):
        if min(self.teams, self.team_size, self.updates_per_thread) < 1:
            raise ValueError("teams, team_size, updates_per_thread must be >= 1")
        if self.min_dist < 1 or self.max_dist < self.min_dist or self.team_delay < 0:
            raise ValueError("need d_l >= 1, d_u >= d_l, d_t >= 0")
        if self.sync not in ("barrier", "relaxed"):
            raise ValueError(f"unknown sync mode {self.sync!r}")
        if self.storage not in ("twogrid", "compressed"):
            raise ValueError(f"unknown storage mode {self.storage!r}")
        if self.depth is not None and not 1 <= self.depth <= MAX_DEPTH:
            raise ValueError(f"device pass depth must be in 1..{MAX_DEPTH}")

    @property
    def n_threads(self) -> int:
        return self.teams * self.team_size

    @property
    def levels_per_sweep(self) -> int:
        """U = n * t * T (R/pipeline.py:65-68)."""
        return self.teams * self.team_size * self.updates_per_thread


def default_block_size(dims: GridDims, cfg: PipelineConfig) -> tuple[int, int, int]:
    """Long-x blocks valid for a shift of U-1 (R/pipeline.py:475-481)."""
    U = cfg.levels_per_sweep
    by = dims.ny if dims.ny < 2 * U else max(U, min(16, dims.ny))
    bz = dims.nz if dims.nz < 2 * U else max(U, min(16, dims.nz))
    return (dims.nx, by, bz)


def check_schedule(dims: GridDims, cfg: PipelineConfig, level_domains=None) -> None:
    """The reference's schedule validation (R/pipeline.py:216-243, 187-201).

    The device wavefront does not use blocks, but a configuration the
    reference would reject is rejected here too, with the same ScheduleError:
    U larger than the smallest extent, the wrong number of level domains, or
    block edges that escape a level's domain once shifted by -(tau-1).
    """
    from .kernel import block_edges
    U = cfg.levels_per_sweep
    shape = dims.shape
    if U > min(shape):
        raise ScheduleError(
            f"U={U} updates per node sweep exceed the smallest interior "
            f"extent {min(shape)}; degenerate pipeline")
    if level_domains is None:
        level_domains = [((0, 0, 0), shape)] * U
    elif len(level_domains) != U:
        raise ScheduleError(f"need {U} level domains, got {len(level_domains)}")
    base_lo, base_hi = level_domains[0]
    if cfg.block is None:
        edges = [[base_lo[d], base_hi[d]] for d in range(3)]
    else:
        bx, by, bz = cfg.block
        edges = [[base_lo[d] + e for e in block_edges(base_hi[d] - base_lo[d], b)]
                 for d, b in zip(range(3), (bz, by, bx))]
    for tau in range(1, U + 1):
        shift = -(tau - 1)
        dom_lo, dom_hi = level_domains[tau - 1]
        for d in range(3):
            e = edges[d]
            m = len(e) - 1
            if m == 1:
                continue
            if e[1] + shift < dom_lo[d] or e[m - 1] + shift > dom_hi[d]:
                raise ScheduleError(
                    f"level {tau}: shifted block edges escape domain "
                    f"(dim {d}, shift {shift}); shrink U or enlarge blocks")


def domains_to_passes(level_domains, U: int, depth: int):
    """Split U levels with domains D_1..D_U into device passes.

    The reference only ever builds domains of the form
    D_t = [lo - e_lo*(U-t), hi + e_hi*(U-t)) with e in {0, 1} per side
    (R/decomp.py:192-205; plain interior when e = 0).  Returns a list of
    (T, lo, hi, e_lo, e_hi) with [lo, hi) the pass's final-level domain.
    """
    lo_u, hi_u = (tuple(v) for v in level_domains[-1])
    e_lo = [0, 0, 0]
    e_hi = [0, 0, 0]
    if U > 1:
        lo_1, hi_1 = level_domains[0]
        for d in range(3):
            dl, dh = lo_u[d] - lo_1[d], hi_1[d] - hi_u[d]
            if dl % (U - 1) or dh % (U - 1) or dl // (U - 1) not in (0, 1) \
                    or dh // (U - 1) not in (0, 1):
                raise ScheduleError("level domains are not shrinking extended slabs")
            e_lo[d], e_hi[d] = dl // (U - 1), dh // (U - 1)
    for t, (lo, hi) in enumerate(level_domains, start=1):
        exp_lo = tuple(lo_u[d] - e_lo[d] * (U - t) for d in range(3))
        exp_hi = tuple(hi_u[d] + e_hi[d] * (U - t) for d in range(3))
        if tuple(lo) != exp_lo or tuple(hi) != exp_hi:
            raise ScheduleError(f"level {t} domain {lo}..{hi} breaks the shrinking-slab form")
    passes = []
    done = 0
    while done < U:
        T = min(depth, U - done)
        last = done + T          # level reached by this pass
        lo = tuple(lo_u[d] - e_lo[d] * (U - last) for d in range(3))
        hi = tuple(hi_u[d] + e_hi[d] * (U - last) for d in range(3))
        passes.append((T, lo, hi, tuple(e_lo), tuple(e_hi)))
        done = last
    return passes


def run_pass(grid: TwoGrid, T: int, lo, hi, e_lo=(0, 0, 0), e_hi=(0, 0, 0),
             out_lo=None, out_hi=None, src=None, dst=None, stream=None, peer=None) -> None:
    """One K2 launch: T levels from ``src`` (default current) into ``dst``.

    ``peer = (lo_buf, lo_shift, hi_buf, hi_shift, halo)``: also store output
    planes z < halo into ``lo_buf`` at plane z + lo_shift and planes
    z >= nz - halo into ``hi_buf`` at z + hi_shift (device buffers of the
    z-neighbours' destination grids, same layout; None skips a side).
    """
    src = grid.current_buffer() if src is None else src
    dst = grid.other_buffer() if dst is None else dst
    s = grid.stream() if stream is None else ctypes.c_void_p(stream)
    with _on(grid.device):
        if peer is not None:
            b_lo, s_lo, b_hi, s_hi, halo = peer
            o_lo = lo if out_lo is None else out_lo
            o_hi = hi if out_hi is None else out_hi
            N.check(N.lib().sp_sweep_tb_part_peer(
                ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), grid.sp_dtype,
                ctypes.byref(grid.layout), int(T), N.i64x3(lo), N.i64x3(hi), N.i32x3(e_lo),
                N.i32x3(e_hi), N.i64x3(o_lo), N.i64x3(o_hi),
                ctypes.c_void_p(b_lo.data_ptr() if b_lo is not None else None), int(s_lo),
                ctypes.c_void_p(b_hi.data_ptr() if b_hi is not None else None), int(s_hi),
                int(halo), s))
        elif out_lo is None:
            N.check(N.lib().sp_sweep_tb(
                ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), grid.sp_dtype,
                ctypes.byref(grid.layout), int(T), N.i64x3(lo), N.i64x3(hi), N.i32x3(e_lo),
                N.i32x3(e_hi), s))
        else:
            N.check(N.lib().sp_sweep_tb_part(
                ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), grid.sp_dtype,
                ctypes.byref(grid.layout), int(T), N.i64x3(lo), N.i64x3(hi), N.i32x3(e_lo),
                N.i32x3(e_hi), N.i64x3(out_lo), N.i64x3(out_hi), s))


def sweeps(grid: TwoGrid, levels: int, depth: int | None = None) -> None:
    """``levels`` full-interior levels as passes of ``depth`` (one call, no host sync)."""
    if getattr(grid, "storage", None) == "compressed":
        depth = depth or DEFAULT_DEPTH_INPLACE[grid.sp_dtype]
    depth = depth or DEFAULT_DEPTH[grid.sp_dtype]
    if not 1 <= depth <= MAX_DEPTH:
        raise ScheduleError(f"device pass depth must be in 1..{MAX_DEPTH}")
    if getattr(grid, "storage", None) == "compressed":
        grid.run_passes(int(levels), int(depth))
        return
    a, b = grid.buffers
    act = ctypes.c_int(grid.active)
    with _on(grid.device):
        N.check(N.lib().sp_run_sweeps(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                                      grid.sp_dtype, ctypes.byref(grid.layout), int(levels),
                                      int(depth), ctypes.byref(act), grid.stream()))
    grid.active = act.value


def run_node_sweeps(grid: TwoGrid, cfg: PipelineConfig, sweeps_: int,
                    level_domains=None) -> None:
    """``sweeps_`` node sweeps of U levels each (R/pipeline.py:459-462).

    Mirrors the reference's schedule checks (U > min extent is a
    ScheduleError, R/pipeline.py:226-229; U level domains required) and then
    runs every sweep as ceil(U / depth) K2 passes.  The grid ends
    sweeps_*U levels ahead; ``current`` holds it.
    """
    compressed = getattr(grid, "storage", None) == "compressed"
    if cfg.storage != grid.storage:   # R/pipeline.py:301-316 checks the same pairing
        raise ValueError(f"config expects {cfg.storage} storage but the device grid is {grid.storage}")
    if not compressed and not isinstance(grid, TwoGrid):
        raise ValueError("config expects two-grid storage")
    U = cfg.levels_per_sweep
    check_schedule(grid.dims, cfg, level_domains)
    depth = cfg.depth or (DEFAULT_DEPTH_INPLACE if compressed else DEFAULT_DEPTH)[grid.sp_dtype]
    if compressed and level_domains is not None:
        raise ScheduleError("compressed storage supports interior domains only")   # R/pipeline.py:312-313
    if compressed and grid.reference_slack:
        # the reference's contract: slack >= U, origin -U / +U per node sweep (R/pipeline.py:308-311,349-387)
        if grid.slack < U:
            raise ScheduleError(f"compressed slack {grid.slack} < U={U}")
        for k in range(sweeps_):
            grid.node_sweep(U, depth, -1 if k % 2 == 0 else 1)
        grid._scatter_shell()
        return
    if level_domains is None:
        for _ in range(sweeps_):
            sweeps(grid, U, depth)
        return
    passes = domains_to_passes(level_domains, U, depth)
    for _ in range(sweeps_):
        for T, lo, hi, e_lo, e_hi in passes:
            run_pass(grid, T, lo, hi, e_lo, e_hi)
            grid.swap()


def instrumented_run(*args, **kwargs):
    raise NotImplementedError("thread-trace auditing belongs to the CPU engine (out of scope)")
