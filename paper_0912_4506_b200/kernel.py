"""Jacobi sweeps on device grids (drop-in for R/kernel.py).

Every variant funnels into the C ABI: ``update_block``/``sweep_naive``/
``sweep_spatial_blocked`` call K1 (``sp_update_region``), i.e. one level over
a box; multi-level work goes through K2 (``sp_sweep_tb``) in pipeline.py.
The per-cell arithmetic is the reference's fixed order
((x- + x+) + (y- + y+)) + (z- + z+), then * ONE_SIXTH (R/kernel.py:15-34).
(R = /root/reference/pkg/src/stencilpipe)
"""

from __future__ import annotations

import ctypes

from . import _native as N
from .grid import CompressedGrid, GridError, TwoGrid, _on

ONE_SIXTH = 1.0 / 6.0


def stencil_point(xm, xp, ym, yp, zm, zp) -> float:
    """Mean of the six face neighbours in the fixed order (R/kernel.py:18-20)."""
    return ((xm + xp) + (ym + yp) + (zm + zp)) * ONE_SIXTH


def _require_device_grid(grid) -> TwoGrid:
    if not isinstance(grid, TwoGrid):
        raise TypeError(f"expected a paper_0912_4506_b200 TwoGrid, got {type(grid).__name__}")
    return grid


def _update(grid: TwoGrid, src, dst, lo, hi) -> None:
    with _on(grid.device):
        N.check(N.lib().sp_update_region(
            ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), grid.sp_dtype,
            ctypes.byref(grid.layout), N.i64x3(lo), N.i64x3(hi), grid.stream()))


def sweep_naive(grid: TwoGrid) -> None:
    """One full sweep: other <- stencil(current), then swap (R/kernel.py:43-47)."""
    _require_device_grid(grid)
    _update(grid, grid.current_buffer(), grid.other_buffer(), (0, 0, 0), grid.dims.shape)
    grid.swap()


def block_edges(extent: int, block: int) -> list[int]:
    """1D block boundaries 0, block, 2*block, ..., extent (R/kernel.py:50-56)."""
    if not 1 <= block:
        raise GridError(f"block extent must be >= 1, got {block}")
    edges = list(range(0, extent, block))
    edges.append(extent)
    return edges


def sweep_spatial_blocked(grid: TwoGrid, bs: tuple[int, int, int]) -> None:
    """Spatially blocked sweep (R/kernel.py:59-80).

    The block size is validated exactly as the reference does.  The
    reference's outer z loop over blocks becomes one single-level launch per
    z-block (blocks in z order, like the reference's traversal); its inner
    y/x blocks are the device kernel's own x-y tiles, which every launch
    marches through z.  Every launch reads ``current`` and writes ``other``,
    so the result is bitwise equal to ``sweep_naive`` (the per-cell
    arithmetic is unchanged; reference test_kernel.py:63-92).
    """
    _require_device_grid(grid)
    d = grid.dims
    bx, by, bz = bs
    for b, n in zip((bx, by, bz), (d.nx, d.ny, d.nz)):
        if not 1 <= b <= n:
            raise GridError(f"block size {bs} outside interior extents")
    ez = block_edges(d.nz, bz)
    src, dst = grid.current_buffer(), grid.other_buffer()
    for z0, z1 in zip(ez[:-1], ez[1:]):
        _update(grid, src, dst, (z0, 0, 0), (z1, d.ny, d.nx))
    grid.swap()


def update_block(grid: TwoGrid, lo, hi, level: int = 1, direction: int = -1) -> None:
    """One region at one level (R/kernel.py:124-147).

    Two-grid: level parity picks src/dst, no swap.  Compressed: reads at the
    offset ``level`` implies relative to the current origin, refreshes the
    ghost faces the region touches and writes one plane off in ``direction``
    (CompressedGrid.update_block); origin bookkeeping is the caller's."""
    for l, h in zip(lo, hi):
        if l > h:
            raise GridError(f"malformed region {lo}..{hi}")
    if isinstance(grid, CompressedGrid):
        grid.update_block(lo, hi, level=level, direction=direction)
        return
    _require_device_grid(grid)
    d = grid.dims
    for l, h, n in zip(lo, hi, d.shape):
        if l < -d.ghost + 1 or h > n + d.ghost - 1:
            raise GridError("region escapes allocation")
    for ax, (l, h, n) in enumerate(zip(lo, hi, d.shape)):
        g = grid.gz if ax == 0 else grid.gxy
        if l < -g + 1 or h > n + g - 1:
            raise GridError("region escapes the device allocation")
    bufs = (grid.current_buffer(), grid.other_buffer())
    _update(grid, bufs[(level - 1) % 2], bufs[level % 2], lo, hi)
