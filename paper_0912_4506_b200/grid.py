"""Device-resident 3D fields with ghost shells (drop-in for R/grid.py).

The reference keeps a ``TwoGrid`` as two dense numpy arrays in (z, y, x)
order (R/grid.py:121-161).  Here the pair lives in HBM, allocated by PyTorch
with a padded row pitch so every interior row starts on a 128-byte boundary
and TMA can stream x-y tiles (include/stencilpipe_b200.h, sp_layout_make).
``current``/``other`` are strided torch views with the reference's
alloc_shape; ``interior()``/``full_view()`` return host numpy copies, which is
what ``compare`` (R/verify.py:50-53) consumes.
(R = /root/reference/pkg/src/stencilpipe)
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N


class GridError(ValueError):
    """Invalid grid geometry or storage request (R/grid.py:25)."""


@dataclass(frozen=True)
class GridDims:
    """Interior extents and ghost width (R/grid.py:29-51)."""
    nx: int
    ny: int
    nz: int
    ghost: int = 1

    def __post_init__(self):
        if min(self.nx, self.ny, self.nz) < 1:
            raise GridError(f"interior extents must be >= 1, got "
                            f"{(self.nx, self.ny, self.nz)}")
        if self.ghost < 1:
            raise GridError(f"ghost width must be >= 1, got {self.ghost}")

    @property
    def shape(self) -> tuple[int, int, int]:
        return (self.nz, self.ny, self.nx)

    @property
    def alloc_shape(self) -> tuple[int, int, int]:
        g = self.ghost
        return tuple(n + 2 * g for n in self.shape)


_KINDS = {"constant": 0, "linear": 1, "hotplate": 2, "random": 3, "random_pm1": 4}


@dataclass(frozen=True)
class FillPattern:
    """Initial-value field over global coordinates (R/grid.py:66-118).

    Evaluated on the device by K3 (``sp_fill``), bit-identical to the
    reference's numpy evaluation.  Two extensions for the BASELINE configs:
    kind ``random_pm1`` (2u-1, config 4) and Dirichlet ``faces`` =
    (z-, z+, y-, y+, x-, x+) over a ``global_shape`` (z, y, x): a cell outside
    the global interior takes the first face it lies beyond, in that order.
    ``origin`` shifts local to global coordinates (R/decomp.py:107-117).
    """

    kind: str
    value: float = 0.0
    seed: int = 0
    faces: tuple | None = None
    global_shape: tuple | None = None
    origin: tuple = (0, 0, 0)

    def __post_init__(self):
        if self.kind not in _KINDS:
            raise GridError(f"unknown fill pattern {self.kind!r}")
        if self.faces is not None and (len(self.faces) != 6 or self.global_shape is None):
            raise GridError("faces need 6 values and a global_shape")

    @classmethod
    def constant(cls, v: float) -> "FillPattern":
        return cls("constant", value=float(v))

    @classmethod
    def linear(cls) -> "FillPattern":
        return cls("linear")

    @classmethod
    def hotplate(cls) -> "FillPattern":
        return cls("hotplate")

    @classmethod
    def random(cls, seed: int) -> "FillPattern":
        return cls("random", seed=int(seed))

    @classmethod
    def dirichlet_box(cls, kind: str, global_shape, faces, seed: int = 0,
                      value: float = 0.0) -> "FillPattern":
        """BASELINE-style box: ``kind`` interior, constant faces (z-,z+,y-,y+,x-,x+)."""
        return cls(kind, value=float(value), seed=int(seed),
                   faces=tuple(float(f) for f in faces),
                   global_shape=tuple(int(n) for n in global_shape))

    def shifted(self, origin) -> "FillPattern":
        o = tuple(int(a) + int(b) for a, b in zip(self.origin, origin))
        return FillPattern(self.kind, self.value, self.seed, self.faces, self.global_shape, o)

    def to_c(self) -> N.Pattern:
        p = N.Pattern()
        p.kind = _KINDS[self.kind]
        p.value = self.value
        p.seed = self.seed & 0xFFFFFFFFFFFFFFFF
        for i in range(3):
            p.gorigin[i] = self.origin[i]
        if self.faces is not None:
            p.has_faces = 1
            for i in range(3):
                p.gn[i] = self.global_shape[i]
            for i in range(6):
                p.faces[i] = self.faces[i]
        return p

    def evaluate(self, lo, hi) -> np.ndarray:
        """Host values over [lo, hi) (z, y, x), computed by the device kernel."""
        shape = tuple(int(h - l) for l, h in zip(lo, hi))
        if min(shape) <= 0:
            return np.zeros(shape)
        g = TwoGrid(GridDims(shape[2], shape[1], shape[0], 1), self.shifted(lo), _init_b=False)
        return g.interior()


def _torch_dtype(dtype):
    import torch
    if dtype in (None, np.float64, "float64", "f64", "fp64") or dtype is torch.float64:
        return torch.float64, N.SP_F64
    if dtype in (np.float32, "float32", "f32", "fp32") or dtype is torch.float32:
        return torch.float32, N.SP_F32
    if isinstance(dtype, np.dtype):
        return _torch_dtype(dtype.type)
    raise GridError(f"unsupported dtype {dtype!r} (float64 or float32)")


class TwoGrid:
    """Ping-pong pair in HBM; ``active`` selects the current level (R/grid.py:121-161).

    ``ghost_xy``/``ghost_z`` override the physical ghost depth per axis group
    (z-slab ranks keep depth-h halos in z only; x/y ghosts beyond depth 1 are
    never read by a 6-neighbour stencil).
    """

    storage = "twogrid"

    def __init__(self, dims: GridDims, pattern, dtype=np.float64, device=None,
                 ghost_xy: int | None = None, ghost_z: int | None = None,
                 _init_b: bool = True):
        import torch
        L = N.lib()
        self.dims = dims
        self.pattern = pattern
        self.torch_dtype, self.sp_dtype = _torch_dtype(dtype)
        self.dtype = np.float64 if self.sp_dtype == N.SP_F64 else np.float32
        dev = torch.device("cuda") if device is None else torch.device(device)
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        gxy = dims.ghost if ghost_xy is None else int(ghost_xy)
        gz = dims.ghost if ghost_z is None else int(ghost_z)
        lay = N.Layout()
        n_alloc = ctypes.c_int64()
        N.check(L.sp_layout_make(dims.nx, dims.ny, dims.nz, gxy, gxy, gz, self.sp_dtype,
                                 ctypes.byref(lay), ctypes.byref(n_alloc)))
        self.layout = lay
        self.gxy, self.gz = gxy, gz
        with torch.cuda.device(self.device):
            self._a = torch.zeros(n_alloc.value, dtype=self.torch_dtype, device=self.device)
            self._b = torch.empty_like(self._a)
        self._fill(pattern)
        if _init_b:
            self._b.copy_(self._a)
        self.active = 0

    # -- storage -------------------------------------------------------------

    def reset(self, pattern=None) -> None:
        """Re-initialise both arrays from ``pattern`` (default: the construction
        pattern) and make A current, as constructing the grid again would."""
        self._fill(self.pattern if pattern is None else pattern)
        self._b.copy_(self._a)
        self.active = 0

    def stream(self):
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _view(self, buf):
        lay = self.layout
        size = (lay.nz + 2 * self.gz, lay.ny + 2 * self.gxy, lay.nx + 2 * self.gxy)
        off = lay.origin - self.gz * lay.pz - self.gxy * lay.py - self.gxy
        return buf.as_strided(size, (lay.pz, lay.py, 1), off)

    def _fill(self, pattern):
        if isinstance(pattern, FillPattern):
            with _on(self.device):
                N.check(N.lib().sp_fill(ctypes.c_void_p(self._a.data_ptr()), self.sp_dtype,
                                        ctypes.byref(self.layout), ctypes.byref(pattern.to_c()),
                                        self.stream()))
            return
        if not hasattr(pattern, "evaluate"):
            raise GridError(f"pattern {pattern!r} has no evaluate(lo, hi)")
        # duck-typed pattern (R/grid.py:126-133): evaluate on the host, upload once
        import torch
        lo = (-self.gz, -self.gxy, -self.gxy)
        hi = (self.dims.nz + self.gz, self.dims.ny + self.gxy, self.dims.nx + self.gxy)
        vals = np.asarray(pattern.evaluate(lo, hi), dtype=self.dtype)
        self._view(self._a).copy_(torch.from_numpy(np.ascontiguousarray(vals)))

    @property
    def buffers(self):
        """(a, b) flat device buffers -- the raw allocations the C ABI receives."""
        return self._a, self._b

    @property
    def current(self):
        return self._view(self._a if self.active == 0 else self._b)

    @property
    def other(self):
        return self._view(self._b if self.active == 0 else self._a)

    def current_buffer(self):
        return self._a if self.active == 0 else self._b

    def other_buffer(self):
        return self._b if self.active == 0 else self._a

    def arrays(self):
        return (self.current, self.other)

    def swap(self) -> None:
        self.active ^= 1

    # -- host views ----------------------------------------------------------

    def interior_device(self):
        gz, g = self.gz, self.gxy
        d = self.dims
        return self.current[gz:gz + d.nz, g:g + d.ny, g:g + d.nx]

    def interior(self) -> np.ndarray:
        return self.interior_device().cpu().numpy()

    # -- host transfers (one pitched DMA each, stream-ordered) --------------------

    def host_shape(self):
        """Shape of the dense ghosted host field upload() takes (R/grid.py:126-134)."""
        d = self.dims
        return (d.nz + 2 * self.gz, d.ny + 2 * self.gxy, d.nx + 2 * self.gxy)

    def upload(self, field, stream=None) -> None:
        """Replace both arrays with a host field of shape host_shape() (torch CPU
        tensor -- pinned for an asynchronous copy -- or numpy), as constructing
        a reference TwoGrid from that field would; active becomes 0."""
        import torch
        t = field if isinstance(field, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(field))
        if tuple(t.shape) != self.host_shape() or t.dtype != self.torch_dtype or not t.is_contiguous():
            raise GridError(f"upload needs a contiguous {self.torch_dtype} field of shape "
                            f"{self.host_shape()}, got {t.dtype} {tuple(t.shape)}")
        s = self.stream() if stream is None else ctypes.c_void_p(stream)
        self.active = 0
        stg, n_stg = self._staging()
        with _on(self.device):
            N.check(N.lib().sp_copy_in(ctypes.c_void_p(t.data_ptr()), self.sp_dtype,
                                       ctypes.byref(self.layout), ctypes.c_void_p(self._a.data_ptr()),
                                       ctypes.c_void_p(self._b.data_ptr()), stg, n_stg, s))

    STAGING_PLANES = 64

    def _staging(self):
        """Device staging buffer for host transfers: STAGING_PLANES ghosted planes
        (linear PCIe copies, repacked on the device), allocated on first use."""
        import torch
        if getattr(self, "_stg", None) is None:
            hz, hy, hx = self.host_shape()
            n = min(hz, self.STAGING_PLANES) * hy * hx
            with torch.cuda.device(self.device):
                self._stg = torch.empty(n, dtype=self.torch_dtype, device=self.device)
        return ctypes.c_void_p(self._stg.data_ptr()), self._stg.numel()

    def download(self, out=None, stream=None):
        """The current interior into host memory (a torch CPU tensor; pass a
        pinned ``out`` of dims.shape for an asynchronous copy)."""
        import torch
        d = self.dims
        fresh = out is None
        if fresh:
            out = torch.empty(d.shape, dtype=self.torch_dtype, pin_memory=True)
        if tuple(out.shape) != tuple(d.shape) or out.dtype != self.torch_dtype or not out.is_contiguous():
            raise GridError(f"download needs a contiguous {self.torch_dtype} tensor of shape {d.shape}")
        s = self.stream() if stream is None else ctypes.c_void_p(stream)
        with _on(self.device):
            stg, n_stg = self._staging()
            N.check(N.lib().sp_copy_out(ctypes.c_void_p(self.current_buffer().data_ptr()), self.sp_dtype,
                                        ctypes.byref(self.layout), ctypes.c_void_p(out.data_ptr()),
                                        stg, n_stg, s))
        if fresh:
            torch.cuda.synchronize(self.device)   # a tensor the caller did not provide: complete
        return out

    def full_view(self) -> np.ndarray:
        return self.current.cpu().numpy()

    def value_at(self, i: int, j: int, k: int) -> float:
        g = self.dims.ghost
        for idx, n in zip((i, j, k), (self.dims.nx, self.dims.ny, self.dims.nz)):
            if not -g <= idx < n + g:
                raise IndexError(f"index {(i, j, k)} outside interior+ghost range")
        return float(self.current[k + self.gz, j + self.gxy, i + self.gxy].item())

    def digest(self, index_base: int = 0) -> int:
        """64-bit digest of the current interior (definition: oracle/jacobi_oracle.c).

        ``index_base`` offsets the cell index, so the digests of the z-slabs of
        a decomposition (index_base = z0*ny*nx) add up (mod 2^64) to the
        digest of the gathered grid."""
        out = ctypes.c_uint64()
        with _on(self.device):
            N.check(N.lib().sp_digest(ctypes.c_void_p(self.current_buffer().data_ptr()),
                                      self.sp_dtype, ctypes.byref(self.layout), int(index_base),
                                      ctypes.byref(out), self.stream()))
        return int(out.value)


class CompressedGrid:
    """Single-array storage in HBM (R/grid.py:164-208): one grid plus slack planes.

    The reference shifts its box one cell diagonally per level and refreshes
    the ghost faces before each block update (R/kernel.py:83-121).  On the
    device the box moves by whole planes in z (``offset``, in planes); x/y
    stay put, so the logical content -- ``interior()``, ``value_at``,
    ``full_view`` at any offset -- is what the reference's diagonal shift
    gives.  Two ways to size the slack:

    * ``slack=None`` (device-native, the memory-saving form): every pass of
      depth T runs IN PLACE (``sp_sweep_tb_inplace``): z-chunks of ``chunk``
      planes go in order and store their level-T planes 2*chunk+T planes away
      from where they read them -- down when ascending, up when descending --
      so a chunk only overwrites planes that chunks two and three back have
      finished reading (device counters enforce it).  The ghost shell is
      packed once (``sp_ghost_shell``) and re-scattered after every pass.
      HBM: (nz + 2 + slack) planes instead of 2 (nz + 2), slack = 4*chunk + 16.
    * ``slack=S`` (the reference's contract, honoured as given): the box
      starts at offset S and moves like the reference's -- ``shift_origin``
      within [0, S], ``update_block(level, direction)`` reads at
      offset + direction*(level-1) and writes one cell off, node sweeps of U
      levels move it by -U / +U (R/pipeline.py:349-387), needing S >= U.  The
      layout is the reference's too: S extra cells on every axis and the box
      shifted DIAGONALLY, which is what keeps a forward blocked traversal from
      overwriting cells later blocks still read.  Those moves are smaller
      than an in-place pass needs, so each level (or pass) is computed into a
      scratch box and copied to the shifted position, as the reference
      materialises each right-hand side.
    """

    storage = "compressed"

    def __init__(self, dims: GridDims, pattern, slack: int | None = None, dtype=np.float64,
                 device=None, chunk: int = 64):
        import torch
        if dims.ghost != 1:
            raise GridError("compressed storage uses a one-layer ghost shell")
        L = N.lib()
        self.dims = dims
        self.pattern = pattern
        self.torch_dtype, self.sp_dtype = _torch_dtype(dtype)
        self.dtype = np.float64 if self.sp_dtype == N.SP_F64 else np.float32
        dev = torch.device("cuda") if device is None else torch.device(device)
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.chunk = max(16, min(int(chunk), dims.nz))     # >= 2T for every T <= 8
        smax = 2 * self.chunk + 8
        if slack is None:
            self.reference_slack = False
            self.slack = 2 * smax
            offset0 = smax
        else:
            if slack < 0:
                raise GridError(f"slack must be >= 0, got {slack}")
            if max(n + 2 + int(slack) for n in dims.shape) ** 3 > np.iinfo(np.int64).max // 8:
                raise GridError("compressed allocation overflows address arithmetic")   # R/grid.py:180-181
            self.reference_slack = True
            self.slack = int(slack)
            offset0 = self.slack                        # R/grid.py:185
        lay = N.Layout()
        n_alloc = ctypes.c_int64()
        sxy = self.slack if self.reference_slack else 0  # reference: slack on every axis
        N.check(L.sp_layout_make(dims.nx + sxy, dims.ny + sxy, dims.nz + self.slack, 1, 1, 1, self.sp_dtype,
                                 ctypes.byref(lay), ctypes.byref(n_alloc)))
        self.blayout = lay                               # the whole allocation
        self.layout = N.Layout(*lay.as_tuple())          # the box at offset 0 (native: relative to _box_ptr)
        self.layout.nx, self.layout.ny, self.layout.nz = dims.nx, dims.ny, dims.nz
        self.offset = offset0                            # box plane z sits at allocation plane z + offset
        self._ascend_next = True
        self._scratch_buf = None
        with torch.cuda.device(self.device):
            self._buf = torch.zeros(n_alloc.value, dtype=self.torch_dtype, device=self.device)
            nshell = L.sp_ghost_shell_elems(dims.nx, dims.ny, dims.nz)
            self._shell = torch.empty(nshell, dtype=self.torch_dtype, device=self.device)
            nch = -(-dims.nz // self.chunk)
            self._counters = torch.zeros(nch, dtype=torch.int32, device=self.device)
        self._offset0 = offset0
        self._fill(pattern)
        self._gather_shell()

    def reset(self, pattern=None) -> None:
        """Re-initialise the box from ``pattern`` (default: the construction pattern) at
        its starting offset, as constructing the grid again would."""
        self.offset = self._offset0
        self._ascend_next = True
        self._fill(self.pattern if pattern is None else pattern)
        self._gather_shell()

    # -- storage -------------------------------------------------------------

    def stream(self):
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _at(self, offset: int | None = None):
        """(base pointer, layout) of the box at ``offset`` (default: current).
        Native: the box slides in z (pointer moves, layout fixed); reference
        slack: it slides diagonally (layout origin moves by o*(pz + py + 1))."""
        o = self.offset if offset is None else offset
        es = self._buf.element_size()
        if self.reference_slack:
            # z and y by the pointer (whole rows keep it 16-byte aligned for TMA), x by the origin
            lay = N.Layout(*self.layout.as_tuple())
            lay.origin += o
            return ctypes.c_void_p(self._buf.data_ptr() + o * (lay.pz + lay.py) * es), lay
        return ctypes.c_void_p(self._buf.data_ptr() + o * self.blayout.pz * es), self.layout

    def _box_ptr(self, offset: int | None = None):
        return self._at(offset)[0]

    def _box_start(self, offset: int | None = None) -> int:
        """Element index of the box's ghost corner (z=-1, y=-1, x=-1) in the allocation."""
        o = self.offset if offset is None else offset
        lay = self.layout
        diag = o * (lay.pz + lay.py + 1) if self.reference_slack else o * lay.pz   # as _at() places it
        return lay.origin + diag - lay.pz - lay.py - 1

    def _box_view(self):
        lay, d = self.layout, self.dims
        return self._buf.as_strided((d.nz + 2, d.ny + 2, d.nx + 2), (lay.pz, lay.py, 1), self._box_start())

    def _fill(self, pattern):
        if isinstance(pattern, FillPattern):
            ptr, lay = self._at()
            with _on(self.device):
                N.check(N.lib().sp_fill(ptr, self.sp_dtype, ctypes.byref(lay),
                                        ctypes.byref(pattern.to_c()), self.stream()))
            return
        if not hasattr(pattern, "evaluate"):
            raise GridError(f"pattern {pattern!r} has no evaluate(lo, hi)")
        import torch
        d = self.dims
        vals = np.asarray(pattern.evaluate((-1, -1, -1), (d.nz + 1, d.ny + 1, d.nx + 1)), dtype=self.dtype)
        self._box_view().copy_(torch.from_numpy(np.ascontiguousarray(vals)))

    def _gather_shell(self):
        """Pack the box's ghost shell (the Dirichlet values, fixed for the run)."""
        ptr, lay = self._at()
        with _on(self.device):
            N.check(N.lib().sp_ghost_shell(ptr, self.sp_dtype, ctypes.byref(lay),
                                           ctypes.c_void_p(self._shell.data_ptr()), 0, self.stream()))
        self._ghosts_at = self.offset

    def _scatter_shell(self, offset: int | None = None):
        o = self.offset if offset is None else offset
        ptr, lay = self._at(o)
        with _on(self.device):
            N.check(N.lib().sp_ghost_shell(ptr, self.sp_dtype, ctypes.byref(lay),
                                           ctypes.c_void_p(self._shell.data_ptr()), 1, self.stream()))
        self._ghosts_at = o

    @property
    def buffers(self):
        return (self._buf,)

    @property
    def current(self):
        """The ghosted box (device view) at the current offset."""
        return self._box_view()

    def shift_origin(self, delta: int) -> None:
        """Move the box origin by ``delta`` planes without moving data (R/grid.py:191-195)."""
        new = self.offset + int(delta)
        if not 0 <= new <= self.slack:
            raise GridError(f"origin offset {new} escapes slack [0, {self.slack}]")
        self.offset = new

    # -- passes --------------------------------------------------------------

    def _scratch(self):
        """A box-sized buffer in the box layout (out-of-place levels; allocated on first use)."""
        import torch
        if self._scratch_buf is None:
            n = (self.dims.nz + 2) * self.blayout.pz
            with torch.cuda.device(self.device):
                self._scratch_buf = torch.empty(n, dtype=self.torch_dtype, device=self.device)
        return self._scratch_buf

    def _pass_shifted(self, T: int, o_read: int, o_write: int, lo, hi) -> None:
        """T levels over the interior box [lo, hi) read at ``o_read`` (walls on the
        box faces: its ghost cells hold the level's boundary) into the scratch box,
        then those cells into the box at ``o_write`` -- the reference's
        materialised right-hand side (R/kernel.py:105-121)."""
        if any(h <= l for l, h in zip(lo, hi)):
            return
        scr = self._scratch()
        ptr, lay = self._at(o_read)
        # the scratch holds the box with its ghost corner at element 0, same pitches
        es = self._buf.element_size()
        scr_base = ctypes.c_void_p(scr.data_ptr() - (lay.origin - lay.pz - lay.py - 1) * es)
        with _on(self.device):
            N.check(N.lib().sp_sweep_tb(ptr, scr_base, self.sp_dtype, ctypes.byref(lay), int(T),
                                        N.i64x3(lo), N.i64x3(hi), None, None, self.stream()))
        shape = tuple(h - l for l, h in zip(lo, hi))
        strides = (lay.pz, lay.py, 1)
        rel = (lo[0] + 1) * lay.pz + (lo[1] + 1) * lay.py + (lo[2] + 1)   # from the ghost corner
        src = scr.as_strided(shape, strides, rel)
        dst = self._buf.as_strided(shape, strides, self._box_start(o_write) + rel)
        dst.copy_(src)

    def update_block(self, lo, hi, level: int = 1, direction: int = -1) -> None:
        """One level over the interior box [lo, hi) (R/kernel.py:141-147): read at
        offset + direction*(level-1), refresh the ghost faces the box touches
        there (R/kernel.py:83-102), write one plane off in ``direction``.
        Origin bookkeeping is the caller's (``shift_origin``), as in the reference."""
        if direction not in (-1, 1):
            raise GridError(f"direction must be -1 or +1, got {direction}")
        lo, hi = tuple(int(v) for v in lo), tuple(int(v) for v in hi)
        for l, h, n in zip(lo, hi, self.dims.shape):
            if l > h:
                raise GridError(f"malformed region {lo}..{hi}")
            if l < 0 or h > n:
                raise GridError(f"compressed update region {lo}..{hi} must lie inside the interior")
        o_read = self.offset + direction * (level - 1)
        o_write = o_read + direction
        if not (0 <= o_read <= self.slack and 0 <= o_write <= self.slack):
            raise GridError(f"level {level} in direction {direction} escapes slack [0, {self.slack}] "
                            f"(read at {o_read}, write at {o_write})")
        ptr, lay = self._at(o_read)
        with _on(self.device):
            N.check(N.lib().sp_ghost_shell_region(ptr, self.sp_dtype, ctypes.byref(lay),
                                                  ctypes.c_void_p(self._shell.data_ptr()), N.i64x3(lo),
                                                  N.i64x3(hi), self.stream()))
        self._pass_shifted(1, o_read, o_write, lo, hi)

    def node_sweep(self, U: int, depth: int, direction: int) -> None:
        """U levels moving the origin by direction*U (R/pipeline.py:381-387), as
        passes of ``depth`` through the scratch box (slack given as in the reference)."""
        from .pipeline import ScheduleError
        end = self.offset + direction * U
        if not 0 <= end <= self.slack:
            raise ScheduleError(f"node sweep of U={U} in direction {direction} from offset {self.offset} "
                                f"escapes slack [0, {self.slack}]")
        d = self.dims
        done = 0
        while done < U:
            T = min(depth, U - done)
            self._scatter_shell()                          # the boundary at the read position
            o_write = self.offset + direction * T
            self._pass_shifted(T, self.offset, o_write, (0, 0, 0), d.shape)
            self.offset = o_write
            done += T

    def run_passes(self, levels: int, depth: int) -> None:
        """``levels`` levels as passes of ``depth`` (stream-ordered)."""
        if self.reference_slack:
            from .pipeline import ScheduleError
            if self.offset - levels >= 0:
                self.node_sweep(levels, depth, -1)
            elif self.offset + levels <= self.slack:
                self.node_sweep(levels, depth, 1)
            else:
                raise ScheduleError(f"{levels} levels do not fit the slack {self.slack} from offset "
                                    f"{self.offset}")
            self._scatter_shell()
            return
        d = self.dims
        if self._ghosts_at != self.offset:
            self._scatter_shell()
        done = 0
        while done < levels:
            T = min(depth, levels - done)
            s = 2 * min(self.chunk, d.nz) + T
            up_ok = self.offset - s >= 0
            down_ok = self.offset + s <= self.slack
            if not (up_ok or down_ok):
                from .pipeline import ScheduleError
                raise ScheduleError(f"in-place pass needs {s} planes of slack on one side of offset "
                                    f"{self.offset} (slack {self.slack})")
            ascend = up_ok if (self._ascend_next or not down_ok) else not down_ok
            lo = (self.offset, 0, 0)
            hi = (self.offset + d.nz, d.ny, d.nx)
            with _on(self.device):
                N.check(N.lib().sp_sweep_tb_inplace(
                    ctypes.c_void_p(self._buf.data_ptr()), self.sp_dtype, ctypes.byref(self.blayout), int(T),
                    N.i64x3(lo), N.i64x3(hi), int(self.chunk), 1 if ascend else -1,
                    ctypes.c_void_p(self._counters.data_ptr()), self._counters.numel(), self.stream()))
            self.offset += -s if ascend else s
            self._scatter_shell()
            self._ascend_next = not ascend
            done += T

    # -- host views ----------------------------------------------------------

    def interior_device(self):
        d = self.dims
        return self._box_view()[1:1 + d.nz, 1:1 + d.ny, 1:1 + d.nx]

    def interior(self) -> np.ndarray:
        return self.interior_device().cpu().numpy()

    def full_view(self) -> np.ndarray:
        return self._box_view().cpu().numpy()

    def value_at(self, i: int, j: int, k: int) -> float:
        for idx, n in zip((i, j, k), (self.dims.nx, self.dims.ny, self.dims.nz)):
            if not -1 <= idx < n + 1:
                raise IndexError(f"index {(i, j, k)} outside interior+ghost range")
        return float(self._box_view()[k + 1, j + 1, i + 1].item())

    def digest(self, index_base: int = 0) -> int:
        out = ctypes.c_uint64()
        ptr, lay = self._at()
        with _on(self.device):
            N.check(N.lib().sp_digest(ptr, self.sp_dtype, ctypes.byref(lay),
                                      int(index_base), ctypes.byref(out), self.stream()))
        return int(out.value)

    @property
    def hbm_bytes(self) -> int:
        return self._buf.numel() * self._buf.element_size()

    # -- host transfers (stream-ordered; same contract as TwoGrid) ---------------

    def host_shape(self):
        d = self.dims
        return (d.nz + 2, d.ny + 2, d.nx + 2)

    STAGING_PLANES = 64

    def _staging(self):
        """Bounded device staging buffer (STAGING_PLANES dense ghosted planes) for
        host transfers: linear PCIe copies repacked on the device by K6, so no
        box-sized temporary is ever made (the box view is strided)."""
        import torch
        if getattr(self, "_stg", None) is None:
            hz, hy, hx = self.host_shape()
            n = min(hz, self.STAGING_PLANES) * hy * hx
            with torch.cuda.device(self.device):
                self._stg = torch.empty(n, dtype=self.torch_dtype, device=self.device)
        return ctypes.c_void_p(self._stg.data_ptr()), self._stg.numel()

    def upload(self, field, stream=None) -> None:
        """Replace the box (ghosts included) with a host field of shape host_shape();
        the packed ghost shell is re-gathered from it."""
        import torch
        t = field if isinstance(field, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(field))
        if tuple(t.shape) != self.host_shape() or t.dtype != self.torch_dtype or not t.is_contiguous():
            raise GridError(f"upload needs a contiguous {self.torch_dtype} field of shape {self.host_shape()}")
        s = self.stream() if stream is None else ctypes.c_void_p(stream)
        stg, n_stg = self._staging()
        ptr, lay = self._at()
        with _on(self.device):
            N.check(N.lib().sp_copy_in(ctypes.c_void_p(t.data_ptr()), self.sp_dtype, ctypes.byref(lay),
                                       ptr, None, stg, n_stg, s))
            N.check(N.lib().sp_ghost_shell(ptr, self.sp_dtype, ctypes.byref(lay),
                                           ctypes.c_void_p(self._shell.data_ptr()), 0, s))
        self._ghosts_at = self.offset

    def download(self, out=None, stream=None):
        """The interior into host memory (pass a pinned ``out`` for an asynchronous copy)."""
        import torch
        d = self.dims
        fresh = out is None
        if fresh:
            out = torch.empty(d.shape, dtype=self.torch_dtype, pin_memory=True)
        if tuple(out.shape) != tuple(d.shape) or out.dtype != self.torch_dtype or not out.is_contiguous():
            raise GridError(f"download needs a contiguous {self.torch_dtype} tensor of shape {d.shape}")
        s = self.stream() if stream is None else ctypes.c_void_p(stream)
        stg, n_stg = self._staging()
        ptr, lay = self._at()
        with _on(self.device):
            N.check(N.lib().sp_copy_out(ptr, self.sp_dtype, ctypes.byref(lay),
                                        ctypes.c_void_p(out.data_ptr()), stg, n_stg, s))
        if fresh:
            torch.cuda.synchronize(self.device)
        return out


class _on:
    """Make ``device`` current for the duration of a C-ABI call."""

    def __init__(self, device):
        self.device = device

    def __enter__(self):
        import torch
        self._ctx = torch.cuda.device(self.device)
        self._ctx.__enter__()

    def __exit__(self, *a):
        self._ctx.__exit__(*a)


class ArrayPattern:
    """Duck-typed pattern over a host field holding the ghosted box
    (z, y, x) of ``dims`` -- e.g. the array ``load_field`` returns -- so a
    dumped grid can be re-created on the device: ``TwoGrid(dims, ArrayPattern(...))``."""

    def __init__(self, field: np.ndarray, ghost: int):
        self.field = np.asarray(field)
        self.ghost = ghost

    def evaluate(self, lo, hi) -> np.ndarray:
        g = self.ghost
        sl = tuple(slice(l + g, h + g) for l, h in zip(lo, hi))
        return self.field[sl]


def dump_field(grid, fh) -> None:
    """Text dump compatible with the reference (R/grid.py:280-289): header
    ``nx ny nz ghost`` then the ghosted box, x fastest, one %.17g value per line."""
    d = grid.dims
    full = grid.full_view()
    if full.shape != d.alloc_shape:
        raise GridError("dump needs a grid with the same ghost depth on every axis")
    fh.write(f"{d.nx} {d.ny} {d.nz} {d.ghost}\n")
    fh.write("".join("%.17g\n" % v for v in full.astype(np.float64).ravel()))


def load_field(fh) -> tuple[GridDims, np.ndarray]:
    """Parse a dump (R/grid.py:293-300) into (dims, ghosted host field)."""
    header = fh.readline().split()
    nx, ny, nz, ghost = (int(t) for t in header)
    dims = GridDims(nx, ny, nz, ghost)
    flat = np.array([float(line) for line in fh], dtype=np.float64)
    if flat.size != int(np.prod(dims.alloc_shape)):
        raise GridError("dump payload does not match header extents")
    return dims, flat.reshape(dims.alloc_shape)


def allocate(dims: GridDims, mode: str, pattern, slack: int | None = None, **kw):
    """Allocate and initialise a device grid (R/grid.py:217-223).

    ``slack`` (compressed only) is honoured as given, as in the reference;
    omitted, the device picks the slack its in-place passes need."""
    if mode == "twogrid":
        return TwoGrid(dims, pattern, **kw)
    if mode == "compressed":
        return CompressedGrid(dims, pattern, slack=slack, **kw)
    raise GridError(f"unknown storage mode {mode!r}")
