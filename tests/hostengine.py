"""Test-only host engine for SlabRunner: grids in CPU memory, passes by the C oracle.

Lets the multi-process halo-exchange logic of paper_0912_4506_b200.dist run on
CPU with the gloo backend (world_size 2) -- the compute is the oracle's
update_region, so this file is test infrastructure, never product code.
The grid uses the device layout (sp_layout_make, callable without a GPU) so
the plane spans exchanged are byte-identical to the CUDA path's.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from oracle import oracle as O
from paper_0912_4506_b200 import _native as N


class HostGrid:
    def __init__(self, dims, pattern: "O.BoxPattern", dtype, gz, gxy=1):
        L = N.load_library()
        lay = N.Layout()
        n = ctypes.c_int64()
        self.sp_dtype = N.SP_F64 if dtype == np.float64 else N.SP_F32
        N.check(L.sp_layout_make(dims.nx, dims.ny, dims.nz, gxy, gxy, gz, self.sp_dtype,
                                 ctypes.byref(lay), ctypes.byref(n)))
        self.layout = lay
        self.dims = dims
        self.dtype = dtype
        td = torch.float64 if dtype == np.float64 else torch.float32
        # shared memory, so the p2p transport can map a neighbour's grids
        self._a = torch.zeros(n.value, dtype=td).share_memory_()
        self._b = torch.zeros(n.value, dtype=td).share_memory_()
        olay = O._Layout(*lay.as_tuple())
        self.olay = olay
        fill = O.lib().or_fill_f64 if dtype == np.float64 else O.lib().or_fill_f32
        fill(self._a.data_ptr(), ctypes.byref(olay), ctypes.byref(O._c_pattern(pattern)))
        self._b.copy_(self._a)
        self._init = self._a.clone()
        self.active = 0

    def reset(self):
        self._a.copy_(self._init)
        self._b.copy_(self._init)
        self.active = 0

    @property
    def buffers(self):
        return (self._a, self._b)

    @property
    def torch_dtype(self):
        return self._a.dtype

    @property
    def current(self):
        return self.current_buffer()

    @property
    def other(self):
        return self.other_buffer()

    def interior_device(self):
        return torch.from_numpy(self.interior())

    def current_buffer(self):
        return self._a if self.active == 0 else self._b

    def other_buffer(self):
        return self._b if self.active == 0 else self._a

    def swap(self):
        self.active ^= 1

    def interior(self):
        lay = self.layout
        buf = self.current_buffer().numpy()
        out = np.empty((lay.nz, lay.ny, lay.nx), dtype=self.dtype)
        for z in range(lay.nz):
            for y in range(lay.ny):
                o = lay.origin + z * lay.pz + y * lay.py
                out[z, y] = buf[o:o + lay.nx]
        return out


class HostEngine:
    """SlabRunner engine: K2 semantics emulated level by level with the oracle."""

    def __init__(self, base_pattern: "O.BoxPattern"):
        self.base = base_pattern

    def make_grid(self, decomp, rank, pattern, dtype, device):
        origin = tuple(r[0] for r in decomp.ranges(rank))
        gxy = 1 if tuple(decomp.layout[:2]) == (1, 1) else decomp.halo
        return HostGrid(decomp.local_dims(rank), self.base.shifted(origin), dtype, decomp.halo, gxy)

    def pack(self, g, axis, ext, rng):
        from paper_0912_4506_b200.decomp import _slab
        return _slab(g, axis, ext, rng).contiguous().clone()

    def unpack(self, g, axis, ext, rng, data):
        from paper_0912_4506_b200.decomp import _slab
        _slab(g, axis, ext, rng).copy_(data)

    def default_depth(self, grid):
        return 4

    def run_pass(self, g, T, lo, hi, e_lo, e_hi, out_lo, out_hi):
        upd = O.lib().or_update_region_f64 if g.dtype == np.float64 else O.lib().or_update_region_f32
        src = g.current_buffer()
        dst = g.other_buffer()
        a = src.clone()
        b = src.clone()
        for t in range(1, T + 1):
            dlo = [lo[d] - e_lo[d] * (T - t) for d in range(3)]
            dhi = [hi[d] + e_hi[d] * (T - t) for d in range(3)]
            s, d_ = (a, b) if t % 2 == 1 else (b, a)
            upd(s.data_ptr(), d_.data_ptr(), ctypes.byref(g.olay),
                (ctypes.c_int64 * 3)(*dlo), (ctypes.c_int64 * 3)(*dhi))
        res = b if T % 2 == 1 else a
        lay = g.layout
        for z in range(out_lo[0], out_hi[0]):
            for y in range(out_lo[1], out_hi[1]):
                o = lay.origin + z * lay.pz + y * lay.py
                dst[o + out_lo[2]:o + out_hi[2]] = res[o + out_lo[2]:o + out_hi[2]]

    def run_pass_peer(self, g, T, lo, hi, e_lo, e_hi, out_lo, out_hi, peer):
        """run_pass, then the kernel's peer stores: output planes z < halo into
        the z- neighbour's grid at z + lo_shift, z >= nz - halo into the z+ one."""
        self.run_pass(g, T, lo, hi, e_lo, e_hi, out_lo, out_hi)
        b_lo, s_lo, b_hi, s_hi, halo = peer
        dst = g.other_buffer()
        lay = g.layout
        for z in range(out_lo[0], out_hi[0]):
            for buf, shift, take in ((b_lo, s_lo, z < halo), (b_hi, s_hi, z >= lay.nz - halo)):
                if buf is None or not take:
                    continue
                for y in range(out_lo[1], out_hi[1]):
                    o = lay.origin + z * lay.pz + y * lay.py
                    r = o + shift * lay.pz
                    buf[r + out_lo[2]:r + out_hi[2]] = dst[o + out_lo[2]:o + out_hi[2]]

    def sync(self, g):
        pass

    def share(self, g):
        import io
        import pickle
        from multiprocessing.reduction import ForkingPickler
        import torch.multiprocessing  # noqa: F401  (registers the tensor reducers)
        blob = io.BytesIO()
        ForkingPickler(blob, pickle.HIGHEST_PROTOCOL).dump(list(g.buffers))
        return blob.getvalue()

    def open(self, g, shared):
        import pickle
        return pickle.loads(shared)

    def close(self, g, bufs):
        pass
