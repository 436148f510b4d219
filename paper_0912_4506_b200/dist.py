"""Multi-process domain-decomposed runner: one process per GPU, halos over torch.distributed.

Mirrors the reference's distributed engine (exchange_halos + outer_step,
R/decomp.py:149-237, R/transport.py as the message layer).  Any Cartesian
layout (px, py, pz) runs the reference's extended-slab exchange x -> y -> z
with device pack/unpack (K6, sp_copy_box) around NCCL send/recv, then the
passes on the extended level domains.  For z-slab layouts (1, 1, P) -- the
8-GPU configuration -- the exchange is moved onto NCCL point-to-point
(``batch_isend_irecv`` of h contiguous padded z-planes, straight from and
into the grid buffers) and OVERLAPPED with compute:

  step k:  wait for halo(S_k)                     (recv posted in step k-1)
           K2 on the two boundary slabs  z in [0,h), [nz-h,nz)  -> S_{k+1}
           post send/recv of S_{k+1}'s boundary planes            (NCCL stream)
           K2 on the interior slab z in [h, nz-h)   -> S_{k+1}   (compute stream)

The interior slab needs no ghost plane (its level-1 reads stay inside
[0, nz)), so it runs concurrently with the transfer.  The reference
alternates exchange and compute strictly; results are
bit-identical either way because the per-cell arithmetic is unchanged.

``transport="p2p"`` fuses the exchange into the boundary kernels: each rank
maps its z-neighbours' grids (CUDA IPC through torch's tensor sharing) and
the boundary K2 launches store their level-T planes a second time straight
into the neighbours' ghost planes over NVLink (sp_sweep_tb_part_peer).  Only
a one-element token per neighbour and step travels through the process group:

  step k:  wait for the neighbours' tokens of step k-1    (their planes have
           landed in my ghosts, and they finished reading the ghosts I write)
           boundary K2 -> my S_{k+1} planes + the neighbours' S_{k+1} ghosts
           send my step-k token                            (after the kernels)
           interior K2

``engine`` abstracts the grid + pass implementation so the exchange logic is
testable on CPU with gloo (tests supply a host engine); the default is the
CUDA engine and there is no fallback.
(R = /root/reference/pkg/src/stencilpipe)
"""

from __future__ import annotations

import numpy as np

from .decomp import (DecompositionError, _slab, build_halo_plan, decompose, face_flags, plane_spans,
                     slab_box)
from .grid import GridDims
from .pipeline import DEFAULT_DEPTH, MAX_DEPTH


class CudaEngine:
    """Device grids + K2 passes through the C ABI."""

    def make_grid(self, decomp, rank, pattern, dtype, device):
        from .decomp import local_grid
        return local_grid(decomp, rank, pattern, dtype=dtype, device=device)

    def default_depth(self, grid):
        """Tuned levels per pass for the grid's dtype (pipeline.DEFAULT_DEPTH)."""
        return DEFAULT_DEPTH[grid.sp_dtype]

    def run_pass(self, grid, T, lo, hi, e_lo, e_hi, out_lo, out_hi):
        from .pipeline import run_pass
        run_pass(grid, T, lo, hi, e_lo, e_hi, out_lo=out_lo, out_hi=out_hi)

    def run_pass_peer(self, grid, T, lo, hi, e_lo, e_hi, out_lo, out_hi, peer):
        from .pipeline import run_pass
        run_pass(grid, T, lo, hi, e_lo, e_hi, out_lo=out_lo, out_hi=out_hi, peer=peer)

    def sync(self, grid):
        import torch
        torch.cuda.current_stream(grid.device).synchronize()

    def pack(self, grid, axis, ext, rng):
        """The halo slab (R/decomp.py:137-179 geometry) of the current state as a
        dense device buffer (K6 box copy, sp_copy_box)."""
        import torch
        from . import _native as N
        lay = grid.layout
        start, shape = slab_box(lay, axis, ext, rng)
        buf = grid.current_buffer()
        out = torch.empty(shape, dtype=buf.dtype, device=buf.device)
        es = buf.element_size()
        N.check(N.lib().sp_copy_box(ctypes_ptr(buf.data_ptr() + start * es), ctypes_ptr(out.data_ptr()),
                                    grid.sp_dtype, *shape, lay.py, lay.pz, shape[2], shape[1] * shape[2],
                                    grid.stream()))
        return out

    def unpack(self, grid, axis, ext, rng, data):
        """A received dense slab into the current state's ghost layers (K6)."""
        from . import _native as N
        lay = grid.layout
        start, shape = slab_box(lay, axis, ext, rng)
        buf = grid.current_buffer()
        es = buf.element_size()
        N.check(N.lib().sp_copy_box(ctypes_ptr(data.data_ptr()), ctypes_ptr(buf.data_ptr() + start * es),
                                    grid.sp_dtype, *shape, shape[2], shape[1] * shape[2], lay.py, lay.pz,
                                    grid.stream()))

    def share(self, grid):
        """CUDA IPC handles of both grids (picklable)."""
        import ctypes
        from . import _native as N
        out = []
        for b in grid.buffers:
            h, off = (ctypes.c_ubyte * 64)(), ctypes.c_int64()
            N.check(N.lib().sp_ipc_export(ctypes.c_void_p(b.data_ptr()), ctypes.byref(h), ctypes.byref(off)))
            out.append((bytes(h), off.value))
        return out

    def open(self, grid, shared):
        """Map a neighbour's grids into this rank's device."""
        import ctypes
        import torch
        from . import _native as N
        bufs = []
        with torch.cuda.device(grid.device):
            for h, off in shared:
                ptr = ctypes.c_void_p()
                N.check(N.lib().sp_ipc_import(ctypes.byref((ctypes.c_ubyte * 64).from_buffer_copy(h)),
                                              off, ctypes.byref(ptr)))
                bufs.append(PeerBuffer(ptr.value, off))
        return bufs

    def close(self, grid, bufs):
        from . import _native as N
        for b in bufs:
            N.check(N.lib().sp_ipc_close(b.ptr, b.offset))


def ctypes_ptr(p: int):
    import ctypes
    return ctypes.c_void_p(p)


class PeerBuffer:
    """A neighbour's grid allocation mapped into this process (CUDA IPC)."""

    def __init__(self, ptr: int, offset: int):
        self.ptr = ptr
        self.offset = offset

    def data_ptr(self) -> int:
        return self.ptr


class SlabRunner:
    """This rank's z-slab of a (1, 1, P) decomposition with halo depth h."""

    def __init__(self, global_dims: GridDims, pattern, h: int, dtype=np.float64,
                 depth: int | None = None, device=None, engine=None, overlap: bool = True,
                 group=None, transport: str = "nccl", layout=None, order=("x", "y", "z")):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.h = h
        # (px, py, pz): z-slabs by default; any Cartesian layout runs the
        # reference's extended-slab exchange x -> y -> z (R/decomp.py:125-179)
        self.layout = tuple(layout) if layout is not None else (1, 1, self.world)
        self.multi_axis = tuple(self.layout[:2]) != (1, 1)
        self.order = tuple(order)
        self.decomp = decompose(global_dims, self.world, self.layout, h)
        self.engine = engine or CudaEngine()
        self.grid = self.engine.make_grid(self.decomp, self.rank, pattern, dtype, device)
        self.depth = depth or self.engine.default_depth(self.grid)
        self.e_lo, self.e_hi = face_flags(self.decomp, self.rank)
        self.lo_nb = self.decomp.neighbor(self.rank, 0, high=False)
        self.hi_nb = self.decomp.neighbor(self.rank, 0, high=True)
        nz = self.grid.dims.nz
        # overlap needs one pass per outer step and a non-empty interior slab (z-slabs)
        self.overlap = overlap and not self.multi_axis and h <= min(self.depth, MAX_DEPTH) and nz > 2 * h
        self._pending = []
        self._primed = False
        self.messages = 0
        self.bytes_sent = 0
        if transport not in ("nccl", "p2p"):
            raise DecompositionError(f"unknown halo transport {transport!r}")
        if transport == "p2p" and self.multi_axis:
            raise DecompositionError("the fused p2p transport serves z-slab layouts (1, 1, P) only")
        self.transport = transport
        if transport == "p2p":
            if not self.overlap:
                raise DecompositionError("p2p halos need one pass per step (h <= depth) and nz > 2h")
            self._map_peers()

    # -- p2p transport -------------------------------------------------------

    def _map_peers(self):
        """Map both grids of each z-neighbour into this process (the engine's
        IPC: CUDA IPC handles for device grids, shared memory for the host
        test engine)."""
        import torch
        dist = self.dist
        everyone = [None] * self.world
        dist.all_gather_object(everyone, self.engine.share(self.grid), group=self.group)
        self._peer = {}
        err = None
        try:
            for nb in (self.lo_nb, self.hi_nb):
                if nb is not None:
                    self._peer[nb] = self.engine.open(self.grid, everyone[nb])
        except Exception as exc:      # decided collectively below, so every rank agrees
            err = exc
        ok = torch.tensor([0 if err else 1], dtype=torch.int32,
                          device=None if dist.get_backend(self.group) != "nccl" else self.grid.buffers[0].device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        if not int(ok.item()):
            for bufs in self._peer.values():
                self.engine.close(self.grid, bufs)
            self._peer = {}
            raise DecompositionError(f"p2p mapping failed on some rank: {err or 'see that rank'}")
        self._nz = [self.decomp.local_dims(r).nz for r in range(self.world)]
        self._host_tokens = dist.get_backend(self.group) != "nccl"
        dev = None if self._host_tokens else self.grid.buffers[0].device
        self._tok_out = torch.zeros(1, dtype=torch.int32, device=dev)
        self._tok_in = {nb: torch.zeros(1, dtype=torch.int32, device=dev) for nb in self._peer}
        self.sync_start()

    def close(self):
        """Unmap the neighbours' grids (p2p transport)."""
        self.finish()
        if getattr(self, "_peer", None):
            self.engine.sync(self.grid)
            self.dist.barrier(group=self.group)      # nobody stores into a grid being unmapped
            for bufs in self._peer.values():
                self.engine.close(self.grid, bufs)
            self._peer = {}

    def sync_start(self):
        """All ranks' grids are written (fill / upload) before anyone's next step
        may store into them; a no-op ordering point for the NCCL transport."""
        self.finish()
        self.engine.sync(self.grid)
        self.dist.barrier(group=self.group)

    def _peer_args(self):
        """(lo_buf, lo_shift, hi_buf, hi_shift, h) for the destination grid of this step."""
        k = 1 - self.grid.active          # ranks swap in lockstep: same buffer index
        lo = self._peer[self.lo_nb][k] if self.lo_nb is not None else None
        hi = self._peer[self.hi_nb][k] if self.hi_nb is not None else None
        lo_shift = self._nz[self.lo_nb] if self.lo_nb is not None else 0
        return lo, lo_shift, hi, -self.grid.dims.nz, self.h

    def _signal(self):
        """Send this step's token to both neighbours, post receives of theirs."""
        dist = self.dist
        if self._host_tokens:
            self.engine.sync(self.grid)   # host-delivered token: the peer stores are done
        ops = []
        for nb in (self.lo_nb, self.hi_nb):
            if nb is None:
                continue
            ops.append(dist.P2POp(dist.isend, self._tok_out, self._global_rank(nb), self.group))
            ops.append(dist.P2POp(dist.irecv, self._tok_in[nb], self._global_rank(nb), self.group))
        if ops:
            self._pending.extend(dist.batch_isend_irecv(ops))
            self.messages += len(ops) // 2

    def _step_p2p(self, r):
        g, h = self.grid, self.h
        self._wait()
        lo, hi = self._domain(r, 0, r)
        nz = g.dims.nz
        low = ((0, lo[1], lo[2]), (h, hi[1], hi[2]))
        high = ((nz - h, lo[1], lo[2]), (nz, hi[1], hi[2]))
        inner = ((h, lo[1], lo[2]), (nz - h, hi[1], hi[2]))
        peer = self._peer_args()
        for olo, ohi in (low, high):
            self.engine.run_pass_peer(g, r, lo, hi, self.e_lo, self.e_hi, olo, ohi, peer)
        self._signal()
        self.engine.run_pass(g, r, lo, hi, self.e_lo, self.e_hi, *inner)
        g.swap()

    # -- halo exchange ---------------------------------------------------------

    def _global_rank(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def _post(self, buf):
        """Post sends of buf's boundary planes and receives into buf's ghost planes."""
        dist = self.dist
        send_lo, send_hi, recv_lo, recv_hi = plane_spans(buf, self.grid.layout, self.h)
        ops = []
        if self.lo_nb is not None:
            ops.append(dist.P2POp(dist.isend, send_lo, self._global_rank(self.lo_nb), self.group))
            ops.append(dist.P2POp(dist.irecv, recv_lo, self._global_rank(self.lo_nb), self.group))
        if self.hi_nb is not None:
            ops.append(dist.P2POp(dist.isend, send_hi, self._global_rank(self.hi_nb), self.group))
            ops.append(dist.P2POp(dist.irecv, recv_hi, self._global_rank(self.hi_nb), self.group))
        if ops:
            self._pending.extend(dist.batch_isend_irecv(ops))
            self.messages += len(ops) // 2
            self.bytes_sent += sum(o.tensor.numel() * o.tensor.element_size()
                                   for o in ops if o.op is dist.isend)

    def _wait(self):
        for w in self._pending:
            w.wait()
        self._pending = []

    def exchange(self):
        """Blocking exchange of the current state's halos (R/decomp.py:149-179)."""
        if self.multi_axis:
            self._exchange_phases()
            return
        self._post(self.grid.current_buffer())
        self._wait()

    def _exchange_phases(self):
        """Multi-axis layouts: the phases in ``order`` one after another, each
        slab carrying the ghost extensions of the canonically earlier axes
        (build_halo_plan), so x -> y -> z delivers edges and corners
        transitively like the reference (test_decomp.py:195-204).  Slabs are
        packed into dense buffers on the device (sp_copy_box), moved by NCCL
        send/recv, and unpacked into the ghost layers; a gloo group stages them
        through host memory."""
        import torch
        dist, g, h = self.dist, self.grid, self.h
        plan = build_halo_plan(h)
        stage = dist.get_backend(self.group) != "nccl" and g.current_buffer().is_cuda
        for name in self.order:
            axis, ext = plan[name]
            n = g.dims.shape[axis]
            ops, pending = [], []
            for high in (False, True):
                nb = self.decomp.neighbor(self.rank, axis, high=high)
                if nb is None:
                    continue
                sbuf = self.engine.pack(g, axis, ext, (n - h, n) if high else (0, h))
                if stage:
                    self.engine.sync(g)
                    sbuf = sbuf.cpu()
                rbuf = torch.empty_like(sbuf)
                ops.append(dist.P2POp(dist.isend, sbuf, self._global_rank(nb), self.group))
                ops.append(dist.P2POp(dist.irecv, rbuf, self._global_rank(nb), self.group))
                pending.append((rbuf, (n, n + h) if high else (-h, 0), sbuf))
                self.bytes_sent += sbuf.numel() * sbuf.element_size()
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
                self.messages += len(ops) // 2
            for rbuf, rng, _ in pending:
                if stage:
                    rbuf = rbuf.to(g.current_buffer().device)
                self.engine.unpack(g, axis, ext, rng, rbuf)

    # -- compute -------------------------------------------------------------

    def _domain(self, levels, done, T):
        """Final-level domain of a pass reaching level done+T of a ``levels`` step."""
        last = done + T
        shape = self.grid.dims.shape
        lo = tuple(-(levels - last) * self.e_lo[d] for d in range(3))
        hi = tuple(shape[d] + (levels - last) * self.e_hi[d] for d in range(3))
        return lo, hi

    def step(self, levels: int | None = None):
        """One outer step of ``levels`` <= h levels (default h).

        Overlapped: wait for the halos of the current state, run K2 on the two
        boundary slabs (the h planes each neighbour needs next), post their
        transfer, then run K2 on the interior slab while NCCL moves them.
        """
        g, h = self.grid, self.h
        r = h if levels is None else int(levels)
        if not 1 <= r <= h:
            raise DecompositionError(f"step of {r} levels needs 1 <= levels <= h={h}")
        if self.transport == "p2p":
            return self._step_p2p(r)
        if not self.overlap or r > self.depth:
            if self._primed:
                self._wait()
            else:
                self.exchange()
            self._primed = False
            done = 0
            while done < r:
                T = min(self.depth, r - done)
                lo, hi = self._domain(r, done, T)
                self.engine.run_pass(g, T, lo, hi, self.e_lo, self.e_hi, lo, hi)
                g.swap()
                done += T
            return
        if not self._primed:
            self._post(g.current_buffer())          # halos of the current state
            self._primed = True
        self._wait()
        lo, hi = self._domain(r, 0, r)
        nz = g.dims.nz
        low = ((0, lo[1], lo[2]), (h, hi[1], hi[2]))
        high = ((nz - h, lo[1], lo[2]), (nz, hi[1], hi[2]))
        inner = ((h, lo[1], lo[2]), (nz - h, hi[1], hi[2]))
        for olo, ohi in (low, high):
            self.engine.run_pass(g, r, lo, hi, self.e_lo, self.e_hi, olo, ohi)
        self._post(g.other_buffer())                 # boundary planes of the new state
        self.engine.run_pass(g, r, lo, hi, self.e_lo, self.e_hi, *inner)
        g.swap()

    def run(self, outer_steps: int):
        for _ in range(outer_steps):
            self.step()
        self.finish()

    def finish(self):
        """Complete in-flight halo transfers (the state is already final)."""
        self._wait()
        self._primed = False

    # -- results -------------------------------------------------------------

    def gather(self):
        """Rank 0 returns the gathered global interior (numpy); others None."""
        field = self.grid.interior()
        out = [None] * self.world if self.rank == 0 else None
        self.dist.gather_object(field, out, dst=self._global_rank(0), group=self.group)
        if self.rank != 0:
            return None
        full = np.empty(self.decomp.global_dims.shape, dtype=field.dtype)
        for r, f in enumerate(out):
            sl = tuple(slice(a, b) for a, b in self.decomp.ranges(r))
            full[sl] = f
        return full


def emulate_peer_slabs(global_dims: GridDims, pattern, ranks: int, h: int, levels, dtype=np.float64,
                       device=None):
    """Single-device emulation of the p2p transport: ``ranks`` z-slab grids in
    this process, each step's boundary launches storing straight into the
    neighbour slabs' ghost planes (the pointers a multi-GPU run maps through
    IPC), then the interior launches; one stream orders everything, which is
    what the per-step tokens guarantee across processes.  Returns the
    gathered global interior (numpy)."""
    from .decomp import local_grid
    from .pipeline import run_pass
    decomp = decompose(global_dims, ranks, (1, 1, ranks), h)
    grids = [local_grid(decomp, r, pattern, dtype=dtype, device=device) for r in range(ranks)]
    flags = [face_flags(decomp, r) for r in range(ranks)]
    nbs = [(decomp.neighbor(r, 0, high=False), decomp.neighbor(r, 0, high=True)) for r in range(ranks)]
    for lv in levels:
        if not 1 <= lv <= h:
            raise DecompositionError(f"step of {lv} levels needs 1 <= levels <= h={h}")
        inner_jobs = []
        for r, g in enumerate(grids):
            e_lo, e_hi = flags[r]
            shape = g.dims.shape
            lo, hi = (0, 0, 0), tuple(shape)
            nz = g.dims.nz
            lo_nb, hi_nb = nbs[r]
            k = 1 - g.active
            peer = (grids[lo_nb].buffers[k] if lo_nb is not None else None,
                    grids[lo_nb].dims.nz if lo_nb is not None else 0,
                    grids[hi_nb].buffers[k] if hi_nb is not None else None, -nz, h)
            for olo, ohi in (((0, 0, 0), (h, shape[1], shape[2])),
                             ((nz - h, 0, 0), (nz, shape[1], shape[2]))):
                run_pass(g, lv, lo, hi, e_lo, e_hi, out_lo=olo, out_hi=ohi, peer=peer)
            inner_jobs.append((g, lv, lo, hi, e_lo, e_hi, (h, 0, 0), (nz - h, shape[1], shape[2])))
        for g, lv, lo, hi, e_lo, e_hi, olo, ohi in inner_jobs:
            run_pass(g, lv, lo, hi, e_lo, e_hi, out_lo=olo, out_hi=ohi)
        for g in grids:
            g.swap()
    full = np.empty(decomp.global_dims.shape, dtype=grids[0].dtype)
    for r, g in enumerate(grids):
        sl = tuple(slice(a, b) for a, b in decomp.ranges(r))
        full[sl] = g.interior()
    return full
