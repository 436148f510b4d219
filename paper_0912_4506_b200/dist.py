"""Multi-process z-slab runner: one process per GPU, halos over torch.distributed.

Mirrors the reference's distributed engine (exchange_halos + outer_step,
R/decomp.py:149-237, R/transport.py as the message layer) for layouts
(1, 1, P), with the halo exchange moved onto NCCL point-to-point
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

``engine`` abstracts the grid + pass implementation so the exchange logic is
testable on CPU with gloo (tests supply a host engine); the default is the
CUDA engine and there is no fallback.
(R = /root/reference/pkg/src/stencilpipe)
"""

from __future__ import annotations

import numpy as np

from .decomp import DecompositionError, decompose, face_flags, plane_spans
from .grid import GridDims
from .pipeline import DEFAULT_DEPTH, MAX_DEPTH


class CudaEngine:
    """Device grids + K2 passes through the C ABI."""

    def make_grid(self, decomp, rank, pattern, dtype, device):
        from .decomp import local_grid
        return local_grid(decomp, rank, pattern, dtype=dtype, device=device)

    def run_pass(self, grid, T, lo, hi, e_lo, e_hi, out_lo, out_hi):
        from .pipeline import run_pass
        run_pass(grid, T, lo, hi, e_lo, e_hi, out_lo=out_lo, out_hi=out_hi)

    def default_depth(self, grid):
        return DEFAULT_DEPTH[grid.sp_dtype]


class SlabRunner:
    """This rank's z-slab of a (1, 1, P) decomposition with halo depth h."""

    def __init__(self, global_dims: GridDims, pattern, h: int, dtype=np.float64,
                 depth: int | None = None, device=None, engine=None, overlap: bool = True,
                 group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.h = h
        self.decomp = decompose(global_dims, self.world, (1, 1, self.world), h)
        self.engine = engine or CudaEngine()
        self.grid = self.engine.make_grid(self.decomp, self.rank, pattern, dtype, device)
        self.depth = depth or self.engine.default_depth(self.grid)
        self.e_lo, self.e_hi = face_flags(self.decomp, self.rank)
        self.lo_nb = self.decomp.neighbor(self.rank, 0, high=False)
        self.hi_nb = self.decomp.neighbor(self.rank, 0, high=True)
        nz = self.grid.dims.nz
        # overlap needs one pass per outer step and a non-empty interior slab
        self.overlap = overlap and h <= min(self.depth, MAX_DEPTH) and nz > 2 * h
        self._pending = []
        self._primed = False
        self.messages = 0
        self.bytes_sent = 0

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
        self._post(self.grid.current_buffer())
        self._wait()

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


def check_layout(layout):
    if tuple(layout[:2]) != (1, 1):
        raise DecompositionError("SlabRunner decomposes in z only: layout (1, 1, P)")
