"""sp_dist_*: the z-slab halo exchange + outer step behind the C ABI,
driven through ctypes the way a host without PyTorch would drive it.

* world = 1 on the one GPU: communicator set-up through NCCL (dlopen), steps,
  tear-down; bitwise against the oracle.
* world = 2 needs two GPUs (NCCL refuses two ranks on one device): the test is
  written and skips on a single-GPU box.
(R = /root/reference/pkg/src/stencilpipe; R/decomp.py:149-268)
"""
import ctypes
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FACES = (0.3, -1.0, 2.0, 0.0, 1.0, -0.5)


def _bitwise(a, b):
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(
        np.ascontiguousarray(a).view(np.uint8), np.ascontiguousarray(b).view(np.uint8))


def _steps(sp, g, comm, steps, T):
    """`steps` outer steps of depth T through sp_dist_step, swapping A/B like outer_step."""
    N = sp._native
    L = N.lib()
    for _ in range(steps):
        N.check(L.sp_dist_step(comm, ctypes.c_void_p(g.current_buffer().data_ptr()),
                               ctypes.c_void_p(g.other_buffer().data_ptr()), g.sp_dtype,
                               ctypes.byref(g.layout), T, g.stream()))
        g.swap()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_single_rank_communicator(sp, O, dtype):
    N = sp._native
    L = N.lib()
    shape = (21, 30, 66)
    g = sp.TwoGrid(sp.GridDims(shape[2], shape[1], shape[0]),
                   sp.FillPattern.dirichlet_box("random", shape, FACES, seed=0), dtype=dtype)
    uid = ctypes.create_string_buffer(128)
    N.check(L.sp_dist_unique_id(uid, 128))
    comm = ctypes.c_void_p()
    N.check(L.sp_dist_create(uid, 0, 1, ctypes.byref(comm)))
    try:
        _steps(sp, g, comm, 3, 4)
        _steps(sp, g, comm, 1, 3)
    finally:
        N.check(L.sp_dist_destroy(comm))
    ref = O.CGrid(shape, O.BoxPattern("random", seed=0, faces=FACES, global_shape=shape), dtype=dtype)
    ref.sweeps(15)
    assert _bitwise(g.interior(), ref.interior())


def test_argument_errors(sp):
    N = sp._native
    L = N.lib()
    uid = ctypes.create_string_buffer(128)
    assert L.sp_dist_unique_id(uid, 64) == N.SP_ERR_ARG
    N.check(L.sp_dist_unique_id(uid, 128))
    comm = ctypes.c_void_p()
    assert L.sp_dist_create(uid, 2, 2, ctypes.byref(comm)) == N.SP_ERR_DECOMP   # R/decomp.py:54-60 class
    with pytest.raises(sp.DecompositionError):
        N.check(L.sp_dist_create(uid, -1, 1, ctypes.byref(comm)))


def _rank_worker(rank, world, uid_bytes, h, steps, q):
    sys.path.insert(0, ROOT)
    import torch
    import paper_0912_4506_b200 as sp
    from paper_0912_4506_b200.decomp import decompose, local_grid
    torch.cuda.set_device(rank)
    N = sp._native
    L = N.lib()
    shape = (48, 20, 70)
    d = decompose(sp.GridDims(shape[2], shape[1], shape[0]), (1, 1, world), h)
    pat = sp.FillPattern.dirichlet_box("random", shape, FACES, seed=0)
    g = local_grid(d, rank, pat, device=torch.device("cuda", rank))
    comm = ctypes.c_void_p()
    N.check(L.sp_dist_create(ctypes.create_string_buffer(uid_bytes, 128), rank, world, ctypes.byref(comm)))
    _steps(sp, g, comm, steps, h)
    torch.cuda.synchronize()
    N.check(L.sp_dist_destroy(comm))
    q.put((rank, g.interior()))


def test_two_ranks_two_gpus(sp, O):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (NCCL refuses two ranks on one device)")
    N = sp._native
    uid = ctypes.create_string_buffer(128)
    N.check(N.lib().sp_dist_unique_id(uid, 128))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    h, steps, world = 4, 3, 2
    procs = [ctx.Process(target=_rank_worker, args=(r, world, uid.raw, h, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(60)
    shape = (48, 20, 70)
    ref = O.CGrid(shape, O.BoxPattern("random", seed=0, faces=FACES, global_shape=shape))
    ref.sweeps(h * steps)
    full = np.concatenate([parts[r] for r in range(world)], axis=0)
    assert _bitwise(full, ref.interior())
