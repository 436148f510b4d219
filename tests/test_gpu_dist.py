"""Fused p2p halo exchange on the device (one B200).

* ``emulate_peer_slabs``: P z-slab grids in one process, the boundary K2
  launches storing straight into the neighbour slabs' ghost planes -- the
  kernel epilogue and pointer arithmetic of sp_sweep_tb_part_peer;
* two processes on the one GPU: SlabRunner(transport="p2p") with CUDA IPC
  mapped neighbour grids and host-delivered (gloo) tokens -- no kernel ever
  waits on another process, so this is safe on a single device.
Both are checked bit for bit against the oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

Z1 = (1.0, 0.0, 0.0, 0.0, 0.0, 0.0)
FACES = (0.3, -1.0, 2.0, 0.0, 1.0, -0.5)


def _oracle(O, shape, faces, levels, dtype=np.float64, kind="random"):
    g = O.CGrid(shape, O.BoxPattern(kind, seed=0, faces=faces, global_shape=shape), dtype=dtype)
    g.sweeps(levels)
    return g.interior()


def _bitwise(a, b):
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(
        np.ascontiguousarray(a).view(np.uint8), np.ascontiguousarray(b).view(np.uint8))


@pytest.mark.parametrize("ranks,h,levels,shape", [
    (2, 2, [2, 2, 2], (40, 34, 70)),
    (3, 4, [4, 3, 4], (41, 20, 130)),     # uneven split (14, 14, 13), remainder step
    (4, 1, [1] * 5, (17, 9, 33)),
    (2, 8, [8, 8], (50, 24, 24)),
    (2, 7, [7, 6, 5], (44, 30, 66)),      # peer-store forms of the depth-5..7 kernels
])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_emulated_peer_slabs(sp, O, ranks, h, levels, shape, dtype):
    from paper_0912_4506_b200.dist import emulate_peer_slabs
    nz, ny, nx = shape
    pat = sp.FillPattern.dirichlet_box("random", shape, FACES, seed=0)
    full = emulate_peer_slabs(sp.GridDims(nx, ny, nz), pat, ranks, h, levels, dtype=dtype)
    ref = _oracle(O, shape, FACES, sum(levels), dtype=dtype)
    assert _bitwise(full, ref)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ipc_worker(rank, world, port, h, levels, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import paper_0912_4506_b200 as sp
    from paper_0912_4506_b200.dist import SlabRunner

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape = (48, 20, 70)
        pat = sp.FillPattern.dirichlet_box("random", shape, FACES, seed=0)
        r = SlabRunner(sp.GridDims(70, 20, 48), pat, h=h, dtype=np.float64, depth=h,
                       device=torch.device("cuda", 0), transport="p2p")
        for lv in levels:
            r.step(levels=lv)
        r.finish()
        full = r.gather()
        if rank == 0:
            q.put((full, r.messages))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,h,levels", [(2, 2, [2, 2, 2, 1]), (3, 4, [4, 4])])
def test_p2p_runner_two_processes_one_gpu(O, world, h, levels):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, h, levels, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, msgs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert msgs > 0
    assert _bitwise(full, _oracle(O, (48, 20, 70), FACES, sum(levels)))


def _default_depth_worker(port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import paper_0912_4506_b200 as sp
    from paper_0912_4506_b200.dist import SlabRunner
    from paper_0912_4506_b200.pipeline import DEFAULT_DEPTH

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        shape = (30, 20, 70)
        pat = sp.FillPattern.dirichlet_box("random", shape, FACES, seed=0)
        # depth=None: the engine's tuned default (CudaEngine.default_depth)
        r = SlabRunner(sp.GridDims(70, 20, 30), pat, h=4, dtype=np.float64, device=torch.device("cuda", 0))
        assert r.depth == DEFAULT_DEPTH[sp._native.SP_F64]
        for lv in (4, 4, 2):
            r.step(levels=lv)
        r.finish()
        q.put(r.gather())
    finally:
        dist.destroy_process_group()


def test_slab_runner_default_depth(O):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_default_depth_worker, args=(_free_port(), q))
    p.start()
    full = q.get(timeout=300)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert _bitwise(full, _oracle(O, (30, 20, 70), FACES, 10))


def _multi_axis_worker(rank, world, port, layout, h, levels, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import paper_0912_4506_b200 as sp
    from paper_0912_4506_b200.dist import SlabRunner

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape = (26, 34, 70)
        pat = sp.FillPattern.dirichlet_box("random", shape, FACES, seed=0)
        r = SlabRunner(sp.GridDims(70, 34, 26), pat, h=h, dtype=np.float64, depth=h,
                       device=torch.device("cuda", 0), layout=layout)
        for lv in levels:
            r.step(levels=lv)
        r.finish()
        full = r.gather()
        if rank == 0:
            q.put((full, r.bytes_sent))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,layout,h,levels", [(2, (2, 1, 1), 2, [2, 2, 2]), (2, (1, 2, 1), 3, [3, 3]),
                                                   (4, (2, 2, 1), 2, [2, 2])])
def test_multi_axis_runner_device_pack(O, world, layout, h, levels):
    """Multi-axis layouts through the CUDA engine: halo slabs packed/unpacked by
    K6 (sp_copy_box) around the process-group exchange, passes on the extended
    domains; ranks share the one GPU (gloo, staged through host memory)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_multi_axis_worker, args=(r, world, port, layout, h, levels, q))
             for r in range(world)]
    for p in procs:
        p.start()
    full, sent = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sent > 0
    assert _bitwise(full, _oracle(O, (26, 34, 70), FACES, sum(levels)))
