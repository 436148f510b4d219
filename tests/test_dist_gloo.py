"""Multi-process z-slab halo exchange on CPU: world_size 2 (and 3), gloo backend.

Runs paper_0912_4506_b200.dist.SlabRunner -- the same exchange/overlap logic
bench.py uses with NCCL -- over a test-only host engine (tests/hostengine.py)
and checks the gathered field bit-for-bit against the reference's own
run_distributed output (tests/golden, R/decomp.py:240-268) and the oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

Z1 = (1.0, 0.0, 0.0, 0.0, 0.0, 0.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, h, steps, overlap, levels, q, transport="nccl"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist
    from hostengine import HostEngine
    from oracle import oracle as O
    import paper_0912_4506_b200 as sp
    from paper_0912_4506_b200.dist import SlabRunner

    import torch.multiprocessing as tmp
    tmp.set_sharing_strategy("file_system")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gshape = (40, 10, 12)
        base = O.BoxPattern("random", seed=0, faces=Z1, global_shape=gshape)
        r = SlabRunner(sp.GridDims(12, 10, 40), None, h=h, dtype=np.float64, depth=h,
                       engine=HostEngine(base), overlap=overlap, transport=transport)
        for lv in levels or [h] * steps:
            r.step(levels=lv)
        r.finish()
        full = r.gather()
        if rank == 0:
            q.put((full, r.overlap, r.messages))
    finally:
        dist.destroy_process_group()


def _run(world, h, steps, overlap=True, levels=None, transport="nccl"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, h, steps, overlap, levels, q, transport))
             for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("h,steps", [(1, 3), (4, 2)])
def test_two_ranks_match_reference(ref_fields, kat, h, steps, overlap):
    full, did_overlap, msgs = _run(2, h, steps, overlap)
    ref = ref_fields[f"dist_P2_h{h}_s{steps}"]
    assert full.shape == ref.shape
    assert np.array_equal(full.view(np.uint64), ref.view(np.uint64))
    assert did_overlap == overlap
    assert msgs > 0


def test_three_ranks_with_remainder_step(O):
    # 2 steps of h=4 then a 3-level remainder step: 11 levels in total
    full, _, _ = _run(3, 4, 0, True, levels=[4, 4, 3])
    g = O.CGrid((40, 10, 12), O.BoxPattern("random", seed=0, faces=Z1, global_shape=(40, 10, 12)))
    g.sweeps(11)
    assert np.array_equal(full.view(np.uint64), g.interior().view(np.uint64))


def _e2e_worker(rank, world, port, q, transport="nccl"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch
    import torch.distributed as dist
    import bench
    from hostengine import HostEngine
    from oracle import oracle as O
    import paper_0912_4506_b200 as sp
    from paper_0912_4506_b200.dist import SlabRunner

    import torch.multiprocessing as tmp
    tmp.set_sharing_strategy("file_system")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gshape = (40, 10, 12)
        base = O.BoxPattern("random", seed=0, faces=Z1, global_shape=gshape)
        r = SlabRunner(sp.GridDims(12, 10, 40), None, h=4, dtype=np.float64, depth=4,
                       engine=HostEngine(base), transport=transport)
        e2e = bench.measure_e2e_dist(torch, dist, [r], [4, 4], torch.device("cpu"), world, 40 * 10 * 12,
                                     steps=2)
        full = r.gather()
        if rank == 0:
            q.put((full, e2e, r.grid.current.numel()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_bench_e2e_at_two_ranks(ref_fields, transport):
    """bench.py's N>1 end-to-end leg: every step re-uploads the slab and reruns the sweeps."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_e2e_worker, args=(r, 2, port, q, transport)) for r in range(2)]
    for p in procs:
        p.start()
    full, e2e, n = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = ref_fields["dist_P2_h4_s2"]            # 8 levels from the initial field
    assert np.array_equal(full.view(np.uint64), ref.view(np.uint64))
    assert e2e["ms_per_step"] > 0 and e2e["unit"] == "GLUP/s"
    assert e2e["h2d_bytes_per_step"] == 2 * n * 8
    assert e2e["d2h_bytes_per_step"] == 2 * 20 * 10 * 12 * 8


@pytest.mark.parametrize("world,h,levels", [(2, 4, [4, 4]), (3, 2, [2, 2, 1, 2]), (2, 1, [1, 1, 1])])
def test_p2p_transport_peer_stores(O, world, h, levels):
    """transport="p2p": boundary passes store into the mapped neighbour grids,
    one token per neighbour and step; bit-identical to the undecomposed sweeps."""
    full, did_overlap, msgs = _run(world, h, 0, True, levels=levels, transport="p2p")
    g = O.CGrid((40, 10, 12), O.BoxPattern("random", seed=0, faces=Z1, global_shape=(40, 10, 12)))
    g.sweeps(sum(levels))
    assert np.array_equal(full.view(np.uint64), g.interior().view(np.uint64))
    assert msgs > 0


def _multi_worker(rank, world, port, layout, h, levels, shape, q, order):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist
    from hostengine import HostEngine
    from oracle import oracle as O
    import paper_0912_4506_b200 as sp
    from paper_0912_4506_b200.dist import SlabRunner

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nz, ny, nx = shape
        base = O.BoxPattern("random", seed=3, faces=FACES6, global_shape=shape)
        r = SlabRunner(sp.GridDims(nx, ny, nz), None, h=h, dtype=np.float64, depth=min(h, 3),
                       engine=HostEngine(base), layout=layout, order=order)
        for lv in levels:
            r.step(levels=lv)
        r.finish()
        full = r.gather()
        if rank == 0:
            q.put((full, r.messages, r.multi_axis))
    finally:
        dist.destroy_process_group()


FACES6 = (0.3, -1.0, 2.0, 0.0, 1.0, -0.5)


def _run_multi(world, layout, h, levels, shape, order=("x", "y", "z")):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_multi_worker, args=(r, world, port, layout, h, levels, shape, q, order))
             for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("world,layout,h,levels,shape", [
    (2, (2, 1, 1), 2, [2, 2, 2], (12, 10, 26)),       # x split
    (2, (1, 2, 1), 3, [3, 3], (11, 21, 14)),          # y split, uneven
    (4, (2, 2, 1), 2, [2, 2, 1], (9, 18, 20)),        # x and y: edge and corner halos
    (4, (1, 2, 2), 4, [4, 4], (30, 17, 12)),          # y and z
    (3, (3, 1, 1), 1, [1, 1, 1, 1], (8, 7, 31)),      # three ranks in x, h = 1
])
def test_multi_axis_runner_matches_oracle(O, world, layout, h, levels, shape):
    """multi-axis layouts in the multi-process runner -- the
    reference's extended-slab exchange x -> y -> z (R/decomp.py:125-179) with
    packed slabs over the process group, bit-identical to the undecomposed sweeps."""
    full, msgs, multi = _run_multi(world, layout, h, levels, shape)
    assert multi and msgs > 0
    g = O.CGrid(shape, O.BoxPattern("random", seed=3, faces=FACES6, global_shape=shape))
    g.sweeps(sum(levels))
    assert np.array_equal(full.view(np.uint64), g.interior().view(np.uint64))


def test_multi_axis_runner_phase_order_matters(O):
    """The reference's negative test (test_decomp.py:195-204): z -> y -> x loses
    the corner values, so the result differs from the oracle."""
    shape = (9, 18, 20)
    full, _, _ = _run_multi(4, (2, 2, 1), 2, [2, 2], shape, order=("y", "x", "z"))
    g = O.CGrid(shape, O.BoxPattern("random", seed=3, faces=FACES6, global_shape=shape))
    g.sweeps(4)
    assert not np.array_equal(full.view(np.uint64), g.interior().view(np.uint64))
