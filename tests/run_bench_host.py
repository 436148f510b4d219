"""Test-only launcher: bench.py's N>1 path on CPU (gloo) with the host test engine.

    python tests/run_bench_host.py --gpus 2 --workload tiny ...

Registers a tiny workload and the host engine (tests/hostengine.py: grids in
CPU memory, passes by the C oracle) in bench.HOOKS, then calls bench.main()
-- which, without torchrun's environment, re-runs THIS script under
torch.distributed.run with one rank per "GPU".  Used by
tests/test_bench_spawn.py; never by the product.
"""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

import bench  # noqa: E402

Z1 = (1.0, 0.0, 0.0, 0.0, 0.0, 0.0)
bench.WORKLOADS["tiny"] = ((20, 10, 12), "random", Z1, "f64", 8, "test: 12x10x20 per rank, 8 sweeps", False)
bench.WORKLOADS["tinys"] = ((40, 10, 12), "random", Z1, "f64", 8, "test: 12x10x40 split N ways, 8 sweeps",
                            True)


def _engine(gshape):
    from hostengine import HostEngine
    from oracle import oracle as O
    return HostEngine(O.BoxPattern("random", seed=0, faces=Z1, global_shape=tuple(gshape)))


def _verify(full):
    from oracle import oracle as O
    g = O.CGrid(full.shape, O.BoxPattern("random", seed=0, faces=Z1, global_shape=full.shape))
    g.sweeps(8)
    return {"checked": True, "match": bool(np.array_equal(full.view(np.uint64),
                                                          g.interior().view(np.uint64)))}


if "WORLD_SIZE" in os.environ:
    import torch.multiprocessing as tmp
    tmp.set_sharing_strategy("file_system")
bench.HOOKS.update(engine=_engine, backend="gloo", verify=_verify)
sys.exit(bench.main())
