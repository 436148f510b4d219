"""B200-native temporally blocked 3D Jacobi (hot path of arXiv 0912.4506).

Drop-in for the hot-path subset of the reference package ``stencilpipe``
(R/__init__.py:8-24): the same names and semantics, with the arithmetic in
sm_100a CUDA kernels behind the C ABI in include/stencilpipe_b200.h.
Grids live in HBM; there is no CPU compute path.
"""

from .grid import (ArrayPattern, CompressedGrid, FillPattern, GridDims, GridError, TwoGrid, allocate,
                   dump_field, load_field)
from .kernel import (ONE_SIXTH, block_edges, stencil_point, sweep_naive,
                     sweep_spatial_blocked, update_block)
from .pipeline import (DEFAULT_DEPTH, PipelineConfig, PipelineTimeout, ScheduleError,
                       default_block_size, run_node_sweeps, sweeps)
from .decomp import (Decomposition, DecompositionError, decompose, level_domains_for_rank,
                     local_grid, outer_step, run_distributed)
from .verify import (Comparison, F32_REL_TOL, REL_TOL, check_maximum_principle, compare, oracle,
                     oracle_trajectory)
from ._native import NativeUnavailable, build, launch_count

__version__ = "0.1.0"
