"""Reference-compatible CLI with GPU rows (R/bench.py).

    python -m paper_0912_4506_b200 bench  [--variant naive|blocked|pipeline] ...
    python -m paper_0912_4506_b200 verify ...
    python -m paper_0912_4506_b200 dist   --layout 1x1xP ...

Same subcommands, flags and CSV/JSON ``COLUMNS`` as the reference's
``stencilpipe`` console script (R/bench.py:26-27,100-122,245-284), so GPU rows
and the reference's CPU rows land in one report.  GPU rows are tagged
``gpu-<variant>``; the ``T`` column stays the reference's updates-per-thread
and the device pass depth is ``--depth``.  Timing follows R/bench.py:125-156
(allocation/init untimed, one warm-up sweep, median of ``--reps``) with CUDA
events instead of ``time.monotonic``.

Verification: against the reference package's own code -- ``stencilpipe``
from ``--reference-path``, from the unmodified install in ``baseline/_ref``,
or from ``sys.path`` -- running ``sweep_naive`` on its own ``TwoGrid``
(R/verify.py:16-21; arrays cast to float32 for ``--dtype float32``, which
numpy keeps in float32, so both dtypes are checked bit for bit).  Without the
reference package ``verify``/``dist`` exit with status 2 and ``bench``
reports "skipped": the device is never compared with itself.
"""

from __future__ import annotations

import argparse
import json
import sys
from dataclasses import dataclass, replace

import numpy as np

from .grid import FillPattern, GridDims, allocate
from .kernel import sweep_naive, sweep_spatial_blocked
from .pipeline import PipelineConfig, default_block_size, run_node_sweeps, sweeps
from .verify import F32_REL_TOL, REL_TOL, compare

COLUMNS = ("variant", "nx", "ny", "nz", "n", "t", "T", "dl", "du", "dt",
           "sync", "storage", "sweeps", "seconds", "mlups", "verified")


@dataclass
class BenchResult:
    variant: str
    dims: GridDims
    cfg: PipelineConfig
    sweeps: int
    seconds: float
    updates: int
    verified: str

    @property
    def mlups(self) -> float:
        return self.updates / self.seconds / 1e6

    def row(self) -> dict:
        d, c = self.dims, self.cfg
        return {"variant": self.variant, "nx": d.nx, "ny": d.ny, "nz": d.nz,
                "n": c.teams, "t": c.team_size, "T": c.updates_per_thread,
                "dl": c.min_dist, "du": c.max_dist, "dt": c.team_delay,
                "sync": c.sync, "storage": c.storage, "sweeps": self.sweeps,
                "seconds": f"{self.seconds:.6f}", "mlups": f"{self.mlups:.3f}",
                "verified": self.verified}


def report(results, fmt: str = "csv") -> str:
    """Deterministic CSV (or JSON with the same fields), R/bench.py:56-63."""
    rows = [r.row() for r in results]
    if fmt == "json":
        return json.dumps(rows, indent=2) + "\n"
    lines = [",".join(COLUMNS)]
    lines += [",".join(str(row[c]) for c in COLUMNS) for row in rows]
    return "\n".join(lines) + "\n"


def _parse_triple(text: str):
    parts = text.lower().split("x")
    if len(parts) != 3:
        raise argparse.ArgumentTypeError(f"expected AxBxC, got {text!r}")
    return tuple(int(p) for p in parts)


def _pattern(args) -> FillPattern:
    if args.pattern == "constant":
        return FillPattern.constant(args.value)
    if args.pattern == "linear":
        return FillPattern.linear()
    if args.pattern == "hotplate":
        return FillPattern.hotplate()
    return FillPattern.random(args.seed)


def _dims(args, ghost: int = 1) -> GridDims:
    if args.dims is not None:
        nx, ny, nz = args.dims
    else:
        nx = ny = nz = args.size
    return GridDims(nx, ny, nz, ghost)


def _config(args) -> PipelineConfig:
    return PipelineConfig(teams=args.teams, team_size=args.team_size,
                          updates_per_thread=args.updates_per_thread, min_dist=args.dl,
                          max_dist=args.du, team_delay=args.dt, sync=args.sync,
                          block=args.block, storage=args.storage, depth=args.depth)


def _dtype(args):
    return np.float64 if args.dtype == "float64" else np.float32


def _timed(fn):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def _run_variant(variant, dims, pattern, cfg, n_sweeps, dtype):
    """Allocate, warm up, run timed; returns (grid, updates, seconds) (R/bench.py:125-156)."""
    interior = dims.nx * dims.ny * dims.nz
    grid = allocate(dims, "twogrid", pattern, dtype=dtype)
    if variant == "naive":
        sweep_naive(grid)
        sec = _timed(lambda: [sweep_naive(grid) for _ in range(n_sweeps)])
        return grid, interior * n_sweeps, sec
    if variant == "blocked":
        bs = cfg.block or default_block_size(dims, cfg)
        sweep_spatial_blocked(grid, bs)
        sec = _timed(lambda: [sweep_spatial_blocked(grid, bs) for _ in range(n_sweeps)])
        return grid, interior * n_sweeps, sec
    if variant == "pipeline":
        if cfg.block is None:
            cfg = replace(cfg, block=default_block_size(dims, cfg))
        if cfg.storage == "compressed":
            # warm-up plus timed run shift the origin by up to two node sweeps (R/bench.py:147-150)
            grid = allocate(dims, "compressed", pattern, slack=2 * cfg.levels_per_sweep, dtype=dtype)
        run_node_sweeps(grid, cfg, 1)
        sec = _timed(lambda: run_node_sweeps(grid, cfg, n_sweeps))
        return grid, interior * n_sweeps * cfg.levels_per_sweep, sec
    raise ValueError(f"unknown variant {variant!r}")


def _levels(variant, cfg, total_sweeps):
    if variant == "pipeline":
        return (total_sweeps + 1) * cfg.levels_per_sweep
    return total_sweeps + 1


class ReferenceUnavailable(RuntimeError):
    """The reference package (stencilpipe) is not importable: nothing to verify against."""


def _import_reference(args):
    import os
    roots = [args.reference_path] if getattr(args, "reference_path", None) else []
    roots.append(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref"))
    for r in roots:
        if r and os.path.isdir(os.path.join(r, "stencilpipe")) and r not in sys.path:
            sys.path.insert(0, r)
    try:
        import stencilpipe.grid as rg
        import stencilpipe.kernel as rk
    except ImportError as exc:
        raise ReferenceUnavailable("verification needs the reference package stencilpipe "
                                   "(--reference-path DIR, or install it into baseline/_ref)") from exc
    return rg, rk


def _reference_field(args, dims, pattern, levels, dtype):
    """Interior after ``levels`` naive sweeps by the reference package's own code
    (its TwoGrid + sweep_naive = R/verify.py:16-21's oracle), in ``dtype``."""
    rg, rk = _import_reference(args)
    rp = {"constant": lambda: rg.FillPattern.constant(args.value),
          "linear": rg.FillPattern.linear, "hotplate": rg.FillPattern.hotplate,
          "random": lambda: rg.FillPattern.random(args.seed)}[args.pattern]()
    g = rg.allocate(rg.GridDims(dims.nx, dims.ny, dims.nz), "twogrid", rp)
    if dtype == np.float32:
        g.a = g.a.astype(np.float32)
        g.b = g.a.copy()
    for _ in range(levels):
        rk.sweep_naive(g)
    return np.ascontiguousarray(g.interior()), "reference"


def _tol(dtype):
    return REL_TOL if dtype == np.float64 else F32_REL_TOL


def cmd_bench(args) -> int:
    dims, pattern, cfg, dtype = _dims(args), _pattern(args), _config(args), _dtype(args)
    results = []
    for variant in args.variant:
        runs = []
        for _ in range(args.reps):
            grid, updates, seconds = _run_variant(variant, dims, pattern, cfg, args.sweeps, dtype)
            runs.append((seconds, updates, grid))
        runs.sort(key=lambda r: r[0])
        seconds, updates, grid = runs[len(runs) // 2]
        verified = "skipped"
        if not args.no_verify and max(dims.shape) <= 64:
            try:
                ref, _ = _reference_field(args, dims, pattern, _levels(variant, cfg, args.sweeps), dtype)
                verified = "yes" if compare(ref, grid, tol=_tol(dtype)).passed else "no"
            except ReferenceUnavailable:
                verified = "skipped"
        results.append(BenchResult("gpu-" + variant, dims, cfg, args.sweeps, seconds, updates, verified))
        if args.dump:                                   # R/bench.py:187-189
            from .grid import dump_field
            with open(args.dump, "w") as fh:
                dump_field(grid, fh)
    sys.stdout.write(report(results, args.format))
    return 1 if any(r.verified == "no" for r in results) else 0


def cmd_verify(args) -> int:
    """R/bench.py:194-207: node sweeps on the device against the reference's oracle."""
    dims, pattern, cfg, dtype = _dims(args), _pattern(args), _config(args), _dtype(args)
    if cfg.block is None:
        cfg = replace(cfg, block=default_block_size(dims, cfg))
    slack = cfg.levels_per_sweep if cfg.storage == "compressed" else None
    grid = allocate(dims, cfg.storage, pattern, slack=slack, dtype=dtype)
    run_node_sweeps(grid, cfg, args.sweeps)
    try:
        ref, source = _reference_field(args, dims, pattern, args.sweeps * cfg.levels_per_sweep, dtype)
    except ReferenceUnavailable as exc:
        print(f"verify: {exc}", file=sys.stderr)
        return 2
    cmp = compare(ref, grid, tol=_tol(dtype))
    print(f"verify gpu-{cfg.storage}/{source} n={cfg.teams} t={cfg.team_size} T={cfg.updates_per_thread} "
          f"depth={cfg.depth or 'auto'} sweeps={args.sweeps}: {cmp}")
    return 0 if cmp.passed else 1


def cmd_dist(args) -> int:
    from .decomp import run_distributed
    dims, pattern, cfg, dtype = _dims(args), _pattern(args), _config(args), _dtype(args)
    gathered, _ = run_distributed(dims, pattern, args.layout, cfg, args.outer_steps, dtype=dtype)
    levels = args.outer_steps * cfg.levels_per_sweep
    try:
        ref, source = _reference_field(args, dims, pattern, levels, dtype)
    except ReferenceUnavailable as exc:
        print(f"dist: {exc}", file=sys.stderr)
        return 2
    cmp = compare(ref, gathered, tol=_tol(dtype))
    print(f"dist layout={'x'.join(map(str, args.layout))} h={cfg.levels_per_sweep} "
          f"steps={args.outer_steps} ({source}): {cmp}")
    return 0 if cmp.passed else 1


def _add_config_flags(p):
    p.add_argument("--size", type=int, default=48, help="cubic interior extent")
    p.add_argument("--dims", type=_parse_triple, default=None, help="interior NXxNYxNZ")
    p.add_argument("--teams", type=int, default=1)
    p.add_argument("--team-size", type=int, default=4)
    p.add_argument("-T", "--updates-per-thread", type=int, default=2)
    p.add_argument("--dl", type=int, default=1)
    p.add_argument("--du", type=int, default=4)
    p.add_argument("--dt", type=int, default=0)
    p.add_argument("--block", type=_parse_triple, default=None)
    p.add_argument("--sync", choices=("barrier", "relaxed"), default="relaxed")
    p.add_argument("--storage", choices=("twogrid", "compressed"), default="twogrid")
    p.add_argument("--pattern", choices=("constant", "linear", "hotplate", "random"), default="random")
    p.add_argument("--value", type=float, default=0.0)
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--sweeps", type=int, default=2)
    p.add_argument("--depth", type=int, default=None, help="device levels per HBM pass (1..8)")
    p.add_argument("--dtype", choices=("float64", "float32"), default="float64")
    p.add_argument("--reference-path", default=None,
                   help="directory holding the reference package stencilpipe (for verification)")


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_0912_4506_b200",
                                     description="B200 temporally blocked 3D Jacobi (stencilpipe-compatible)")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("bench", help="time device variants and report MLUP/s")
    _add_config_flags(p)
    p.add_argument("--variant", action="append", choices=("naive", "blocked", "pipeline"), default=None)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--no-verify", action="store_true")
    p.add_argument("--format", choices=("csv", "json"), default="csv")
    p.add_argument("--dump", default=None, help="write the final field here (the reference's text format)")
    p.set_defaults(func=cmd_bench)
    p = sub.add_parser("verify", help="oracle equivalence for one configuration")
    _add_config_flags(p)
    p.set_defaults(func=cmd_verify)
    p = sub.add_parser("dist", help="z-slab multi-rank run with verification")
    _add_config_flags(p)
    p.add_argument("--layout", type=_parse_triple, default=(1, 1, 2))
    p.add_argument("--outer-steps", type=int, default=2)
    p.set_defaults(func=cmd_dist)
    return parser


def cli_main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    if getattr(args, "variant", "sentinel") is None:
        args.variant = ["naive"]
    return args.func(args)


def main() -> None:
    sys.exit(cli_main())
