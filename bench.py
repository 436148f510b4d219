#!/usr/bin/env python
"""Benchmark: temporally blocked 3D Jacobi on B200 (BASELINE.json metric GLUP/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c3|c2|c4|c5w|c5s] [--depth T]

One "step" = one full BASELINE run of the workload (C3: 100 sweeps of the
1024^3 fp64 grid) over inputs already resident in HBM.  N=1 runs C3 on one
GPU.  N>1 runs BASELINE C5 as z-slabs, one process per GPU: `c5w` (the N>1
default) is weak scaling, 1024 x 1024 x 512 per GPU; `c5s` is strong
scaling, the global 1024 x 1024 x 2048 grid split N ways.  Halos of depth
h = T (default 4, BASELINE C5's h in {1, 4, 8}) are exchanged every T
sweeps and overlapped with interior compute (dist.SlabRunner).  Without
torchrun's environment, `--gpus N` (N > 1) re-runs this script under
`torch.distributed.run` itself, one rank per GPU.

Rank 0 prints ONE JSON line.  Besides the driver's keys it carries:
  roofline          the dominant kernel (K2) against measured HBM bandwidth
                    (algorithmic bytes 16 B/cell per pass / CUDA-event pass time)
  temporal_roofline GLUP/s against R(T) = min(P_fp64/6, B_hbm*T/16) with the
                    FP64 add rate measured on this GPU at run time
  cpu_baseline      the C oracle (a port of the reference's sweep) on this
                    host's cores, bounded sample (rank 0, N=1 only)
  e2e               the same metric through the public API with the grid
                    uploaded from pinned host memory and the interior read
                    back every step (a stream of independent problems
                    pipelined over three device grids and three streams)
  clocks            nvidia-smi samples taken during the timed region
--impl reference times the reference algorithm's CPU implementation (the
oracle port, all host threads) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

Z1 = (1.0, 0.0, 0.0, 0.0, 0.0, 0.0)
WORKLOADS = {
    # name: (shape (nz, ny, nx) per GPU -- global for strong scaling, kind, faces, dtype, sweeps,
    #        description, strong)
    "c3": ((1024, 1024, 1024), "random", (1.0, 0.0, 0.5, 0.0, 0.25, 0.0), "f64", 100,
           "C3: fp64 interior 1024^3, Dirichlet faces (z-,z+,y-,y+,x-,x+)=(1,0,0.5,0,0.25,0), "
           "random(0) interior, 100 sweeps", False),
    "c2": ((512, 512, 512), "random", Z1, "f64", 200,
           "C2: fp64 interior 512^3, face z-=1, random(0), 200 sweeps", False),
    "c4": ((2048, 1024, 1024), "random_pm1", (0.0,) * 6, "f32", 200,
           "C4: fp32 interior 1024x1024x2048, uniform[-1,1) from random(0), zero faces, 200 sweeps", False),
    "c5w": ((512, 1024, 1024), "random", Z1, "f64", 100,
            "C5 weak: fp64 1024x1024x512 per GPU, face z-=1, random(0), 100 sweeps", False),
    "c5s": ((2048, 1024, 1024), "random", Z1, "f64", 100,
            "C5 strong: fp64 global 1024x1024x2048 split into N z-slabs, face z-=1, random(0), "
            "100 sweeps", True),
}
C5_DEPTH = 4        # BASELINE C5: ghost depth h = T in {1, 4, 8}

# Test-only injection (tests/run_bench_host.py): {"engine": factory(pattern_shape) -> engine,
# "backend": "gloo"} runs the N>1 path on CPU with the host test engine.  Empty in production.
HOOKS = {}


def load_json(path):
    try:
        with open(path) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return None


def measured_peaks():
    p = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"))
    if p and "hbm_gbs" in p:
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU legs (oracle port of the reference algorithm) -- rank 0 only
# ---------------------------------------------------------------------------

def cpu_sample(shape_full, kind, faces, dtype, budget_s=10.0, planes=64, sweeps_per_rep=4):
    """GLUP/s of the oracle (C port of sweep_naive, all host threads) on a
    z-slab of the workload; repeats until ``budget_s`` of CPU time elapsed."""
    import numpy as np
    from oracle import oracle as O
    O.build_c()
    nz, ny, nx = shape_full
    pz = min(planes, nz)
    shape = (pz, ny, nx)
    g = O.CGrid(shape, O.BoxPattern(kind, seed=0, faces=faces, global_shape=shape_full),
                dtype=np.float64 if dtype == "f64" else np.float32)
    g.sweeps(1)   # warm-up (page faults, threads)
    t0 = time.monotonic()
    lups = 0
    while True:
        g.sweeps(sweeps_per_rep)
        lups += nx * ny * pz * sweeps_per_rep
        if time.monotonic() - t0 >= budget_s:
            break
    dt = time.monotonic() - t0
    sample = (f"{nx}x{ny}x{pz} slab of the workload (same init/faces), "
              f"{lups // (nx * ny * pz)} sweeps, {dt:.1f} s")
    return lups / dt / 1e9, O.num_threads(), sample


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def reference_variants(shape_full, dt, T, budget_s=10.0):
    """The reference package's OWN CPU code (stencilpipe, installed unmodified
    into baseline/_ref by `pip install --target baseline/_ref`), timed like
    its bench (R/bench.py:125-156: allocate + one untimed warm-up sweep, then
    repeat until ``budget_s`` has elapsed) on a z-slab of the workload.  The
    four variants SURVEY 8(d) names: sweep_naive and sweep_spatial_blocked
    (numpy ufuncs: one core), run_node_sweeps with PipelineConfig(1, C, 1)
    (the paper's pipelined scheme at full width, C = host cores) and with
    PipelineConfig(1, 1, T) (the GPU's depth)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "stencilpipe")):
        return {"unavailable": "baseline/_ref not installed (pip install --target baseline/_ref)"}
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import numpy as np
    from stencilpipe.grid import FillPattern, GridDims, allocate
    from stencilpipe.kernel import sweep_naive, sweep_spatial_blocked
    from stencilpipe.pipeline import PipelineConfig, default_block_size, run_node_sweeps

    cores = len(os.sched_getaffinity(0))
    nz, ny, nx = shape_full
    wide = max(2, min(cores, 64))
    planes = min(nz, max(32, wide))
    dims = GridDims(nx, ny, planes)
    cells = nx * ny * planes

    def grid():
        g = allocate(dims, "twogrid", FillPattern.random(0))
        if dt == "f32":                          # numpy keeps f32 arithmetic in f32 (NEP 50)
            g.a = g.a.astype(np.float32)
            g.b = g.a.copy()
        return g

    def timed(name, one, levels_per_call, detail):
        g = grid()
        one(g)                                   # warm-up, untimed
        t0 = time.monotonic()
        calls = 0
        while True:
            one(g)
            calls += 1
            if time.monotonic() - t0 >= budget_s:
                break
        el = time.monotonic() - t0
        return {"variant": name, "glups": round(cells * levels_per_call * calls / el / 1e9, 5),
                "seconds": round(el, 2), "levels": levels_per_call * calls, "detail": detail}

    rows = []
    bs = (nx, ny, 16)
    rows.append(timed("naive", sweep_naive, 1, "sweep_naive (R/kernel.py:43-47), 1 core"))
    rows.append(timed("blocked", lambda g: sweep_spatial_blocked(g, bs), 1,
                      f"sweep_spatial_blocked bs={bs} (R/kernel.py:59-80), 1 core"))
    for label, cfg in ((f"pipeline(1,{wide},1)", PipelineConfig(teams=1, team_size=wide, updates_per_thread=1)),
                       (f"pipeline(1,1,{T})", PipelineConfig(teams=1, team_size=1, updates_per_thread=T))):
        cfg = PipelineConfig(teams=cfg.teams, team_size=cfg.team_size, updates_per_thread=cfg.updates_per_thread,
                             block=default_block_size(dims, cfg))
        rows.append(timed(label, lambda g, c=cfg: run_node_sweeps(g, c, 1), cfg.levels_per_sweep,
                          f"run_node_sweeps {label} block={cfg.block} (R/pipeline.py:459-462), "
                          f"{cfg.n_threads} threads"))
    return {"sample": f"{nx}x{ny}x{planes} z-slab (random(0) fill), {budget_s:.0f} s per variant",
            "cores": cores, "cpu_model": cpu_model(), "variants": rows}


def run_reference_arm(args, rank):
    """The reference arm: the reference algorithm's CPU implementation on this
    host.  Reported value: the C port of sweep_naive (oracle/, all host
    threads; faster than the reference's numpy code), timed >= 5 s per run;
    beside it the reference package's own code (reference_variants)."""
    if rank != 0:
        return 0
    shape, kind, faces, dt, sweeps, desc, strong = WORKLOADS[args.workload]
    if strong:                 # a bounded sample: the per-rank slab shape does not matter here
        shape = (shape[0] // max(args.gpus, 1), shape[1], shape[2])
    import numpy as np
    from oracle import oracle as O
    O.build_c()
    nz, ny, nx = shape
    planes = 32
    g = O.CGrid((planes, ny, nx), O.BoxPattern(kind, seed=0, faces=faces, global_shape=shape),
                dtype=np.float64 if dt == "f64" else np.float32)
    # sweeps of the slab per step: enough that the K timed steps take >= 5 s
    g.sweeps(1)                                   # first touch, thread start-up
    t0 = time.monotonic()
    g.sweeps(2)
    one = max((time.monotonic() - t0) / 2, 1e-3)
    per_step = max(2, int(np.ceil(6.0 / (one * max(args.steps, 1)))))
    for _ in range(args.warmup):
        g.sweeps(per_step)
    t0 = time.monotonic()
    for _ in range(args.steps):
        g.sweeps(per_step)
    el = time.monotonic() - t0
    lups = nx * ny * planes * per_step * args.steps
    v = lups / el / 1e9
    cores = O.num_threads()
    sample = (f"{nx}x{ny}x{planes} z-slab of {args.workload} ({per_step} sweeps per step, {el:.1f} s timed), "
              f"oracle C port of sweep_naive (R/kernel.py:43-47) on {cores} threads")
    T = args.depth or (C5_DEPTH if args.workload.startswith("c5") else 2)
    variants = reference_variants(shape, dt, T, budget_s=args.cpu_seconds) if not args.no_cpu else None
    line = {
        "metric": "GLUP/s", "value": round(v, 3), "unit": "GLUP/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": dt, "data": "synthetic",
        "config": {"workload": desc, "sample": sample},
        "cpu_baseline": {"value": round(v, 3), "unit": "GLUP/s", "cores": cores, "kind": "port",
                         "sample": sample, "cpu_model": cpu_model()},
        "reference_package": variants,
        "e2e": {"value": round(v, 3), "unit": "GLUP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args):
    """`--gpus N` (N > 1) without torchrun's environment: re-run this script
    under torch.distributed.run, one rank per GPU (127.0.0.1 rendezvous); rank
    0's JSON line reaches our stdout."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(sys.argv[0]),
           *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=None,
                    help="default: c3 at N=1, c5w (weak scaling) at N>1")
    ap.add_argument("--depth", type=int, default=0,
                    help="levels per HBM pass = halo depth h for c5* (0 = tuned default; c5*: 4)")
    ap.add_argument("--variant", type=int, default=0, help="kernel variant override (dev)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg")
    ap.add_argument("--no-verify", action="store_true",
                    help="skip the parity check (one more run of the workload from its initial "
                         "field, digest against tests/golden/big_digests.json)")
    ap.add_argument("--storage", choices=("twogrid", "compressed"), default="twogrid",
                    help="A/B grids or single-array in-place storage (N=1)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--transport", choices=("p2p", "nccl"), default="p2p",
                    help="N>1 halo exchange: p2p = boundary kernels store into the neighbours' "
                         "grids (CUDA IPC, NVLink), nccl = NCCL send/recv of the planes")
    ap.add_argument("--slab-runner", action="store_true",
                    help="dev: use the multi-GPU SlabRunner path even at N=1 (run under torchrun)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.workload is None:
        args.workload = "c3" if world == 1 and args.gpus <= 1 else "c5w"

    if args.impl == "reference":
        return run_reference_arm(args, rank)

    import numpy as np
    import torch
    import paper_0912_4506_b200 as sp
    from paper_0912_4506_b200 import _native as N
    from paper_0912_4506_b200.pipeline import DEFAULT_DEPTH

    engine = HOOKS.get("engine")
    cuda = engine is None
    if cuda:
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
    else:
        dev = torch.device("cpu")
    dist = None
    use_runner = world > 1 or args.slab_runner
    if use_runner and args.storage != "twogrid":
        raise SystemExit("--storage compressed has no multi-GPU (slab runner) form")
    if use_runner:
        import torch.distributed as dist
        if cuda:
            # communicator-init lines (rank count) on stderr; stdout keeps the one JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(HOOKS.get("backend", "gloo"))

    shape, kind, faces, dt, sweeps, desc, strong = WORKLOADS[args.workload]
    dtype = np.float64 if dt == "f64" else np.float32
    es = 8 if dt == "f64" else 4
    lib = N.lib() if cuda else None
    if args.variant:
        lib.sp_set_tuning(args.variant, 0)
    sp_dtype = N.SP_F64 if dt == "f64" else N.SP_F32
    from paper_0912_4506_b200.pipeline import DEFAULT_DEPTH_INPLACE
    T = args.depth or (C5_DEPTH if args.workload.startswith("c5") else
                       DEFAULT_DEPTH_INPLACE[sp_dtype] if args.storage == "compressed" else DEFAULT_DEPTH[sp_dtype])
    if strong:
        gshape = shape
    else:
        gshape = (shape[0] * world, shape[1], shape[2])
    nz_g, ny, nx = gshape
    passes = [T] * (sweeps // T) + ([sweeps % T] if sweeps % T else [])

    # --- FP64 compute roof, measured on this GPU ---
    import ctypes
    p_fp64 = float("nan")
    if cuda:
        rate, ms = ctypes.c_double(), ctypes.c_double()
        N.check(lib.sp_probe_fp64(ctypes.byref(rate), ctypes.byref(ms)))
        p_fp64 = rate.value

    pat = sp.FillPattern.dirichlet_box(kind, gshape, faces, seed=0)
    stream = torch.cuda.current_stream(dev) if cuda else None
    pass_times = []
    transport = None

    class Clock:
        """CUDA events on the launching stream; perf_counter for the CPU test engine."""

        def __init__(self):
            if cuda:
                self.e = torch.cuda.Event(enable_timing=True)
                self.e.record(stream)
            else:
                self.t = time.perf_counter()

        def until(self, other):
            return self.e.elapsed_time(other.e) / 1e3 if cuda else other.t - self.t

    runners = []
    if not use_runner:
        Grid = sp.CompressedGrid if args.storage == "compressed" else sp.TwoGrid
        grid = Grid(sp.GridDims(nx, ny, nz_g), pat, dtype=dtype, device=dev)
        cells_rank = nx * ny * nz_g

        def run_pass(t):
            sp.sweeps(grid, t, depth=t)

        def finish():
            pass
    else:
        from paper_0912_4506_b200.dist import SlabRunner
        transport = args.transport if world > 1 else "nccl"

        def make_runner(tr):
            kw = {"engine": engine(gshape)} if engine is not None else {}
            return SlabRunner(sp.GridDims(nx, ny, nz_g), pat, h=T, dtype=dtype, device=dev,
                              depth=T, transport=tr, **kw)
        try:
            runner = make_runner(transport)
        except Exception as exc:          # p2p mapping refused (no peer access): NCCL planes
            if transport != "p2p":
                raise
            transport = f"nccl (p2p setup failed: {type(exc).__name__}: {exc})"[:200]
            runner = make_runner("nccl")
        runners.append(runner)
        grid = runner.grid
        cells_rank = grid.dims.nx * grid.dims.ny * grid.dims.nz

        def run_pass(t):
            runner.step(levels=t)

        def finish():
            runner.finish()

    def step(record=False):
        for t in passes:
            c0 = Clock() if record else None
            run_pass(t)
            if record:
                pass_times.append((t, c0, Clock()))
        finish()

    def barrier():
        if dist is not None:
            dist.barrier()
        if cuda:
            torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    barrier()

    sampler = ClockSampler(local) if rank == 0 and cuda else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    n0 = N.launch_count()
    barrier()
    c0 = Clock()
    for k in range(args.steps):
        step(record=True)
    c1 = Clock()
    barrier()
    launches = N.launch_count() - n0
    clocks = sampler.stop() if sampler else None
    elapsed = c0.until(c1)
    if dist is not None:
        t = torch.tensor([elapsed], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    total_lups = nx * ny * nz_g * sweeps * args.steps
    value = total_lups / elapsed / 1e9

    # dominant kernel: full-depth passes (K2 at depth T; at N>1 the boundary + interior launches)
    full = [a.until(b) for t, a, b in pass_times if t == T]
    t_pass = sum(full) / len(full)
    alg_bytes = 2 * es * cells_rank                 # read A once + write B once per pass
    achieved = alg_bytes / t_pass / 1e9
    hbm, hbm_src = measured_peaks()
    traffic = None
    tj = load_json(os.path.join(ROOT, "profiles", "traffic.json")) or {}
    key = f"{args.workload}_T{T}_v{args.variant or 0}_n{world}" + (
        "_compressed" if args.storage == "compressed" else "")
    ncu_evidence = None
    if key in tj:
        traffic = tj[key].get("dram_bytes_per_launch")
        # per-LUP DRAM bytes and FP64 pipe use of the same kernel (one ncu --set full capture)
        ncu_evidence = {"dram_bytes_per_lup": round(traffic / (cells_rank * T), 3) if traffic else None,
                        "algorithmic_bytes_per_lup": round(2 * es / T, 3),
                        "fp64_pipe_active_pct": tj[key].get("fp64_pipe_active_pct"),
                        "issue_active_pct": tj[key].get("issue_active_pct"),
                        "lsu_pipe_pct": tj[key].get("lsu_pipe_pct"),
                        "source": tj[key].get("source")}

    # the K2 kernel of this depth: tq_kernel (z-queue in tensor memory) or tb_kernel (register queue)
    k2_desc = N.describe_variant(sp_dtype, T) if cuda else ""
    if args.storage == "twogrid":
        k2_name = "tq_kernel" if "tensor memory" in k2_desc else "tb_kernel"
    else:   # in-place passes: the FQ forms of tq_kernel from T=3 (csrc/host.cuh, kInplace*)
        k2_name = "tq_kernel (in place)" if T >= (3 if dt == "f64" else 4) else "tb_kernel (in place)"
    R_hbm = hbm * T / (2 * es)                      # GLUP/s, HBM term
    R_fp = p_fp64 / 6 / 1e9 if dt == "f64" and cuda else float("inf")
    R = min(R_hbm, R_fp) * world

    # --- e2e: the public API with host buffers ---
    e2e = None
    if not args.no_e2e:
        if not use_runner:
            # a stream of independent problems: >= 24 steps so the pipeline's fill
            # (first upload) and drain (last download) are a small share
            e2e = measure_e2e(sp, torch, np, grid, dtype, passes, dev, stream, steps=max(args.steps, 24))
        else:
            # three NCCL-transport runners: upload k+1 | sweeps k | download k-1 on three streams
            # (the fused p2p transport stores into neighbours' grids, which an upload would race)
            e2e_runners = [r for r in runners if r.transport == "nccl"]
            while len(e2e_runners) < 3:
                kw = {"engine": engine(gshape)} if engine is not None else {}
                e2e_runners.append(SlabRunner(sp.GridDims(nx, ny, nz_g), pat, h=T, dtype=dtype, device=dev,
                                              depth=T, transport="nccl", **kw))
                runners.append(e2e_runners[-1])
            e2e = measure_e2e_dist(torch, dist, e2e_runners, passes, dev, world, nx * ny * nz_g,
                                   steps=max(args.steps, 12) if cuda else max(args.steps, 2))

    verify = None if args.no_verify else verify_result(
        args, torch, dist, rank, world, cuda, grid, runners, passes, gshape, kind, faces, dt, sweeps)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.slab_runner:
        v, cores, sample = cpu_sample(shape, kind, faces, dt, budget_s=args.cpu_seconds)
        cpu = {"value": round(v, 3), "unit": "GLUP/s", "cores": cores, "kind": "port",
               "sample": sample}

    if rank == 0:
        line = {
            "metric": "GLUP/s",
            "value": round(value, 2),
            "unit": "GLUP/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(elapsed / args.steps * 1e3, 3),
            "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None,
            "dtype": dt,
            "data": "synthetic (seeded coordinate hash random(0), Dirichlet faces; no dataset)",
            "config": {"workload": desc, "T": T, "halo_depth": T if use_runner else None,
                       "passes_per_step": len(passes),
                       "global_interior_zyx": list(gshape),
                       "per_gpu_interior_zyx": [grid.dims.nz, grid.dims.ny, grid.dims.nx],
                       "parallelism": f"zslab{world}", "variant": args.variant or "auto",
                       "kernel": (N.describe_variant(sp_dtype, T) if args.storage == "twogrid"
                                  else "in-place variant (compressed storage, sp_sweep_tb_inplace)")
                       if cuda else "host test engine",
                       "storage": args.storage,
                       "halo_transport": transport if use_runner else None,
                       "l2": "inputs larger than L2 (one grid = %.1f GB >> 126 MB)" % (
                           grid.buffers[0].numel() * es / 1e9),
                       "hbm_grid_bytes": sum(b.numel() * b.element_size() for b in grid.buffers)},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(achieved / hbm, 4), "traffic": traffic,
                         "kernel": "%s T=%d" % (k2_name, T), "peak_source": hbm_src,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "avg_launch_ms": round(t_pass * 1e3, 3), "ncu": ncu_evidence},
            "temporal_roofline": {"T": T, "R_glups": round(R, 1), "frac": round(value / R, 4),
                                  "R_hbm_glups": round(R_hbm * world, 1),
                                  "R_fp64_glups": round(R_fp * world, 1) if R_fp != float("inf") else None,
                                  "fp64_dadd_per_s": p_fp64 if cuda else None, "hbm_gbs": hbm},
            "gpu_launches": launches,
            "verify": verify,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "impl": "ours",
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        for r in runners:
            r.close()
        dist.barrier()
        dist.destroy_process_group()
    return 0


def verify_result(args, torch, dist, rank, world, cuda, grid, runners, passes, gshape, kind, faces, dt,
                  sweeps):
    """Parity of the measured path: rerun the workload once from its initial
    field (untimed) and compare the 64-bit digest of the (gathered) interior
    -- slab digests summed mod 2^64 at N>1 -- with the oracle's golden digest
    for this global grid (tests/golden/big_digests.json, written by the pinned
    C oracle).  The CPU test engine hands the gathered field to HOOKS."""
    if not (cuda or "verify" in HOOKS):
        return None
    want = None
    if cuda:
        golden = load_json(os.path.join(ROOT, "tests", "golden", "big_digests.json")) or {}
        for key, g in golden.items():
            if (tuple(g["shape"]) == tuple(gshape) and g["kind"] == kind
                    and tuple(g["faces"]) == tuple(faces) and str(sweeps) in g["digests"]
                    and g["dtype"] == ("float64" if dt == "f64" else "float32")):
                want = (key, int(g["digests"][str(sweeps)]))
        if want is None:
            return {"checked": False, "reason": f"no golden digest for {list(gshape)} x {sweeps} sweeps"}
    if runners:
        r = runners[0]
        r.finish()
        r.grid.reset()
        r.sync_start()
        for t in passes:
            r.step(levels=t)
        r.finish()
        if not cuda:
            full = r.gather()
            return HOOKS["verify"](full) if rank == 0 else None
        g = r.grid
        z0 = r.decomp.ranges(r.rank)[0][0]
        v = g.digest(index_base=z0 * g.dims.ny * g.dims.nx)
        d = torch.tensor([v - (1 << 64) if v >= 1 << 63 else v], dtype=torch.int64, device=g.device)
        dist.all_reduce(d)                                 # int64 sum wraps mod 2^64
        got = int(d.item()) & ((1 << 64) - 1)
    else:
        import paper_0912_4506_b200 as sp
        grid.reset()
        sp.sweeps(grid, sweeps, depth=max(passes))
        got = grid.digest()
    return {"checked": True, "golden": want[0], "sweeps": sweeps, "digest": str(got),
            "expected": str(want[1]), "match": got == want[1]}


def measure_e2e_dist(torch, dist, runners, passes, dev, world, global_cells, steps=3):
    """e2e at N GPUs: a stream of independent problems, each uploaded per rank
    (the rank's ghosted z-slab from pinned host memory), swept through
    SlabRunner (NCCL halos) and read back (interior to pinned memory); time is
    the max over ranks.  On the GPU the problems are pipelined like N=1 --
    upload k+1 | sweeps k | download k-1 over three runners' grids and three
    streams, the halo traffic ordered on the compute stream -- so the
    measurement matches the single-GPU methodology.  The CPU test engine runs
    them one after another."""
    g = runners[0].grid
    cuda = torch.device(dev).type == "cuda"       # CPU only in the gloo test of this function
    host_in = torch.empty(tuple(g.current.shape), dtype=g.torch_dtype, pin_memory=cuda)
    host_in.copy_(g.current.cpu())                 # this rank's current field (untimed)
    host_out = [torch.empty(tuple(g.dims.shape), dtype=g.torch_dtype, pin_memory=cuda) for _ in range(2)]

    if cuda:
        s_up, s_comp, s_down = (torch.cuda.Stream(dev) for _ in range(3))
        cur = torch.cuda.current_stream(dev)
        free = [torch.cuda.Event() for _ in runners]
        for f in free:
            f.record(cur)

        def one(k):
            i = k % len(runners)
            r = runners[i]
            loaded, done = torch.cuda.Event(), torch.cuda.Event()
            s_up.wait_event(free[i])
            r.grid.upload(host_in, stream=s_up.cuda_stream)            # H2D + B = A
            loaded.record(s_up)
            with torch.cuda.stream(s_comp):
                s_comp.wait_event(loaded)
                for t in passes:
                    r.step(levels=t)                                    # NCCL halos on s_comp's order
                r.finish()
                done.record(s_comp)
            s_down.wait_event(done)
            r.grid.download(host_out[k % 2], stream=s_down.cuda_stream)  # D2H
            free[i].record(s_down)
    else:
        def one(k):
            r = runners[k % len(runners)]
            g = r.grid
            g.active = 0
            g.current.copy_(host_in)
            g.other.copy_(g.current)
            r.sync_start()
            for t in passes:
                r.step(levels=t)
            r.finish()
            host_out[k % 2].copy_(g.interior_device())

    def sync():
        if cuda:
            torch.cuda.synchronize(dev)

    for k in range(len(runners)):      # warm-up: every runner once
        one(k)
    sync()
    dist.barrier()
    t0 = time.perf_counter()
    for k in range(steps):
        one(k)
    sync()
    el = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    el = float(el.item())
    lups = global_cells * sum(passes) * steps
    es = host_in.element_size()
    nbytes = torch.tensor([host_in.numel() * es, host_out[0].numel() * es], device=dev, dtype=torch.int64)
    dist.all_reduce(nbytes)                        # every rank's slab, summed
    return {"value": round(lups / el / 1e9, 2), "unit": "GLUP/s",
            "h2d_bytes_per_step": int(nbytes[0]),
            "d2h_bytes_per_step": int(nbytes[1]),
            "steps": steps, "ms_per_step": round(el / steps * 1e3, 2),
            "api": "per rank: TwoGrid.upload(pinned) -> SlabRunner.step() x passes (NCCL halos) "
                   "-> TwoGrid.download(pinned); pipelined over 3 runners and 3 streams; max over ranks"}


def measure_e2e(sp, torch, np, grid, dtype, passes, dev, stream, steps=3):
    """Same metric through the public API with the field on the host.

    Every step uploads the ghosted initial field (dense (nz+2, ny+2, nx+2),
    as the reference's TwoGrid holds it) from pinned memory into a device
    grid (TwoGrid.upload: one pitched DMA + the B = A device copy), runs the
    100 sweeps, and reads the interior back into pinned memory
    (TwoGrid.download, one pitched DMA).  Steps are independent, so they are
    pipelined over three device grids and three streams -- upload k+1 |
    compute k | download k-1 -- and the two PCIe directions run at once.
    """
    d = grid.dims
    host_in = torch.empty(grid.host_shape(), dtype=grid.torch_dtype, pin_memory=True)
    host_in.copy_(grid.current.cpu())            # the initial field (untimed)
    host_out = [torch.empty(d.shape, dtype=grid.torch_dtype, pin_memory=True) for _ in range(2)]
    grids = [grid] + [type(grid)(d, sp.FillPattern.constant(0.0), dtype=dtype, device=dev)
                      for _ in range(2)]
    s_up, s_comp, s_down = (torch.cuda.Stream(dev) for _ in range(3))
    ev = lambda: torch.cuda.Event()                                      # noqa: E731
    free = [ev() for _ in grids]
    sweeps_n = sum(passes)
    T = max(passes)
    for f in free:
        f.record(stream)

    def one(k):
        i = k % len(grids)
        g = grids[i]
        loaded, done = ev(), ev()
        s_up.wait_event(free[i])
        g.upload(host_in, stream=s_up.cuda_stream)                     # H2D
        loaded.record(s_up)
        with torch.cuda.stream(s_comp):
            s_comp.wait_event(loaded)
            sp.sweeps(g, sweeps_n, depth=T)                            # public API
            done.record(s_comp)
        s_down.wait_event(done)
        g.download(host_out[k % 2], stream=s_down.cuda_stream)         # D2H
        free[i].record(s_down)

    one(0)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for k in range(steps):
        one(k)
    torch.cuda.synchronize(dev)
    el = time.perf_counter() - t0
    lups = d.nx * d.ny * d.nz * sweeps_n * steps
    es = host_in.element_size()
    return {"value": round(lups / el / 1e9, 2), "unit": "GLUP/s",
            "h2d_bytes_per_step": host_in.numel() * es, "d2h_bytes_per_step": host_out[0].numel() * es,
            "steps": steps, "ms_per_step": round(el / steps * 1e3, 2),
            "api": "TwoGrid.upload(pinned) -> sweeps() -> TwoGrid.download(pinned); steps "
                   "pipelined on 3 streams over 3 device grids"}


if __name__ == "__main__":
    sys.exit(main())
