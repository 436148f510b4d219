#!/usr/bin/env python
"""Benchmark: temporally blocked 3D Jacobi on B200 (BASELINE.json metric GLUP/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c3|c2|c4|c5w] [--depth T]

One "step" = one full BASELINE run of the workload (C3: 100 sweeps of the
1024^3 fp64 grid) over inputs already resident in HBM.  N=1 runs C3 on one
GPU; under torchrun (N>1) every rank owns a 1024^3 z-slab of a
1024 x 1024 x (1024 N) global grid (weak scaling), exchanging depth-T halos over
NCCL with the exchange overlapped with interior compute (dist.SlabRunner).

Rank 0 prints ONE JSON line.  Besides the driver's keys it carries:
  roofline          the dominant kernel (K2) against measured HBM bandwidth
                    (algorithmic bytes 16 B/cell per pass / CUDA-event pass time)
  temporal_roofline GLUP/s against R(T) = min(P_fp64/6, B_hbm*T/16) with the
                    FP64 add rate measured on this GPU at run time
  cpu_baseline      the C oracle (a port of the reference's sweep) on this
                    host's cores, bounded sample (rank 0, N=1 only)
  e2e               the same metric through the public API with the grid
                    uploaded from pinned host memory and the interior read
                    back every step
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

WORKLOADS = {
    # name: (shape (nz, ny, nx) per GPU, kind, faces, dtype, sweeps, description)
    "c3": ((1024, 1024, 1024), "random", (1.0, 0.0, 0.5, 0.0, 0.25, 0.0), "f64", 100,
           "C3: fp64 interior 1024^3, Dirichlet faces (z-,z+,y-,y+,x-,x+)=(1,0,0.5,0,0.25,0), "
           "random(0) interior, 100 sweeps"),
    "c2": ((512, 512, 512), "random", (1.0, 0.0, 0.0, 0.0, 0.0, 0.0), "f64", 200,
           "C2: fp64 interior 512^3, face z-=1, random(0), 200 sweeps"),
    "c4": ((2048, 1024, 1024), "random_pm1", (0.0,) * 6, "f32", 200,
           "C4: fp32 interior 1024x1024x2048, uniform[-1,1) from random(0), zero faces, 200 sweeps"),
    "c5w": ((512, 1024, 1024), "random", (1.0, 0.0, 0.0, 0.0, 0.0, 0.0), "f64", 100,
            "C5 weak: fp64 1024x1024x512 per GPU, face z-=1, random(0), 100 sweeps"),
}


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


def run_reference_arm(args, rank):
    if rank != 0:
        return 0
    shape, kind, faces, dt, sweeps, desc = WORKLOADS[args.workload]
    import numpy as np
    from oracle import oracle as O
    O.build_c()
    nz, ny, nx = shape
    planes = 32
    g = O.CGrid((planes, ny, nx), O.BoxPattern(kind, seed=0, faces=faces, global_shape=shape),
                dtype=np.float64 if dt == "f64" else np.float32)
    per_step = 2   # sweeps of the slab per step (bounded sample)
    for _ in range(args.warmup):
        g.sweeps(per_step)
    t0 = time.monotonic()
    for _ in range(args.steps):
        g.sweeps(per_step)
    el = time.monotonic() - t0
    lups = nx * ny * planes * per_step * args.steps
    v = lups / el / 1e9
    cores = O.num_threads()
    sample = (f"{nx}x{ny}x{planes} z-slab of {args.workload} ({per_step} sweeps per step), "
              f"oracle C port of sweep_naive (R/kernel.py:43-47) on {cores} threads")
    line = {
        "metric": "GLUP/s", "value": round(v, 3), "unit": "GLUP/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": dt, "data": "synthetic",
        "config": {"workload": desc, "sample": sample},
        "cpu_baseline": {"value": round(v, 3), "unit": "GLUP/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(v, 3), "unit": "GLUP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--depth", type=int, default=0, help="levels per HBM pass (0 = tuned default)")
    ap.add_argument("--variant", type=int, default=0, help="kernel variant override (dev)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg")
    ap.add_argument("--storage", choices=("twogrid", "compressed"), default="twogrid",
                    help="A/B grids or single-array in-place storage (N=1)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--transport", choices=("p2p", "nccl"), default="p2p",
                    help="N>1 halo exchange: p2p = boundary kernels store into the neighbours' "
                         "grids (CUDA IPC, NVLink), nccl = NCCL send/recv of the planes")
    ap.add_argument("--slab-runner", action="store_true",
                    help="dev: use the multi-GPU SlabRunner path even at N=1 (run under torchrun)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference_arm(args, rank)

    import numpy as np
    import torch
    import paper_0912_4506_b200 as sp
    from paper_0912_4506_b200 import _native as N
    from paper_0912_4506_b200.pipeline import DEFAULT_DEPTH

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    use_runner = world > 1 or args.slab_runner
    if use_runner and args.storage != "twogrid":
        raise SystemExit("--storage compressed has no multi-GPU (slab runner) form")
    if use_runner:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    shape, kind, faces, dt, sweeps, desc = WORKLOADS[args.workload]
    dtype = np.float64 if dt == "f64" else np.float32
    es = 8 if dt == "f64" else 4
    lib = N.lib()
    if args.variant:
        lib.sp_set_tuning(args.variant, 0)
    sp_dtype = N.SP_F64 if dt == "f64" else N.SP_F32
    T = args.depth or DEFAULT_DEPTH[sp_dtype]
    nz, ny, nx = shape
    gshape = (nz * world, ny, nx)
    cells_rank = nz * ny * nx
    passes = [T] * (sweeps // T) + ([sweeps % T] if sweeps % T else [])

    # --- FP64 compute roof, measured on this GPU ---
    import ctypes
    rate, ms = ctypes.c_double(), ctypes.c_double()
    N.check(lib.sp_probe_fp64(ctypes.byref(rate), ctypes.byref(ms)))
    p_fp64 = rate.value

    pat = sp.FillPattern.dirichlet_box(kind, gshape, faces, seed=0)
    stream = torch.cuda.current_stream(dev)
    pass_events = []

    if not use_runner:
        Grid = sp.CompressedGrid if args.storage == "compressed" else sp.TwoGrid
        grid = Grid(sp.GridDims(nx, ny, nz), pat, dtype=dtype, device=dev)

        def step(record=False):
            for t in passes:
                if record:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                sp.sweeps(grid, t, depth=t)
                if record:
                    e1.record(stream)
                    pass_events.append((t, e0, e1))
    else:
        from paper_0912_4506_b200.dist import SlabRunner
        transport = args.transport if world > 1 else "nccl"
        try:
            runner = SlabRunner(sp.GridDims(nx, ny, nz * world), pat, h=T, dtype=dtype, device=dev,
                                depth=T, transport=transport)
        except Exception as exc:          # p2p mapping refused (no peer access): NCCL planes
            if transport != "p2p":
                raise
            transport = f"nccl (p2p setup failed: {type(exc).__name__}: {exc})"[:200]
            runner = SlabRunner(sp.GridDims(nx, ny, nz * world), pat, h=T, dtype=dtype, device=dev,
                                depth=T, transport="nccl")
        grid = runner.grid

        def step(record=False):
            for t in passes:
                if record:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                runner.step(levels=t)
                if record:
                    e1.record(stream)
                    pass_events.append((t, e0, e1))
            runner.finish()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    barrier()

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    n0 = N.launch_count()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for k in range(args.steps):
        step(record=True)
    ev1.record(stream)
    barrier()
    launches = N.launch_count() - n0
    clocks = sampler.stop() if sampler else None
    elapsed = ev0.elapsed_time(ev1) / 1e3
    if dist is not None:
        t = torch.tensor([elapsed], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    total_lups = cells_rank * world * sweeps * args.steps
    value = total_lups / elapsed / 1e9

    # dominant kernel: full-depth passes (K2 at depth T)
    full = [e0.elapsed_time(e1) / 1e3 for t, e0, e1 in pass_events if t == T]
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
                        "source": tj[key].get("source")}

    R_hbm = hbm * T / (2 * es)                      # GLUP/s, HBM term
    R_fp = p_fp64 / 6 / 1e9 if dt == "f64" else float("inf")
    R = min(R_hbm, R_fp) * world

    # --- e2e: the public API with host buffers ---
    e2e = None
    if not args.no_e2e:
        if not use_runner:
            # a stream of independent problems: >= 24 steps so the pipeline's fill
            # (first upload) and drain (last download) are a small share
            e2e = measure_e2e(sp, torch, np, grid, dtype, passes, dev, stream, steps=max(args.steps, 24))
        else:
            e2e = measure_e2e_dist(torch, dist, runner, passes, dev, world, steps=max(args.steps, 3))

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
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": dt,
            "data": "synthetic (seeded coordinate hash random(0), Dirichlet faces; no dataset)",
            "config": {"workload": desc, "T": T, "passes_per_step": len(passes),
                       "global_interior_zyx": list(gshape), "per_gpu_interior_zyx": list(shape),
                       "parallelism": f"zslab{world}", "variant": args.variant or "auto",
                       "kernel": N.describe_variant(sp_dtype, T) if args.storage == "twogrid"
                       else "in-place variant (compressed storage, sp_sweep_tb_inplace)",
                       "storage": args.storage,
                       "halo_transport": transport if use_runner else None,
                       "l2": "inputs larger than L2 (one grid = %.1f GB >> 126 MB)" % (
                           grid.buffers[0].numel() * es / 1e9),
                       "hbm_grid_bytes": sum(b.numel() * b.element_size() for b in grid.buffers)},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(achieved / hbm, 4), "traffic": traffic,
                         "kernel": f"tb_kernel T={T}", "peak_source": hbm_src,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "avg_launch_ms": round(t_pass * 1e3, 3), "ncu": ncu_evidence},
            "temporal_roofline": {"T": T, "R_glups": round(R, 1), "frac": round(value / R, 4),
                                  "R_hbm_glups": round(R_hbm * world, 1),
                                  "R_fp64_glups": round(R_fp * world, 1) if R_fp != float("inf") else None,
                                  "fp64_dadd_per_s": p_fp64, "hbm_gbs": hbm},
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "impl": "ours",
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        if use_runner:
            runner.close()
        dist.barrier()
        dist.destroy_process_group()
    return 0


def measure_e2e_dist(torch, dist, runner, passes, dev, world, steps=3):
    """e2e at N GPUs: every rank uploads its ghosted z-slab from pinned host
    memory, runs the sweeps through SlabRunner (NCCL halos), and reads its
    interior back; time is the max over ranks (barrier on both sides)."""
    g = runner.grid
    cuda = torch.device(dev).type == "cuda"       # CPU only in the gloo test of this function
    host_in = torch.empty(tuple(g.current.shape), dtype=g.torch_dtype, pin_memory=cuda)
    host_in.copy_(g.current.cpu())                 # this rank's current field (untimed)
    host_out = torch.empty(tuple(g.dims.shape), dtype=g.torch_dtype, pin_memory=cuda)
    upload = getattr(g, "upload", None)

    def sync():
        if cuda:
            torch.cuda.synchronize(dev)

    def one():
        if upload is not None:
            g.upload(host_in)                                # H2D + B = A (TwoGrid.upload)
        else:                                                # host test engine
            g.active = 0
            g.current.copy_(host_in)
            g.other.copy_(g.current)
        runner.sync_start()     # every rank's upload lands before a neighbour stores into it
        for t in passes:
            runner.step(levels=t)
        runner.finish()
        if upload is not None:
            g.download(host_out)                             # D2H (TwoGrid.download)
        else:
            host_out.copy_(g.interior_device())

    one()
    sync()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    sync()
    el = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    el = float(el.item())
    d = g.dims
    lups = d.nx * d.ny * d.nz * sum(passes) * steps * world
    es = host_in.element_size()
    return {"value": round(lups / el / 1e9, 2), "unit": "GLUP/s",
            "h2d_bytes_per_step": host_in.numel() * es * world,
            "d2h_bytes_per_step": host_out.numel() * es * world,
            "steps": steps, "ms_per_step": round(el / steps * 1e3, 2),
            "api": "per rank: slab.current.copy_(pinned) -> SlabRunner.step() x passes (NCCL halos) "
                   "-> interior_device() -> pinned; max over ranks"}


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
