"""ctypes binding of libstencilpipe_b200.so (include/stencilpipe_b200.h).

The library is built in-tree (``build()`` / ``__graft_entry__.build()``) and
loaded from this package directory.  There is no CPU fallback: if the library
is missing or no CUDA device is visible, calls raise ``NativeUnavailable``.
Error codes map to the reference's exception types:
GridError, ScheduleError, DecompositionError (all ValueError) and
RuntimeError for device failures.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
LIB_NAME = "libstencilpipe_b200.so"
LIB_PATH = os.environ.get("SP_LIB_PATH") or os.path.join(_HERE, LIB_NAME)
SOURCES = [os.path.join(_HERE, "csrc", f) for f in ("capi.cu", "jacobi_kernels.cuh", "host.cuh", "tb_inst.cu", "tq.cuh",
                                                     "wave2.cuh", "dist_nccl.cu")]
HEADER = os.path.join(_ROOT, "include", "stencilpipe_b200.h")

SP_OK, SP_ERR_GRID, SP_ERR_SCHEDULE, SP_ERR_DECOMP, SP_ERR_DEVICE, SP_ERR_ARG = range(6)
SP_F64, SP_F32 = 0, 1

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--shared", "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]

# Symbols include/stencilpipe_b200.h declares (checked by the CPU tests).
EXPORTS = ("sp_version", "sp_last_error", "sp_launch_count", "sp_layout_make", "sp_fill",
           "sp_update_region", "sp_sweep_tb", "sp_sweep_tb_part", "sp_sweep_tb_part_peer", "sp_run_sweeps",
           "sp_digest", "sp_probe_fp64", "sp_set_tuning", "sp_set_schedule", "sp_ipc_export",
           "sp_ipc_import", "sp_ipc_close", "sp_copy_in", "sp_copy_out", "sp_describe_variant",
           "sp_sweep_tb_inplace", "sp_ghost_shell", "sp_ghost_shell_elems", "sp_ghost_shell_region", "sp_copy_box",
           "sp_dist_unique_id", "sp_dist_create", "sp_dist_destroy", "sp_dist_exchange_z", "sp_dist_step")


class NativeUnavailable(RuntimeError):
    """The CUDA library is not built or no B200 is visible."""


class Layout(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("nx", "ny", "nz", "gx", "gy", "gz", "py", "pz", "origin")]

    def as_tuple(self):
        return tuple(getattr(self, f) for f, _ in self._fields_)


class Pattern(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("has_faces", ctypes.c_int32),
                ("value", ctypes.c_double), ("seed", ctypes.c_uint64),
                ("gorigin", ctypes.c_int64 * 3), ("gn", ctypes.c_int64 * 3),
                ("faces", ctypes.c_double * 6)]


def build(verbose: bool = False, force: bool = False, out: str | None = None,
          defines=()) -> str:
    """Compile the sm_100a library in-tree with nvcc; returns its path."""
    target = out or LIB_PATH
    newest = max(os.path.getmtime(p) for p in SOURCES + [HEADER])
    if not force and not defines and os.path.exists(target) and os.path.getmtime(target) >= newest:
        return target
    nvcc = os.environ.get("NVCC", "nvcc")
    if not any(os.access(os.path.join(p, "nvcc"), os.X_OK)
               for p in os.environ.get("PATH", "").split(os.pathsep)):
        if os.path.exists("/usr/local/cuda/bin/nvcc"):
            nvcc = "/usr/local/cuda/bin/nvcc"
    tmp = target + ".tmp"
    objdir = os.path.join(os.path.dirname(target), "build", "obj" + ("_" + os.path.basename(target) if out else ""))
    os.makedirs(objdir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    cflags = [f for f in NVCC_FLAGS if f != "--shared"]
    # one unit for the C ABI + small kernels, one per (dtype, T) for the K2
    # instantiations (host.cuh / tb_inst.cu): compiled in parallel
    jobs = [("capi", [os.path.join(_HERE, "csrc", "capi.cu")]),
            ("dist_nccl", [os.path.join(_HERE, "csrc", "dist_nccl.cu")])]
    for r in ("double", "float"):
        for t in range(1, 9):
            jobs.append((f"tb_{r}_{t}", [f"-DSP_INST_R={r}", f"-DSP_INST_T={t}",
                                         os.path.join(_HERE, "csrc", "tb_inst.cu")]))

    def compile_one(job):
        name, args = job
        obj = os.path.join(objdir, name + ".o")
        r = subprocess.run([nvcc, *cflags, *dflags, "-c", "-o", obj, *args], capture_output=True, text=True)
        return obj, r

    from concurrent.futures import ThreadPoolExecutor
    workers = max(1, min(len(jobs), (os.cpu_count() or 4)))
    # the heaviest units first (deep fp64 / fp32 instantiations)
    order = sorted(jobs, key=lambda j: (not j[0].startswith("tb_"), -int(j[0][-1]) if j[0].startswith("tb_") else 0))
    with ThreadPoolExecutor(workers) as ex:
        results = list(ex.map(compile_one, order))
    log = []
    for (obj, r), (name, _) in zip(results, order):
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed ({name}):\n{r.stderr}")
        log.append(f"== {name}\n{r.stderr}")
    res = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "--shared", "-Xcompiler",
                          "-fPIC", "-o", tmp, *[o for o, _ in results]],
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stderr}")
    if verbose:
        sys.stderr.write("".join(log))
    os.replace(tmp, target)
    with open(target + ".ptxas.log" if out else os.path.join(_HERE, "csrc", "ptxas.log"), "w") as fh:
        fh.write("\n".join(log))
    return target


_lib = None


def load_library():
    """Load (not initialise CUDA) -- usable on CPU-only hosts for symbol checks."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(f"{LIB_PATH} is not built; run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    override = bool(os.environ.get("SP_LIB_PATH"))
    P = ctypes.POINTER
    vp = ctypes.c_void_p
    i64p = P(ctypes.c_int64)
    i32p = P(ctypes.c_int32)
    L.sp_version.restype = ctypes.c_int
    L.sp_last_error.restype = ctypes.c_char_p
    L.sp_launch_count.restype = ctypes.c_uint64
    L.sp_layout_make.argtypes = [ctypes.c_int64] * 6 + [ctypes.c_int, P(Layout), i64p]
    L.sp_fill.argtypes = [vp, ctypes.c_int, P(Layout), P(Pattern), vp]
    L.sp_update_region.argtypes = [vp, vp, ctypes.c_int, P(Layout), i64p, i64p, vp]
    L.sp_sweep_tb.argtypes = [vp, vp, ctypes.c_int, P(Layout), ctypes.c_int, i64p, i64p,
                              i32p, i32p, vp]
    L.sp_sweep_tb_part.argtypes = [vp, vp, ctypes.c_int, P(Layout), ctypes.c_int, i64p, i64p,
                                   i32p, i32p, i64p, i64p, vp]
    if hasattr(L, "sp_sweep_tb_part_peer") or not override:
        L.sp_sweep_tb_part_peer.argtypes = [vp, vp, ctypes.c_int, P(Layout), ctypes.c_int, i64p, i64p,
                                            i32p, i32p, i64p, i64p, vp, ctypes.c_int64, vp,
                                            ctypes.c_int64, ctypes.c_int64, vp]
    if hasattr(L, "sp_copy_in") or not override:
        L.sp_copy_in.argtypes = [vp, ctypes.c_int, P(Layout), vp, vp, vp, ctypes.c_int64, vp]
        L.sp_copy_out.argtypes = [vp, ctypes.c_int, P(Layout), vp, vp, ctypes.c_int64, vp]
    if hasattr(L, "sp_ipc_export") or not override:
        L.sp_ipc_export.argtypes = [vp, P(ctypes.c_ubyte * 64), P(ctypes.c_int64)]
        L.sp_ipc_import.argtypes = [P(ctypes.c_ubyte * 64), ctypes.c_int64, P(vp)]
        L.sp_ipc_close.argtypes = [vp, ctypes.c_int64]
    L.sp_run_sweeps.argtypes = [vp, vp, ctypes.c_int, P(Layout), ctypes.c_int64, ctypes.c_int,
                                P(ctypes.c_int), vp]
    L.sp_digest.argtypes = [vp, ctypes.c_int, P(Layout), ctypes.c_int64, P(ctypes.c_uint64), vp]
    L.sp_probe_fp64.argtypes = [P(ctypes.c_double), P(ctypes.c_double)]
    L.sp_set_tuning.argtypes = [ctypes.c_int, ctypes.c_int]
    if hasattr(L, "sp_sweep_tb_inplace") or not override:
        L.sp_sweep_tb_inplace.argtypes = [vp, ctypes.c_int, P(Layout), ctypes.c_int, i64p, i64p,
                                          ctypes.c_int64, ctypes.c_int, vp, ctypes.c_int64, vp]
        L.sp_ghost_shell.argtypes = [vp, ctypes.c_int, P(Layout), vp, ctypes.c_int, vp]
        L.sp_ghost_shell_region.argtypes = [vp, ctypes.c_int, P(Layout), vp, i64p, i64p, vp]
        L.sp_copy_box.argtypes = [vp, vp, ctypes.c_int] + [ctypes.c_int64] * 7 + [vp]
        L.sp_ghost_shell_elems.restype = ctypes.c_int64
        L.sp_ghost_shell_elems.argtypes = [ctypes.c_int64] * 3
    if hasattr(L, "sp_dist_create") or not override:
        L.sp_dist_unique_id.argtypes = [vp, ctypes.c_int64]
        L.sp_dist_create.argtypes = [vp, ctypes.c_int, ctypes.c_int, P(vp)]
        L.sp_dist_destroy.argtypes = [vp]
        L.sp_dist_exchange_z.argtypes = [vp, vp, ctypes.c_int, P(Layout), ctypes.c_int64, vp]
        L.sp_dist_step.argtypes = [vp, vp, vp, ctypes.c_int, P(Layout), ctypes.c_int, vp]
    if hasattr(L, "sp_describe_variant") or not override:
        L.sp_describe_variant.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_int]
    for name in EXPORTS:
        if override and not hasattr(L, name):
            continue   # older library under A/B comparison: tuning hooks may be absent
        getattr(L, name).restype = getattr(L, name).restype or ctypes.c_int
    if hasattr(L, "sp_set_schedule") or not override:
        L.sp_set_schedule.argtypes = [ctypes.c_int, ctypes.c_int]
    _lib = L
    return L


def lib():
    """The library, after checking a CUDA device is present (no fallback)."""
    L = load_library()
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible: the Jacobi engine has no CPU path")
    return L


def check(rc: int) -> None:
    if rc == SP_OK:
        return
    msg = (load_library().sp_last_error() or b"").decode()
    from .grid import GridError
    from .pipeline import ScheduleError
    from .decomp import DecompositionError
    exc = {SP_ERR_GRID: GridError, SP_ERR_SCHEDULE: ScheduleError,
           SP_ERR_DECOMP: DecompositionError, SP_ERR_ARG: ValueError}.get(rc, RuntimeError)
    raise exc(msg)


def i64x3(v):
    return (ctypes.c_int64 * 3)(*[int(x) for x in v])


def i32x3(v):
    return (ctypes.c_int32 * 3)(*[int(x) for x in v])


def launch_count() -> int:
    return int(load_library().sp_launch_count())


def describe_variant(sp_dtype: int, T: int) -> str:
    """One-line description of the K2 variant a depth-T pass runs (sp_describe_variant)."""
    buf = ctypes.create_string_buffer(256)
    v = load_library().sp_describe_variant(sp_dtype, T, buf, len(buf))   # host-only: no device needed
    if v < 0:
        check(-v)
    return buf.value.decode()
