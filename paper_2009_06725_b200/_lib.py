"""ctypes binding of libss_b200.so (the C ABI declared in include/spectralstokes_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is present, every compute
entry point raises.  Error codes map onto the reference's exception types (errors.py).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .errors import DeviceError, MeshError

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libss_b200.so"
# A/B tooling only (tools/build_variant.py): load a differently built copy of the same library.
if os.environ.get("SS_B200_LIB"):
    LIB_PATH = Path(os.environ["SS_B200_LIB"]).resolve()

P = C.c_void_p
I32 = C.c_int
I64 = C.c_int64
D = C.c_double
PD = C.POINTER(C.c_double)
PI64 = C.POINTER(C.c_int64)
PI32 = C.POINTER(C.c_int32)
PU8 = C.POINTER(C.c_uint8)
PF = C.POINTER(C.c_float)

# name -> (restype, argtypes)
SIGNATURES = {
    "ss_last_error": (C.c_char_p, []),
    "ss_version": (I32, []),
    "ss_launch_count": (I64, []),
    "ss_reference_tables": (I32, [I32, PD, PD, PD]),
    "ss_pattern_create": (I32, [I32, I64, I64, I64, PI64, PU8, I32, I32, C.POINTER(P)]),
    "ss_pattern_destroy": (None, [P]),
    "ss_pattern_info": (I32, [P, PI64]),
    "ss_pattern_export": (I32, [P, PI32, PI32]),
    "ss_pattern_dof_maps": (I32, [P, PI64, PI64]),
    "ss_constrained_rows": (I32, [P, D, PI64, PI64, PI32, PD]),
    "ss_pattern_export_rows": (I32, [P, I64, PI64, PI64, PI32, I64]),
    "ss_assemble": (I32, [P, PD, D, D, P]),
    "ss_export_values": (I32, [P, D, P, P]),
    "ss_surface_load": (I32, [I32, I64, PD, I64, PI64, I32, PD, PD]),
    "ss_rhs_batched": (I32, [P, I32, P, P, P, P, I64, P]),
    "ss_spmv_batched": (I32, [P, I32, P, P, P, I64, I32, P]),
    "ss_spmv_batched_interleaved": (I32, [P, I32, P, P, P, I64, I32, P]),
    "ss_spmv_bytes": (I64, [P, I32]),
    "ss_jacobi": (I32, [P, I32, P, P, I64, P]),
    "ss_residual_norms": (I32, [P, I32, P, P, P, I64, PD, P]),
    "ss_expand": (I32, [P, I32, P, I64, P, P, P, P]),
    "ss_l2_norms": (I32, [P, I32, I32, P, PD, P]),
    "ss_quadrature_points": (I32, [I32, C.POINTER(C.c_int)]),
    "ss_write_snapshot": (I32, [C.c_char_p, I32, I64, I64, PD, PD, PD, D]),
    "ss_write_vtk": (I32, [C.c_char_p, C.c_char_p, I32, I64, I64, PD, I64, I32, PI64, PI64, PD, PD]),
    "ss_read_snapshot": (I32, [C.c_char_p, I32, I64, I64, PD, PD, PD]),
    "ss_interp_quadrature": (I32, [P, I32, P, P, P, P, P]),
    "ss_krylov_create_saddle": (I32, [P, I32, I32, I64, C.POINTER(P)]),
    "ss_krylov_create_csr": (I32, [I32, I32, I64, PI32, PI32, I32, PD, PD, I32, I32, I32, I64, C.POINTER(P)]),
    "ss_krylov_destroy": (None, [P]),
    "ss_krylov_info": (I32, [P, PI64]),
    "ss_krylov_set_option": (I32, [P, C.c_char_p, I64]),
    "ss_krylov_get_option": (I32, [P, C.c_char_p, PI64]),
    "ss_krylov_buffers": (I32, [P, C.POINTER(P), C.POINTER(P), PI64]),
    "ss_krylov_solve": (I32, [P, I32, PD, C.POINTER(I32), P, P, I64, I32, D, I64, I32, P, PI64, PD]),
    "ss_krylov_history": (I32, [P, I32, I64, PD]),
    "ss_krylov_last_stats": (I32, [P, PI64, PI64]),
    "ss_krylov_done_ticks": (I32, [P, I32, PI64]),
    "ss_krylov_residuals": (I32, [P, I32, P, PD]),
    "ss_krylov_copy": (I32, [P, I32, I32, P, I64, P]),
    "ss_krylov_csr_scale": (I32, [P, I32, PD]),
    "ss_krylov_profile": (I32, [P, I32, PD, D, I64, I32, P, PD, PI64, PI64]),
    "ss_krylov_bench_pass": (I32, [P, I32, I32, I32, I32, P, PF, PI64]),
    "ss_reconstruct": (I32, [I32, I32, I64, P, P, P, P]),
    "ss_comm_nccl_version": (I32, []),
    "ss_comm_unique_id": (I32, [PU8]),
    "ss_comm_create": (I32, [I32, I32, PU8, I32, C.POINTER(P)]),
    "ss_comm_destroy": (None, [P]),
    "ss_comm_gather_modes": (I32, [P, P, I64, I64, I64, P, PI64, PI64, I32, P]),
    "ss_comm_allreduce_max": (I32, [P, P, I64, P]),
    "ss_comm_reduce_sum": (I32, [P, P, I64, I32, P]),
}

_lib = None

# Must equal SS_ABI_VERSION in include/spectralstokes_b200.h (bumped whenever an entry point changes).
ABI_VERSION = 5


def load(build_if_missing: bool = True):
    """Load (building in-tree first if needed) the native library."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists() or os.environ.get("SS_B200_REBUILD"):
        if not build_if_missing:
            raise DeviceError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
        from .build import build
        build()
    lib = C.CDLL(str(LIB_PATH))
    lib.ss_version.restype = I32
    if lib.ss_version() != ABI_VERSION:
        # a stale in-tree build (the .so is git-ignored): rebuild once, then refuse
        if not build_if_missing or os.environ.get("SS_B200_LIB"):
            raise DeviceError(f"{LIB_PATH} has ABI {lib.ss_version()}, expected {ABI_VERSION}: rebuild it")
        from .build import build
        build(force=True)
        return _load_fresh()
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _load_fresh():
    """Load a freshly rebuilt library under a new file name (the stale one stays mapped)."""
    global _lib
    import shutil
    import tempfile

    tmp = Path(tempfile.mkdtemp(prefix="ss_b200_")) / LIB_PATH.name
    shutil.copy2(LIB_PATH, tmp)
    lib = C.CDLL(str(tmp))
    lib.ss_version.restype = I32
    if lib.ss_version() != ABI_VERSION:
        raise DeviceError(f"rebuilt {LIB_PATH} still reports ABI {lib.ss_version()}, expected {ABI_VERSION}")
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int):
    if rc == 0:
        return
    msg = (load().ss_last_error() or b"").decode(errors="replace")
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise MeshError(msg)
    if rc == 3:
        raise DeviceError(msg)
    raise RuntimeError(msg)


def call(name, *args):
    check(getattr(load(), name)(*args))


def ptr(arr: np.ndarray, ctype=C.c_double):
    return arr.ctypes.data_as(C.POINTER(ctype))


def launch_count() -> int:
    return int(load().ss_launch_count())


# --- torch plumbing (device memory + streams only) ----------------------------------------------

def torch_mod():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the spectral-Stokes hot path runs only on the GPU (no CPU fallback)")
    return torch


def stream_ptr(device=None):
    torch = torch_mod()
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def dptr(t):
    return C.c_void_p(t.data_ptr())
