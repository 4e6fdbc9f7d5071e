"""ctypes binding of the C ABI in include/bse_b200.h.

The shared library is built in-tree (``python build_ext.py``).  There is no
fallback: if the library or a CUDA device is missing, the solver entry points
raise instead of computing anything on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libbse_b200.so"

BSE_OK = 0
BSE_NOT_POSITIVE_DEFINITE = 1
BSE_NO_CONVERGENCE = 2
BSE_BAD_ARGUMENT = 3
BSE_CUDA_ERROR = 4
BSE_SPECTRUM_NOT_POSITIVE = 5

FLAG_VALUES_ONLY = 0x1
FLAG_NATIVE_FP64 = 0x4


class BseInfo(C.Structure):
    _fields_ = [("pivot_index", C.c_int64), ("pivot_value", C.c_double),
                ("failed_factor", C.c_int32), ("clusters", C.c_int32),
                ("min_pivot", C.c_double)]


# (name, restype, argtypes) -- mirrors include/bse_b200.h one-for-one.
_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double
_INT = C.c_int
SIGNATURES = {
    "bse_version": (_INT, []),
    "bse_last_error": (C.c_char_p, []),
    "bse_solve_workspace_bytes": (C.c_size_t, [_I64, _INT]),
    "bse_solve_spd_pair_dev": (_INT, [_I64, _P, _I64, _P, _I64, _P, _P, _I64, _P, _I64, _P,
                                      C.c_size_t, _INT, _P, C.POINTER(BseInfo)]),
    "bse_solve_spd_pair_host": (_INT, [_I64, _P, _I64, _P, _I64, _P, _P, _I64, _P, _I64, _INT,
                                       C.POINTER(BseInfo)]),
    "bse_solve_complex_workspace_bytes": (C.c_size_t, [_I64, _INT]),
    "bse_solve_complex_dev": (_INT, [_I64, _P, _I64, _P, _I64, _P, _P, _I64, _P, _I64, _P,
                                     C.c_size_t, _INT, _P, C.POINTER(BseInfo)]),
    "bse_solve_complex_host": (_INT, [_I64, _P, _I64, _P, _I64, _P, _P, _I64, _P, _I64, _INT,
                                      C.POINTER(BseInfo)]),
    "bse_potrf_dev": (_INT, [_I64, _P, _I64, _P, C.POINTER(BseInfo)]),
    "bse_syevd_workspace_bytes": (C.c_size_t, [_I64, _INT]),
    "bse_syevd_dev": (_INT, [_I64, _P, _I64, _P, _P, _I64, _P, C.c_size_t, _INT, _P]),
    "bse_stedc_workspace_bytes": (C.c_size_t, [_I64]),
    "bse_stedc_dev": (_INT, [_I64, _P, _P, _P, _I64, _P, C.c_size_t, _P]),
    "bse_absorption_dev": (_INT, [_I64, _P, _P, _I64, _P, _I64, _P, _P, _I64, _P, _D, _P, _P,
                                  _P, _P, _P]),
    "bse_residual_workspace_bytes": (C.c_size_t, [_I64]),
    "bse_pair_residuals_dev": (_INT, [_I64, _P, _I64, _P, _I64, _P, _P, _I64, _P, _I64, _P, _P,
                                      _P, _P, C.c_size_t, _P]),
    "bse_gemm_dev": (_INT, [_INT, _INT, _I64, _I64, _I64, _D, _P, _I64, _P, _I64, _D, _P, _I64,
                            _P, _P]),
    "bse_ozgemm_dev": (_INT, [_INT, _INT, _I64, _I64, _I64, _D, _P, _I64, _P, _I64, _D, _P, _I64,
                              _P, _I64, _P]),
    "bse_oz_set_engine": (_INT, [_INT]),
    "bse_trsm_dev": (_INT, [_INT, _I64, _P, _I64, _P, _I64, _I64, _P]),
    "bse_profile_enable": (_INT, [_INT]),
    "bse_profile_read": (_INT, [_INT, C.POINTER(_D), C.c_char_p]),
    "bse_memcpy2d_staged": (_INT, [_INT, _P, C.c_size_t, _P, C.c_size_t, C.c_size_t,
                                   C.c_size_t, _P]),
    "bse_profile_count": (_INT, []),
    "bse_launch_count": (C.c_longlong, []),
    "bse_release_cached_memory": (_INT, []),
    "bse_peak_fp64": (_INT, [_INT, _INT, _INT, _INT, C.POINTER(_D), C.POINTER(_D)]),
    # column-sharded multi-GPU solve
    "bse_comm_nccl_unique_id": (_INT, [_P]),
    "bse_comm_create_nccl": (_INT, [_INT, _INT, _P, C.POINTER(_P)]),
    "bse_comm_create_host": (_INT, [_INT, _INT, _P, _P, C.POINTER(_P)]),
    "bse_comm_create_solo": (_INT, [_INT, _INT, C.POINTER(_P)]),
    "bse_comm_destroy": (_INT, [_P]),
    "bse_shard_range": (_INT, [_I64, _INT, _INT, C.POINTER(_I64), C.POINTER(_I64)]),
    "bse_comm_allgather_cols_dev": (_INT, [_P, _P, _I64, _I64, _P]),
    "bse_solve_spd_pair_dist_dev": (_INT, [_P, _I64, _P, _I64, _P, _I64, _P, _P, _I64, _P, _I64,
                                           _P, C.c_size_t, _INT, _P, C.POINTER(BseInfo)]),
    # memory-distributed multi-GPU solve (block-cyclic column tiles)
    "bse_bc_local_cols": (_I64, [_I64, _INT, _INT, _INT]),
    "bse_bc_global_col": (_I64, [_I64, _INT, _INT, _INT]),
    "bse_solve_bc_workspace_bytes": (C.c_size_t, [_I64, _INT, _INT, _INT, _INT,
                                                  C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "bse_solve_spd_pair_bc_dev": (_INT, [_P, _I64, _INT, _P, _I64, _P, _I64, _P, _P, _I64, _P,
                                         _I64, _P, C.c_size_t, _INT, _P, C.POINTER(BseInfo)]),
    "bse_comm_allreduce_sum_dev": (_INT, [_P, _P, C.c_size_t, _P]),
}

_lib = None


def load(path: os.PathLike | None = None, strict: bool = False):
    """Load the shared library (cached).  ``strict`` requires every symbol of
    the header to be present."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(f"{p} not built: run `python build_ext.py` (CUDA extension required; "
                          f"there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:
            if strict:
                raise ImportError(f"{p} does not export {name}")
            continue
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def last_error() -> str:
    msg = load().bse_last_error()
    return msg.decode() if msg else ""
