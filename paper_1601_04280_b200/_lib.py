"""ctypes binding of libsrlu.so (include/srlu.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every compute entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os

import torch

from .errors import ParameterError, ShapeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libsrlu.so")

SRLU_OK = 0
SRLU_ERR_ARG = -1
SRLU_ERR_CUDA = -2
SRLU_ERR_UNSUPPORTED = -3
SRLU_ERR_WORKSPACE = -4
SRLU_F32 = 0
SRLU_F64 = 1

P = ctypes.c_void_p
I64 = ctypes.c_int64
U64 = ctypes.c_uint64
INT = ctypes.c_int
DBL = ctypes.c_double
SZ = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/srlu.h
SIGNATURES = {
    "srlu_last_error": (ctypes.c_char_p, []),
    "srlu_version": (INT, []),
    "srlu_seed_key": (INT, [U64, P]),
    "srlu_draw_fast_transform": (INT, [U64, I64, I64, P, P, P]),
    "srlu_draw_sem_workspace": (SZ, [I64, I64]),
    "srlu_build_composite_workspace": (SZ, [I64, I64]),
    "srlu_build_composite_staging": (SZ, [I64, I64]),
    "srlu_build_composite": (INT, [U64, I64, I64, I64, P, P, P, P, P, P, P, P, SZ, P, SZ, P]),
    "srlu_build_composite_k1": (INT, [U64, I64, I64, I64, P, P, P, P, P, P, P, P, SZ, P, SZ,
                                      INT, P, SZ, P]),
    "srlu_composite_sketch_right_dense": (INT, [U64, I64, I64, I64, P, P, P, P, P, P, P, P, SZ,
                                                P, SZ, P, SZ, P, INT, I64, I64, DBL, P, I64, P,
                                                P]),
    "srlu_draw_sem": (INT, [U64, I64, I64, P, P, P, SZ, P]),
    "srlu_sem_plan_workspace": (SZ, [I64, I64]),
    "srlu_sem_plan": (INT, [P, P, I64, I64, P, P, P, SZ, P]),
    "srlu_sketch_right_dense": (INT, [P, INT, I64, I64, I64, P, P, I64, P, P, I64, I64, DBL,
                                      P, I64, P, P]),
    "srlu_k1_schedule_bytes": (SZ, [I64, I64, I64, INT]),
    "srlu_k1_config": (INT, [I64, I64, I64, INT, P]),
    "srlu_k1_schedule": (INT, [P, P, I64, I64, I64, INT, P, SZ, P]),
    "srlu_sketch_right_dense_sched": (INT, [P, INT, I64, I64, I64, P, SZ, I64, P, P, I64, I64,
                                            DBL, P, I64, P, P]),
    "srlu_sketch_right_csr": (INT, [P, P, P, INT, I64, I64, P, P, I64, P, P, I64, I64, DBL,
                                    P, I64, P, P]),
    "srlu_sem_gather_dense": (INT, [P, INT, I64, I64, I64, P, P, I64, P, I64, P]),
    "srlu_fwht_rows": (INT, [P, I64, I64, I64, P]),
    "srlu_sem_members": (INT, [P, I64, P, I64, I64, P, P, P]),
    "srlu_sketch_left_workspace": (SZ, [I64, I64, I64]),
    "srlu_sketch_left_dense": (INT, [P, INT, I64, I64, I64, P, P, P, I64, P, P, I64, I64, DBL,
                                     P, I64, P, SZ, P]),
    "srlu_sem_scatter_dense": (INT, [P, INT, I64, I64, I64, P, P, P, I64, P, I64, P]),
    "srlu_sem_gather_csr": (INT, [P, P, P, INT, I64, P, P, P, I64, P]),
    "srlu_sem_scatter_csc": (INT, [P, P, P, INT, I64, P, P, P, I64, P]),
    "srlu_sketch_left_csr_workspace": (SZ, [I64, I64, I64, I64, I64]),
    "srlu_sketch_left_csr": (INT, [P, P, P, INT, I64, I64, I64, P, P, P, I64, P, P, I64, I64,
                                   DBL, P, I64, P, SZ, P, P]),
    "srlu_qr_pinv_smem_bytes": (SZ, [I64, I64]),
    "srlu_qr_pinv_workspace": (SZ, [I64, I64]),
    "srlu_qr_pinv": (INT, [P, I64, I64, I64, P, I64, P, P, SZ, P]),
    "srlu_rank_estimate": (INT, [P, I64, I64, P, I64, P, P]),
    "srlu_qr_rank": (INT, [P, I64, I64, P, P]),
    "srlu_qr_rank_certified": (INT, [P, I64, I64, P, I64, P, P]),
    "srlu_rank_exact_workspace": (SZ, [I64]),
    "srlu_rank_exact": (INT, [P, I64, I64, P, SZ, P, P]),
    "srlu_dgemm": (INT, [P, I64, P, I64, P, I64, I64, I64, I64, P]),
    "srlu_dgemm_ex": (INT, [P, I64, P, I64, P, I64, I64, I64, I64, INT, P]),
    "srlu_lu_error_workspace": (SZ, [I64, I64, I64]),
    "srlu_lu_error_dense": (INT, [P, I64, P, I64, P, P, P, INT, I64, I64, I64, I64, P, P, SZ,
                                  P]),
    "srlu_lu_error_csr": (INT, [P, I64, P, I64, P, P, P, P, P, INT, I64, I64, I64, P, P, SZ,
                                P]),
    "srlu_lu_workspace": (SZ, [I64, I64]),
    "srlu_lu_rowpiv": (INT, [P, I64, I64, I64, P, P, I64, P, I64, INT, P, SZ, P]),
    "srlu_lu_colpiv": (INT, [P, I64, I64, I64, P, P, I64, P, I64, INT, P, SZ, P]),
}

_lib = None


def load(required_symbols: bool = True):
    """Load libsrlu.so (no device needed).  Raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libsrlu.so not found at {LIB_PATH}: build it with "
            "`python -m paper_1601_04280_b200.build` (nvcc, sm_100a). "
            "There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:
            if required_symbols:
                raise RuntimeError(f"libsrlu.so lacks symbol {name}")
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_cuda_checked = False


def lib():
    """The loaded library; raises without a CUDA device (no CPU fallback).
    The device check runs once: this is on the host-bound start of every
    decomposition."""
    global _cuda_checked
    L = _lib if _lib is not None else load()
    if not _cuda_checked:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1601_04280_b200 needs a CUDA device (B200, sm_100a); "
                               "there is no CPU fallback")
        _cuda_checked = True
    return L


class _LaunchCounter:
    """Number of libsrlu kernels enqueued (bench.py's ``gpu_launches``)."""

    PER_CALL = {"build_sem": 3, "sem_plan": 4, "build_composite": 7, "build_composite_k1": 8, "build_composite_k1_g": 9, "composite_sketch_right_dense": 9, "composite_sketch_right_dense_g": 10, "composite_sketch_right_dense_nosched": 8, "sketch_right_dense": 1, "sketch_right_csr": 1,
                "k1_schedule": 2, "k1_schedule_1": 1, "sketch_right_dense_sched": 1,
                "sem_gather_dense": 1, "sem_gather_csr": 1, "sem_scatter_csc": 1, "fwht_rows": 1, "sem_members": 1,
                "sketch_left_dense": 2, "sem_scatter_dense": 1, "sketch_left_csr": 6, "sketch_left_csr_big": 9,
                "lu_row_pivot": 1, "lu_col_pivot": 1, "qr_pinv": 2, "rank_estimate": 1, "qr_rank": 1, "rank_exact": 1,
                "dgemm": 1, "lu_error": 3}

    def __init__(self):
        self.total = 0

    def reset(self):
        self.total = 0


LAUNCHES = _LaunchCounter()


def check(rc: int, what: str = ""):
    if rc == SRLU_OK:
        LAUNCHES.total += _LaunchCounter.PER_CALL.get(what, 0)
        return
    msg = (load().srlu_last_error() or b"").decode(errors="replace")
    if rc == SRLU_ERR_ARG:
        if "need rows" in msg or "shape" in msg:
            raise ShapeError(msg)
        raise ParameterError(msg)
    if rc == SRLU_ERR_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: libsrlu error {rc}: {msg}")


def ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def stream_handle(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return SRLU_F32
    if dt == torch.float64:
        return SRLU_F64
    raise ParameterError(f"unsupported element dtype {dt}; need float32 or float64")
