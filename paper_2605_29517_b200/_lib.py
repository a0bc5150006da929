"""ctypes binding of libmaxsim_b200.so (include/maxsim_b200.h).

The library is the only compute path: if it is missing or fails to load, every operator
raises.  There is no CPU or PyTorch fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors
from ._build import LIB_PATH

_lock = threading.Lock()
_lib = None

c_int = ctypes.c_int
c_i64 = ctypes.c_int64
c_vp = ctypes.c_void_p
c_dbl = ctypes.c_double
c_size = ctypes.c_size_t

# name -> argtypes (restype is int unless listed in _RESTYPES)
_SIGNATURES = {
    "mxs_version": [],
    "mxs_status_string": [c_int],
    "mxs_last_error": [],
    "mxs_device_sm_count": [],
    "mxs_fused_score_batch": [c_int, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_int, c_vp],
    "mxs_fused_rowmax_batch": [c_int, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_int, c_vp],
    "mxs_fused_score_int8": [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp],
    "mxs_rowsum": [c_vp, c_i64, c_i64, c_vp, c_vp],
    "mxs_softmax_ce": [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp],
    "mxs_fused_score_varlen": [c_int, c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_int,
                               c_vp],
    "mxs_quantize_per_token": [c_int, c_vp, c_i64, c_i64, c_int, c_vp, c_vp, c_vp],
    "mxs_csr_workspace_bytes": [c_i64, c_i64],
    "mxs_build_inverse_csr": [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_size, c_vp],
    "mxs_grad_docs_csr": [c_int, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp],
    "mxs_grad_query": [c_int, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp],
    "mxs_grad_docs_csr_f64": [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp],
    "mxs_grad_query_f64": [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp],
    "mxs_topk_workspace_bytes": [c_i64, c_i64],
    "mxs_topk": [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_size, c_vp],
    "mxs_topk_candidates": [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp],
    "mxs_sq_norms": [c_vp, c_i64, c_i64, c_vp, c_vp],
    "mxs_chamfer_nn": [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp],
    "mxs_chamfer_grad": [c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_dbl, c_dbl, c_vp, c_vp],
    "mxs_mxs1_open": [ctypes.c_char_p, ctypes.POINTER(c_vp)],
    "mxs_mxs1_info": [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
    "mxs_mxs1_cu_seqlens": [c_vp, c_vp],
    "mxs_mxs1_block_bytes": [c_vp, c_i64, c_i64],
    "mxs_mxs1_read_block": [c_vp, c_i64, c_i64, c_vp, c_size],
    "mxs_mxs1_read_scales": [c_vp, c_vp, c_size],
    "mxs_mxs1_close": [c_vp],
    "mxs_validate_lens": [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp],
    "mxs_validate_cu_seqlens": [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp],
}
_RESTYPES = {
    "mxs_version": ctypes.c_char_p,
    "mxs_status_string": ctypes.c_char_p,
    "mxs_last_error": ctypes.c_char_p,
    "mxs_csr_workspace_bytes": ctypes.c_size_t,
    "mxs_topk_workspace_bytes": ctypes.c_size_t,
    "mxs_mxs1_block_bytes": ctypes.c_int64,
    "mxs_mxs1_close": None,
}

MXS_F32, MXS_F16, MXS_BF16, MXS_I8 = 0, 1, 2, 3

_STATUS_TO_ERROR = {
    1: errors.DimMismatch,
    2: errors.ShapeMismatch,
    3: errors.EmptyDocument,
    4: errors.IndexOutOfRange,
    5: errors.StaleCsr,
    6: errors.KTooLarge,
    7: errors.NaNInput,
    8: errors.BadTileConfig,
    9: errors.Unsupported,
    10: errors.CudaError,
    11: errors.ShapeMismatch,
    12: errors.IoError,
    13: errors.BadMagic,
    14: errors.VersionUnsupported,
    15: errors.TruncatedPayload,
    16: errors.StaleArgmin,
}


def lib_path() -> str:
    return os.environ.get("MXS_LIB_PATH", LIB_PATH)


def load():
    """Load (once) and return the ctypes handle; raises if the native library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if not os.path.exists(path):
            raise RuntimeError(
                f"libmaxsim_b200.so not found at {path}; run `python -m paper_2605_29517_b200._build` "
                "(the operator has no CPU fallback)"
            )
        lib = ctypes.CDLL(path)
        for name, args in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, c_int)
        _lib = lib
    return _lib


def declared_symbols():
    return list(_SIGNATURES)


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    msg = load().mxs_last_error().decode(errors="replace")
    cls = _STATUS_TO_ERROR.get(status, errors.CudaError)
    text = f"{what}: {msg}" if what else msg
    if hasattr(cls, "from_message"):
        raise cls.from_message(text)
    raise cls(text)

def call(name: str, *args) -> None:
    fn = getattr(load(), name)
    check(fn(*args), name)
