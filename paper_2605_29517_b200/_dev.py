"""Device plumbing shared by the operator modules: tensors, pointers, streams, dtype codes."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import Unsupported

_DT_CODE = {torch.float32: _lib.MXS_F32, torch.float16: _lib.MXS_F16, torch.bfloat16: _lib.MXS_BF16,
            torch.int8: _lib.MXS_I8}
_ELEM_TAG = {torch.float32: "f32", torch.float16: "f16", torch.bfloat16: "bf16", torch.int8: "i8"}


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2605_29517_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x, dtype=None) -> torch.Tensor:
    """Array-like / tensor -> contiguous CUDA tensor (no copy when already there).

    Without a CUDA device the tensor stays on the host so that the host-side logic (types,
    validation, error mapping) stays testable; every compute entry point then raises through
    require_cuda() -- there is no CPU compute path.
    """
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.as_tensor(np.asarray(x))
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    if not t.is_cuda and torch.cuda.is_available():
        t = t.to(device(), non_blocking=False)
    return t.contiguous()


def require_cuda(*tensors) -> None:
    """Raise unless every tensor lives on a CUDA device (the kernels are the only compute path)."""
    _lib.load()
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise RuntimeError("paper_2605_29517_b200 operators run only on CUDA tensors (sm_100a); "
                               "there is no CPU fallback")


def ptr(t) -> ctypes.c_void_p | None:
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def stream_handle(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT_CODE[t.dtype]
    except KeyError:
        raise Unsupported(f"dtype {t.dtype} is not supported by the sm_100a kernels") from None


def elem_tag(t: torch.Tensor) -> str:
    return _ELEM_TAG.get(t.dtype, str(t.dtype))


def itemsize(t: torch.Tensor) -> int:
    return t.element_size()
