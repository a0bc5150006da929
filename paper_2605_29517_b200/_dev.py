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


def stream_handle(stream=None, dev=None) -> ctypes.c_void_p:
    """The given stream, else the current stream of `dev` (a tensor's device), else of the current device."""
    if stream is None:
        stream = torch.cuda.current_stream(dev) if dev is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def on_device(t: torch.Tensor):
    """Context that makes t's GPU the current device for a launch (kernels, TMA maps and the
    per-device shared-memory opt-ins all follow the current device)."""
    return torch.cuda.device(t.device)


def keep_alive(t: torch.Tensor | None, stream=None) -> torch.Tensor | None:
    """Record a temporary's use on a non-current launch stream so the caching allocator cannot
    hand its block out again before the kernel has read it."""
    if t is not None and stream is not None and t.is_cuda:
        t.record_stream(stream)
    return t


def validate_lens(valid_lens: torch.Tensor, l_pad: int, stream=None) -> None:
    """Reference checks of maxsim/forward.py:173-176 on device-resident valid_lens (synchronous)."""
    from .errors import EmptyDocument, ShapeMismatch

    bi, bv = ctypes.c_int64(-1), ctypes.c_int64(0)
    st = _lib.load().mxs_validate_lens(ptr(valid_lens), valid_lens.numel(), l_pad, ctypes.byref(bi),
                                       ctypes.byref(bv), stream_handle(stream, valid_lens.device))
    if st == 0:
        return
    if st == 3:
        raise EmptyDocument(int(bi.value))
    if st == 2:
        raise ShapeMismatch(f"valid_len {int(bv.value)} exceeds document rows {l_pad}")
    _lib.check(st, "mxs_validate_lens")


def validate_cu(cu: torch.Tensor, n_tokens: int, stream=None) -> None:
    """Reference checks of maxsim/varlen.py:35-41 on a device-resident cu_seqlens (synchronous)."""
    from .errors import EmptyDocument

    if cu.dim() != 1 or cu.numel() < 2:
        from .errors import ShapeMismatch

        raise ShapeMismatch("cu_seqlens must be 1-D with cu[0] = 0 and one entry per document plus one")
    bi, bv = ctypes.c_int64(-1), ctypes.c_int64(0)
    st = _lib.load().mxs_validate_cu_seqlens(ptr(cu), cu.numel() - 1, n_tokens, ctypes.byref(bi), ctypes.byref(bv),
                                             stream_handle(stream, cu.device))
    if st == 3:
        raise EmptyDocument(int(bi.value))
    _lib.check(st, "mxs_validate_cu_seqlens")


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT_CODE[t.dtype]
    except KeyError:
        raise Unsupported(f"dtype {t.dtype} is not supported by the sm_100a kernels") from None


def elem_tag(t: torch.Tensor) -> str:
    return _ELEM_TAG.get(t.dtype, str(t.dtype))


def itemsize(t: torch.Tensor) -> int:
    return t.element_size()
