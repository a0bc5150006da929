"""Chamfer distance on the device (maxsim/chamfer.py:1-218): the second instance of the
hard-selection pattern -- online MIN of squared Euclidean distances, argmins saved for the
backward, whose scatter halves run through the same inverse-CSR builder (K6) as the MaxSim
backward.

Forward and backward are bit-exact with the reference's arithmetic (float32 distances in the
reference's operation order, float64 gradients in its accumulation order); see
csrc/chamfer.cuh.  Inputs live on the GPU; there is no CPU fallback.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib
from .backward import csr_tensors
from .errors import DimMismatch, NaNInput, ShapeMismatch, StaleArgmin
from .instrument import TrafficReport
from .types import DEFAULT_TILE, ArgmaxMap, TileConfig

__all__ = ["PointSet", "chamfer_forward", "chamfer_backward", "dense_chamfer_forward", "dense_chamfer_backward"]


class PointSet:
    """n points of fixed dimension (3 for clouds), finite float32 rows (maxsim/chamfer.py:26-46)."""

    __slots__ = ("data", "n", "dim")

    def __init__(self, points):
        # our PointSet, or the reference's (numpy .data with .n / .dim) -- duck-typed
        src = points.data if isinstance(points, PointSet) or (hasattr(points, "data") and hasattr(points, "n")) \
            else points
        if isinstance(src, torch.Tensor):
            t = src.detach().to(torch.float32)
        else:
            t = torch.as_tensor(np.ascontiguousarray(src, dtype=np.float32))
        if t.dim() != 2:
            raise ShapeMismatch(f"point set must be 2-D [n x dim], got shape {tuple(t.shape)}")
        if t.shape[0] < 1:
            raise ShapeMismatch("point set must hold at least one point")
        finite = torch.isfinite(t)
        if not bool(finite.all()):
            bad = np.unravel_index(int(torch.argmin(finite.reshape(-1).to(torch.int8))), tuple(t.shape))
            raise NaNInput(("points",) + tuple(int(i) for i in bad))
        self.data = _dev.to_device(t.contiguous())
        self.n = int(t.shape[0])
        self.dim = int(t.shape[1])

    def __repr__(self):
        return f"PointSet(n={self.n}, dim={self.dim})"


def _as_points(x) -> PointSet:
    return x if isinstance(x, PointSet) else PointSet(x)


def _norms(x: torch.Tensor, stream=None) -> torch.Tensor:
    out = torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
    with _dev.on_device(x):
        _lib.call("mxs_sq_norms", _dev.ptr(x), x.shape[0], x.shape[1], _dev.ptr(out), _dev.stream_handle(stream, x.device))
    return out


def _nearest(a, an, b, bn, stream=None):
    best = torch.empty(a.shape[0], dtype=torch.float32, device=a.device)
    idx = torch.empty(a.shape[0], dtype=torch.int32, device=a.device)
    with _dev.on_device(a):
        _lib.call("mxs_chamfer_nn", _dev.ptr(a), _dev.ptr(an), a.shape[0], _dev.ptr(b), _dev.ptr(bn), b.shape[0],
                  a.shape[1], _dev.ptr(best), _dev.ptr(idx), _dev.stream_handle(stream, a.device))
    return best, idx


def _seq_sum_f64(values: torch.Tensor, stream=None) -> float:
    """Strict left-to-right float64 sum (maxsim/kernels.py:22-26) via the certified rowsum kernel."""
    out = torch.empty(1, dtype=torch.float64, device=values.device)
    with _dev.on_device(values):
        _lib.call("mxs_rowsum", _dev.ptr(values), 1, values.numel(), _dev.ptr(out),
                  _dev.stream_handle(stream, values.device))
    return float(out.item())


def chamfer_forward(p_set, s_set, tile: TileConfig = DEFAULT_TILE, report: TrafficReport | None = None):
    """Symmetric mean of squared nearest-neighbour distances (maxsim/chamfer.py:81-106).

    Returns (distance float, argmin_ps int32 [n] (device), argmin_sp int32 [m] (device)).  The
    [n x m] distance matrix never exists; tile is accepted for API parity (results are
    tile-invariant).
    """
    del tile
    p, s = _as_points(p_set), _as_points(s_set)
    if p.dim != s.dim:
        raise DimMismatch(p.dim, s.dim)
    rep = report if report is not None else TrafficReport()
    pn, sn = _norms(p.data), _norms(s.data)
    with rep.scratch(pn, sn):
        best_ps, argmin_ps = _nearest(p.data, pn, s.data, sn)
        best_sp, argmin_sp = _nearest(s.data, sn, p.data, pn)
        for a, b in ((p, s), (s, p)):
            rep.add_read(a.data.numel() * 4 + b.data.numel() * 4)
            rep.add_macs(2 * a.n * b.n * a.dim)
        rep.alloc(best_ps.numel() * 8 + best_sp.numel() * 8)
        cd = _seq_sum_f64(best_ps) / p.n + _seq_sum_f64(best_sp) / s.n
    rep.add_write(8)
    return cd, argmin_ps, argmin_sp


def dense_chamfer_forward(p_set, s_set, precision: str = "f32"):
    """Reference path materializing the pairwise matrix (maxsim/chamfer.py:109-142), on the device.

    "f32": the reference's elementwise float32 arrangement (same bits as chamfer_forward);
    "f64": distances from coordinate differences in float64, the independent tolerance oracle.
    """
    p, s = _as_points(p_set), _as_points(s_set)
    if p.dim != s.dim:
        raise DimMismatch(p.dim, s.dim)
    if precision == "f64":
        diff = p.data.double()[:, None, :] - s.data.double()[None, :, :]
        dist = (diff * diff).sum(dim=2)
        a1 = dist.argmin(dim=1).to(torch.int32)
        a2 = dist.argmin(dim=0).to(torch.int32)
        d1 = dist.min(dim=1).values
        d2 = dist.min(dim=0).values
        cd = float(torch.cumsum(d1, 0)[-1]) / p.n + float(torch.cumsum(d2, 0)[-1]) / s.n
        return cd, a1, a2
    if precision != "f32":
        raise ValueError(f"unknown precision {precision!r}")
    return chamfer_forward(p, s)


def _check_argmins(p: PointSet, s: PointSet, argmin_ps, argmin_sp):
    a1 = torch.as_tensor(argmin_ps).to(p.data.device).to(torch.int64)
    a2 = torch.as_tensor(argmin_sp).to(p.data.device).to(torch.int64)
    if tuple(a1.shape) != (p.n,) or tuple(a2.shape) != (s.n,):
        raise StaleArgmin("argmin lists do not match the point set sizes")
    if a1.numel() and (int(a1.min()) < 0 or int(a1.max()) >= s.n):
        raise StaleArgmin("argmin into the second set out of range")
    if a2.numel() and (int(a2.min()) < 0 or int(a2.max()) >= p.n):
        raise StaleArgmin("argmin into the first set out of range")
    return a1.to(torch.int32).contiguous(), a2.to(torch.int32).contiguous()


def _csr_of(nn: torch.Tensor, n_dest: int):
    """Inverse CSR of a nearest-neighbour list: one document of n_dest rows (the shared K6)."""
    dev = nn.device
    off = torch.zeros(1, dtype=torch.int64, device=dev)
    lens = torch.full((1,), n_dest, dtype=torch.int64, device=dev)
    row_ptr, col_idx, _ = csr_tensors(nn.reshape(1, 1, -1), off, lens, n_dest, n_dest)
    return row_ptr, col_idx


def _external_csr(builder, nn: torch.Tensor, n_dest: int, dev):
    """builder(ArgmaxMap of one document of n_dest rows) -> object with row_ptr / col_idx."""
    am = ArgmaxMap(nn.reshape(1, 1, -1), [n_dest], padded_len=n_dest)
    csr = builder(am)
    as_dev = lambda x: torch.as_tensor(np.asarray(x.cpu() if isinstance(x, torch.Tensor) else x)).to(  # noqa: E731
        device=dev, dtype=torch.int32).contiguous()
    return as_dev(csr.row_ptr), as_dev(csr.col_idx)


def chamfer_backward(p_set, s_set, argmin_ps, argmin_sp, upstream: float = 1.0,
                     report: TrafficReport | None = None, csr_builder=None):
    """Gradient through the fixed nearest-neighbour match (maxsim/chamfer.py:167-218).

    Returns (dP, dS) float64 on the device, bit-identical to the reference's loops.
    """
    p, s = _as_points(p_set), _as_points(s_set)
    a1, a2 = _check_argmins(p, s, argmin_ps, argmin_sp)
    rep = report if report is not None else TrafficReport()
    u = float(upstream)
    c_ps = 2.0 * u / p.n
    c_sp = 2.0 * u / s.n
    if csr_builder is None:
        rp_s, ci_s = _csr_of(a1, s.n)  # bucket r of S <- sources i of P (dS scatter half)
        rp_p, ci_p = _csr_of(a2, p.n)  # bucket r of P <- sources j of S (dP scatter half)
    else:  # an external inverse-CSR builder (the drop-in binding's shared-builder hook)
        rp_s, ci_s = _external_csr(csr_builder, a1, s.n, p.data.device)
        rp_p, ci_p = _external_csr(csr_builder, a2, p.n, p.data.device)
    rep.alloc(4 * (rp_s.numel() + ci_s.numel() + rp_p.numel() + ci_p.numel()))
    d_p = torch.empty((p.n, p.dim), dtype=torch.float64, device=p.data.device)
    d_s = torch.empty((s.n, s.dim), dtype=torch.float64, device=p.data.device)
    with _dev.on_device(p.data):
        st = _dev.stream_handle(None, p.data.device)
        _lib.call("mxs_chamfer_grad", _dev.ptr(p.data), p.n, _dev.ptr(s.data), p.dim, _dev.ptr(a1), _dev.ptr(rp_p),
                  _dev.ptr(ci_p), c_ps, c_sp, _dev.ptr(d_p), st)
        _lib.call("mxs_chamfer_grad", _dev.ptr(s.data), s.n, _dev.ptr(p.data), s.dim, _dev.ptr(a2), _dev.ptr(rp_s),
                  _dev.ptr(ci_s), c_sp, c_ps, _dev.ptr(d_s), st)
    return d_p, d_s


def dense_chamfer_backward(p_set, s_set, argmin_ps, argmin_sp, upstream: float = 1.0):
    """Reference gradient without CSR (maxsim/chamfer.py:201-218): source-order scatter adds in
    float64 on the device (index_add_, order not guaranteed -- a tolerance reference)."""
    p, s = _as_points(p_set), _as_points(s_set)
    a1, a2 = _check_argmins(p, s, argmin_ps, argmin_sp)
    P, S = p.data.double(), s.data.double()
    u = float(upstream)
    d1 = P - S[a1.long()]
    d2 = S - P[a2.long()]
    d_p = (2.0 * u / p.n) * d1
    d_s = (2.0 * u / s.n) * d2
    d_s = d_s.index_add(0, a1.long(), -(2.0 * u / p.n) * d1)
    d_p = d_p.index_add(0, a2.long(), -(2.0 * u / s.n) * d2)
    return d_p, d_s
