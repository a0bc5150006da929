"""Dense, materializing brute-force path on the device (maxsim/reference.py:1-170).

The API twin of the reference's tolerance oracle, for callers (and tests) that compare the fused
operator against the obvious computation: build the full [B, L_q, L_d] similarity tensor, mask
padding to -inf, reduce.  Not a hot path -- it allocates the tensor the fused kernels never write.

* precision "f32": the reference's element arithmetic (products rounded to fp32, then added in k
  order, never fused), so on fp32 inputs its scores and argmax match the exact fused kernel bit for
  bit;
* precision "f64": float64 similarities, the independent tolerance oracle.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from .errors import EmptyDocument, ShapeMismatch
from .instrument import TrafficReport
from .types import ArgmaxMap, DocBatch, as_embedding

__all__ = ["DenseSimTensor", "materialize_sims", "dense_score", "dense_score_batch", "dense_backward",
           "finite_diff_grad"]


@dataclass
class DenseSimTensor:
    """Materialized similarities (B, L_q, L_d), padding masked to -inf."""

    values: torch.Tensor

    @property
    def shape(self):
        return tuple(self.values.shape)


def _docs(docs) -> DocBatch:
    if isinstance(docs, DocBatch):
        return docs
    from .forward import as_docbatch

    return as_docbatch(docs)


def materialize_sims(query, docs, precision: str = "f32", report: TrafficReport | None = None) -> DenseSimTensor:
    """Full similarity tensor of one query against a batch (maxsim/reference.py:38-73)."""
    rep = report if report is not None else TrafficReport()
    q = as_embedding(query).data
    batch = _docs(docs)
    d3 = batch.data
    if precision == "f64":
        sims = torch.matmul(q.double()[None], d3.double().transpose(1, 2))
    elif precision == "f32":
        qf, df = q.float(), d3.float()
        sims = qf[None, :, 0, None] * df[:, None, :, 0]
        for k in range(1, qf.shape[1]):
            sims = sims + qf[None, :, k, None] * df[:, None, :, k]  # rounded product, then rounded add
    else:
        raise ValueError(f"unknown precision {precision!r}")
    rep.alloc(sims.numel() * sims.element_size())
    rep.add_read(q.numel() * q.element_size() + d3.numel() * d3.element_size())
    cols = torch.arange(sims.shape[2], device=sims.device)
    mask = cols[None, None, :] >= batch.valid_lens.to(sims.device)[:, None, None]
    return DenseSimTensor(sims.masked_fill(mask, float("-inf")))


def dense_score(query, docs, precision: str = "f32", report: TrafficReport | None = None):
    """(scores f64 [B], ArgmaxMap [1, B, L_q]) the brute-force way (maxsim/reference.py:76-104)."""
    batch = _docs(docs)
    lens = batch.valid_lens_host
    for b in range(batch.n_docs):
        if int(lens[b]) < 1:
            raise EmptyDocument(b)
    q = as_embedding(query)
    if q.dim != batch.dim:
        from .errors import DimMismatch

        raise DimMismatch(q.dim, batch.dim)
    rep = report if report is not None else TrafficReport()
    s = materialize_sims(q, batch, precision=precision, report=rep).values
    maxima, winners = s.max(dim=2)  # lowest index on ties
    scores = torch.cumsum(maxima.double(), dim=1)[:, -1]  # sequential f64 sum per document
    rep.add_write(scores.numel() * 8)
    rep.release(s.numel() * s.element_size())
    return scores, ArgmaxMap(winners.to(torch.int32)[None], lens, padded_len=batch.padded_len)


def dense_score_batch(queries, docs, precision: str = "f32", report: TrafficReport | None = None):
    """All-pairs (scores f64 [N_q, B], ArgmaxMap) by looping dense_score (maxsim/reference.py:107-120)."""
    rep = report if report is not None else TrafficReport()
    batch = _docs(docs)
    qs = list(queries) if not isinstance(queries, torch.Tensor) else list(queries)
    outs = [dense_score(q, batch, precision=precision, report=rep) for q in qs]
    scores = torch.stack([o[0] for o in outs])
    idx = torch.cat([o[1].indices for o in outs])
    return scores, ArgmaxMap(idx, batch.valid_lens_host, padded_len=batch.padded_len)


def dense_backward(queries, docs, upstream, argmax):
    """Gradients of sum(upstream * scores), float64 (maxsim/reference.py:123-155).

    dQ is a gather; dD a scatter (index_add_ -- a tolerance reference: the device does not
    promise the reference's sequential scatter order, the fused CSR path does).
    """
    batch = _docs(docs)
    qs = torch.stack([as_embedding(q).data for q in queries]) if not isinstance(queries, torch.Tensor) else queries
    g = torch.as_tensor(np.asarray(upstream, dtype=np.float64) if not isinstance(upstream, torch.Tensor) else upstream)
    n_q, b = qs.shape[0], batch.n_docs
    if tuple(g.shape) != (n_q, b):
        raise ShapeMismatch(f"upstream shape {tuple(g.shape)} does not match ({n_q}, {b})")
    idx = argmax.indices if isinstance(argmax, ArgmaxMap) else torch.as_tensor(np.asarray(argmax))
    idx = idx.to(_dev.device()).long()
    if tuple(idx.shape[:2]) != (n_q, b):
        raise ShapeMismatch("argmax map does not match the query/document batch")
    g = g.to(_dev.device(), torch.float64)
    D = batch.data.double()
    Q = qs.to(_dev.device()).double()
    rows = D[torch.arange(b, device=D.device)[None, :, None], idx]  # [N_q, B, L_q, d]
    d_q = (g[:, :, None, None] * rows).sum(dim=1)
    d_d = torch.zeros_like(D)
    flat = (torch.arange(b, device=D.device)[None, :, None] * batch.padded_len + idx).reshape(-1)
    src = (g[:, :, None, None] * Q[:, None, :, :]).reshape(-1, Q.shape[-1])
    d_d.view(-1, Q.shape[-1]).index_add_(0, flat, src)
    return d_q, d_d


def finite_diff_grad(score_fn, point, eps: float) -> np.ndarray:
    """Central-difference gradient of a scalar function, float64 (maxsim/reference.py:158-170)."""
    if eps <= 0:
        raise ValueError(f"finite-difference step must be positive, got {eps}")
    x = np.array(point, dtype=np.float64)
    grad = np.zeros_like(x)
    xf, gf = x.reshape(-1), grad.reshape(-1)
    for i in range(xf.size):
        keep = xf[i]
        xf[i] = keep + eps
        hi = float(score_fn(x))
        xf[i] = keep - eps
        lo = float(score_fn(x))
        xf[i] = keep
        gf[i] = (hi - lo) / (2.0 * eps)
    return grad
