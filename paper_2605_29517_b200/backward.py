"""Exact MaxSim backward on the device (mirror of maxsim/backward.py:1-279).

The forward saves one winning document-token index per (query, document, query token); the
max is then resolved and the score is piecewise linear:

    dQ[q, s] = sum_b g[q, b] * D[b, argmax[q, b, s]]             (gather, K8)
    dD[b, t] = sum over sources that picked t of g * Q row         (CSR reduction, K7)

The scatter side is inverted on the device into the reference's CSR (stable bucket order,
K6) and reduced destination-owned: one warp per output row, fp32 accumulation, exactly one
store per row, no atomics.  The reference's atomic-scatter fallback (`grad_docs_scatter`) has
the same result contract; here it routes through the same atomic-free CSR reduction.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .errors import ShapeMismatch, StaleCsr
from .instrument import TrafficReport
from .types import ArgmaxMap, DocBatch, EmbeddingMatrix, as_embedding

DEFAULT_SCATTER_THRESHOLD = 8


@dataclass
class CsrInverse:
    """Destination-owned inversion of an ArgmaxMap (maxsim/backward.py:47-78).

    row_ptr int32 [n_dest + 1], col_idx int32 [n_sources] (CUDA); each bucket lists flat source
    positions (q, b, s) in ascending order.  `to_numpy()` gives the reference's int64 arrays.
    """

    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    n_dest: int
    src_shape: tuple
    padded_len: int | None

    @property
    def n_sources(self) -> int:
        return int(self.col_idx.numel())

    def destinations_per_source(self) -> torch.Tensor:
        counts = (self.row_ptr[1:] - self.row_ptr[:-1]).to(torch.int64)
        per_pos = torch.repeat_interleave(torch.arange(self.n_dest, device=counts.device), counts)
        dst = torch.empty(self.n_sources, dtype=torch.int64, device=counts.device)
        dst[self.col_idx.to(torch.int64)] = per_pos
        return dst

    def check_sources(self, n_queries: int, n_docs: int, len_q: int) -> None:
        if tuple(self.src_shape) != (n_queries, n_docs, len_q):
            raise StaleCsr(
                f"CSR built for source shape {tuple(self.src_shape)}, applied to ({n_queries}, {n_docs}, {len_q})"
            )

    def to_numpy(self):
        return self.row_ptr.cpu().numpy().astype(np.int64), self.col_idx.cpu().numpy().astype(np.int64)


def as_argmax_map(argmax) -> ArgmaxMap:
    if isinstance(argmax, ArgmaxMap):
        return argmax
    return ArgmaxMap(np.asarray(argmax.indices), argmax.doc_lens, padded_len=argmax.padded_len)


def csr_tensors(indices: torch.Tensor, dest_off: torch.Tensor, dest_len: torch.Tensor, n_dest: int, max_len: int,
                stream=None):
    """Tensor-level CSR build: indices int32 [n_q, B, l_q], dest_off / dest_len int64 [B] (CUDA).

    Returns (row_ptr int32 [n_dest + 1], col_idx int32 [n_q * B * l_q], workspace bytes used).
    """
    _dev.require_cuda(indices, dest_off, dest_len)
    n_q, b, l_q = indices.shape
    dev = indices.device
    row_ptr = torch.empty(n_dest + 1, dtype=torch.int32, device=dev)
    col_idx = torch.empty(indices.numel(), dtype=torch.int32, device=dev)
    ws_bytes = int(_lib.load().mxs_csr_workspace_bytes(n_q, n_dest))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    idx = indices.contiguous()  # bound to a name: alive until the launch is queued
    with _dev.on_device(idx):
        _lib.call("mxs_build_inverse_csr", _dev.ptr(idx), n_q, b, l_q, _dev.ptr(dest_off), _dev.ptr(dest_len), n_dest,
                  max_len, _dev.ptr(row_ptr), _dev.ptr(col_idx), _dev.ptr(ws), ws_bytes,
                  _dev.stream_handle(stream, dev))
    for t in (idx, dest_off, dest_len, ws):
        _dev.keep_alive(t, stream)  # non-current launch stream: the allocator must not recycle them early
    return row_ptr, col_idx, ws_bytes


def build_inverse_csr(argmax, report: TrafficReport | None = None, stream=None) -> CsrInverse:
    """Invert the argmax map on the device (maxsim/backward.py:81-109)."""
    am = as_argmax_map(argmax)
    rep = report if report is not None else TrafficReport()
    n_q, b, l_q = am.indices.shape
    n_dest = am.n_dest_rows
    off, lens = am.device_offsets()
    max_len = int(am.dest_row_lens().max()) if b else 0
    row_ptr, col_idx, ws_bytes = csr_tensors(am.indices, off, lens, n_dest, max_len, stream)
    rep.alloc(ws_bytes)
    rep.release(ws_bytes)
    rep.alloc(row_ptr.numel() * 4 + col_idx.numel() * 4)
    return CsrInverse(row_ptr=row_ptr, col_idx=col_idx, n_dest=n_dest, src_shape=(n_q, b, l_q),
                      padded_len=am.padded_len)


def _check_upstream(upstream, n_queries: int, n_docs: int, device, dtype=torch.float32) -> torch.Tensor:
    g = upstream if isinstance(upstream, torch.Tensor) else torch.as_tensor(np.asarray(upstream, dtype=np.float64))
    if tuple(g.shape) != (n_queries, n_docs):
        raise ShapeMismatch(f"upstream gradient shape {tuple(g.shape)}, expected ({n_queries}, {n_docs})")
    return g.to(device=device, dtype=dtype).contiguous()


def _stack_query_rows(queries) -> torch.Tensor:
    if isinstance(queries, torch.Tensor):
        return queries if queries.dim() == 3 else queries[None]
    mats = [as_embedding(q) for q in queries]
    for m in mats:
        if m.data.shape != mats[0].data.shape:
            raise ShapeMismatch("queries must share shape for the batched backward")
    return torch.stack([m.data for m in mats])


def grad_docs_csr(csr: CsrInverse, upstream, queries, report: TrafficReport | None = None, out=None,
                  stream=None) -> torch.Tensor:
    """Destination-owned document gradient (maxsim/backward.py:135-173) -> flat (n_dest, dim).

    FP32 queries: float64, the reference's exact arithmetic and order (bit-identical).  bf16 /
    fp16 queries (the tensor-core path): fp32 accumulation (north_star: gradients within 1e-3).
    """
    rep = report if report is not None else TrafficReport()
    Q = _stack_query_rows(queries).contiguous()
    _dev.require_cuda(Q, csr.row_ptr)
    n_q, l_q, dim = Q.shape
    n_docs = csr.src_shape[1]
    exact = Q.dtype == torch.float32
    odt = torch.float64 if exact else torch.float32
    g = _check_upstream(upstream, n_q, n_docs, Q.device, odt)
    csr.check_sources(n_q, n_docs, l_q)
    if csr.n_sources != n_q * n_docs * l_q:
        raise StaleCsr("CSR source count disagrees with the argmax shape")
    if out is None or out.dtype != odt:
        out = torch.empty((csr.n_dest, dim), dtype=odt, device=Q.device)
    with _dev.on_device(Q):
        st = _dev.stream_handle(stream, Q.device)
        if exact:
            _lib.call("mxs_grad_docs_csr_f64", _dev.ptr(csr.row_ptr), _dev.ptr(csr.col_idx), csr.n_dest, _dev.ptr(g),
                      _dev.ptr(Q), n_q, n_docs, l_q, dim, _dev.ptr(out), st)
        else:
            _lib.call("mxs_grad_docs_csr", _dev.dtype_code(Q), _dev.ptr(csr.row_ptr), _dev.ptr(csr.col_idx),
                      csr.n_dest, _dev.ptr(g), _dev.ptr(Q), n_q, n_docs, l_q, dim, _dev.ptr(out), st)
    for t in (Q, g):
        _dev.keep_alive(t, stream)
    rep.add_read(csr.n_sources * (4 + dim * Q.element_size()))
    rep.add_write(csr.n_dest * dim * out.element_size())
    return out


def grad_docs_scatter(argmax, upstream, queries, report: TrafficReport | None = None) -> torch.Tensor:
    """Same contract as maxsim/backward.py:176-207; computed through the atomic-free CSR path."""
    am = as_argmax_map(argmax)
    Q = _stack_query_rows(queries)
    if am.len_q != Q.shape[1]:
        raise ShapeMismatch("argmax map and queries disagree on query length")
    return grad_docs_csr(build_inverse_csr(am, report=report), upstream, Q, report=report)


def _doc_rows(docs):
    """Flat [rows, dim] document buffer and per-document first-row offsets."""
    from .varlen import PackedCorpus

    if isinstance(docs, DocBatch):
        b, l, d = docs.data.shape
        off = torch.arange(b, dtype=torch.int64, device=docs.data.device) * l
        return docs.data.reshape(b * l, d), off
    if isinstance(docs, PackedCorpus):
        return docs.tokens, docs.cu_dev[:-1].contiguous()
    if isinstance(docs, torch.Tensor) and docs.dim() == 3:
        b, l, d = docs.shape
        return docs.reshape(b * l, d), torch.arange(b, dtype=torch.int64, device=docs.device) * l
    if hasattr(docs, "tokens") and hasattr(docs, "cu_seqlens"):  # the reference's PackedCorpus
        return _doc_rows(PackedCorpus(docs.tokens, docs.cu_seqlens))
    if hasattr(docs, "valid_lens") and hasattr(docs, "data"):  # the reference's DocBatch
        return _doc_rows(DocBatch.from_reference(docs))
    raise ShapeMismatch(f"unsupported document container {type(docs).__name__}")


def grad_query(argmax, upstream, docs, stream=None) -> torch.Tensor:
    """Query gradient, a pure gather (maxsim/backward.py:218-231) -> (N_q, L_q, dim): float64
    (bit-identical) for fp32 documents, fp32 accumulation for bf16 / fp16."""
    am = as_argmax_map(argmax)
    rows, off = _doc_rows(docs)
    _dev.require_cuda(am.indices, rows)
    n_q, b, l_q = am.indices.shape
    dim = rows.shape[-1]
    exact = rows.dtype == torch.float32
    odt = torch.float64 if exact else torch.float32
    g = _check_upstream(upstream, n_q, b, rows.device, odt)
    out = torch.empty((n_q, l_q, dim), dtype=odt, device=rows.device)
    rows = rows.contiguous()
    idx = am.indices.contiguous()
    with _dev.on_device(rows):
        st = _dev.stream_handle(stream, rows.device)
        if exact:
            _lib.call("mxs_grad_query_f64", _dev.ptr(idx), _dev.ptr(g), _dev.ptr(rows), _dev.ptr(off), n_q, b, l_q, dim,
                      _dev.ptr(out), st)
        else:
            _lib.call("mxs_grad_query", _dev.dtype_code(rows), _dev.ptr(idx), _dev.ptr(g), _dev.ptr(rows),
                      _dev.ptr(off), n_q, b, l_q, dim, _dev.ptr(out), st)
    for t in (rows, idx, g, off):
        _dev.keep_alive(t, stream)
    return out


def choose_gradient_path(argmax, threshold: int = DEFAULT_SCATTER_THRESHOLD) -> str:
    """"csr" when the max bucket load exceeds the threshold (maxsim/backward.py:234-243)."""
    am = as_argmax_map(argmax)
    if am.n_sources == 0:
        return "scatter"
    counts = torch.bincount(am.flat_destinations(), minlength=am.n_dest_rows)
    return "csr" if int(counts.max().item()) > threshold else "scatter"


def doc_grads_in_layout(flat: torch.Tensor, argmax) -> torch.Tensor:
    """(B, padded_len, dim) for padded corpora, flat (sum L_d, dim) when packed (maxsim/backward.py:246-255)."""
    am = as_argmax_map(argmax)
    if am.padded_len is not None:
        return flat.reshape(am.n_docs, am.padded_len, flat.shape[1])
    return flat


def backward_dispatch(argmax, upstream, queries, docs, threshold: int = DEFAULT_SCATTER_THRESHOLD,
                      report: TrafficReport | None = None):
    """Full backward (maxsim/backward.py:258-279) -> (dQ, dD): float64 for fp32 inputs (the
    reference's arithmetic, bit-identical), fp32 accumulation for bf16 / fp16.

    The device always runs the atomic-free CSR reduction; `threshold` is accepted for API
    parity (the reference's result contract does not depend on the chosen path).
    """
    rep = report if report is not None else TrafficReport()
    am = as_argmax_map(argmax)
    if not isinstance(docs, DocBatch):
        from .varlen import PackedCorpus

        if hasattr(docs, "tokens") and hasattr(docs, "cu_seqlens") and not isinstance(docs, PackedCorpus):
            docs = PackedCorpus(docs.tokens, docs.cu_seqlens)  # the reference's PackedCorpus
        if not isinstance(docs, PackedCorpus):
            from .forward import as_docbatch

            docs = as_docbatch(docs)
    csr = build_inverse_csr(am, report=rep)
    flat = grad_docs_csr(csr, upstream, queries, report=rep)
    d_q = grad_query(am, upstream, docs)
    return d_q, doc_grads_in_layout(flat, am)
