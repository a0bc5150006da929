"""Materialization-free MaxSim forward on sm_100a (mirror of maxsim/forward.py:1-265).

The per-pair fold of the reference (`_fold_pair`, maxsim/forward.py:108-155) runs inside
libmaxsim_b200: the tcgen05 kernel (bf16 / fp16 inputs, fp32 accumulation in TMEM) or the
bit-exact fp32 kernel (float32 inputs, the reference's sequential fold).  Either way the
[L_q x L_d] similarity tile never reaches HBM; only per-row (max, argmax) and the f64 score do.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .errors import EmptyDocument, ShapeMismatch, Unsupported
from .instrument import TrafficReport
from .types import (
    DEFAULT_TILE,
    ArgmaxMap,
    DocBatch,
    EmbeddingMatrix,
    ScoreMatrix,
    TileConfig,
    as_embedding,
    validate_pair,
)

STRATEGY_TAGS = ("single_query_rerank", "batched_multiquery", "varlen_packed", "int8_two_stage")


@dataclass
class RunningRowState:
    """Streaming state for the query rows in flight (maxsim/forward.py:39-49).

    On the device this state lives in registers of the epilogue warps (one TMEM lane = one
    query row); the dataclass is kept for API parity.
    """

    m: np.ndarray
    arg: np.ndarray
    acc: float = 0.0


@dataclass(frozen=True)
class ForwardStrategy:
    tag: str
    tile: TileConfig = field(default_factory=lambda: DEFAULT_TILE)


DOC_LEN_LONG = 2048
TILE_LOOKUP = {
    "default": TileConfig(bq=32, bd=64, qchunk=128),
    "long_doc": TileConfig(bq=32, bd=128, qchunk=128),
    "int8": TileConfig(bq=32, bd=128, qchunk=128),
}


def dispatch(n_queries, n_docs, len_q, len_d, dim, dtype="f32", packed=False) -> ForwardStrategy:
    """Same deterministic rules as maxsim/forward.py:73-90 (i8, then packed, then N_q == 1)."""
    for v in (n_queries, n_docs, len_q, len_d, dim):
        if v < 1:
            raise ValueError("dispatch expects positive shape values")
    if dtype == "i8":
        return ForwardStrategy("int8_two_stage", TILE_LOOKUP["int8"])
    tile = TILE_LOOKUP["long_doc"] if len_d >= DOC_LEN_LONG else TILE_LOOKUP["default"]
    if packed:
        return ForwardStrategy("varlen_packed", tile)
    if n_queries == 1:
        return ForwardStrategy("single_query_rerank", tile)
    return ForwardStrategy("batched_multiquery", tile)


def query_chunk_decompose(query: EmbeddingMatrix, chunk_len: int):
    """Row chunks whose partial scores sum to the whole (maxsim/forward.py:93-105)."""
    if chunk_len < 1:
        raise ValueError(f"chunk_len must be >= 1, got {chunk_len}")
    query = as_embedding(query)
    chunks = [EmbeddingMatrix(query.data[r0 : r0 + chunk_len]) for r0 in range(0, query.rows, chunk_len)]
    return chunks if chunks else [query]


# --------------------------------------------------------------------------- core launcher
def use_exact_path(dtype: torch.dtype, dim: int, exact: bool | None) -> bool:
    if exact is not None:
        if not exact and dtype == torch.float32:
            raise Unsupported("float32 inputs run on the bit-exact fp32 kernel; cast to bf16/fp16 for tcgen05")
        return bool(exact)
    return dtype == torch.float32 or dim % 8 != 0


def score_dense(Q: torch.Tensor, D: torch.Tensor, valid_lens: torch.Tensor | None = None, *, exact: bool | None = None,
                want_argmax: bool = True, want_rowmax: bool = False, out=None, stream=None, validate: bool = True):
    """Tensor-level dense forward: Q [n_q, l_q, d], D [B, L_pad, d] on CUDA.

    Returns (scores f64 [n_q, B], argmax int32 [n_q, B, l_q] or None, rowmax f32 [n_q, B, l_q] or None).
    The per-token maxima are materialised only with want_rowmax=True (the tensor-core kernels fold
    the f64 score into their epilogue).  `out` may supply preallocated (scores, argmax, rowmax)
    buffers (CUDA-graph friendly; argmax / rowmax entries may be None).  With validate=True (the
    default) device-resident valid_lens are checked like maxsim/forward.py:173-176 (one sync);
    callers holding validated lengths (DocBatch, graphs) pass validate=False.
    """
    _dev.require_cuda(Q, D, valid_lens)
    if Q.dim() != 3 or D.dim() != 3:
        raise ShapeMismatch("score_dense expects Q [n_q, l_q, d] and D [B, L, d]")
    n_q, l_q, d = Q.shape
    b, l_pad, d2 = D.shape
    if d != d2:
        from .errors import DimMismatch

        raise DimMismatch(int(d), int(d2))
    if Q.dtype != D.dtype:
        Q = Q.to(D.dtype)
    Q = Q.contiguous()
    D = D.contiguous()
    exact_path = use_exact_path(D.dtype, int(d), exact)
    with _dev.on_device(D):
        if valid_lens is not None:
            if valid_lens.dtype != torch.int32 or not valid_lens.is_contiguous():
                valid_lens = valid_lens.to(torch.int32).contiguous()
            if valid_lens.numel() != b:
                raise ShapeMismatch(f"valid_lens holds {valid_lens.numel()} entries for {b} documents")
            if validate:
                _dev.validate_lens(valid_lens, l_pad, stream)
        if out is not None:
            scores, argmax, rowmax = out
        else:
            scores = torch.empty((n_q, b), dtype=torch.float64, device=D.device)
            argmax = torch.empty((n_q, b, l_q), dtype=torch.int32, device=D.device) if want_argmax else None
            rowmax = torch.empty((n_q, b, l_q), dtype=torch.float32, device=D.device) if want_rowmax else None
        for t in (Q, D, valid_lens):
            _dev.keep_alive(t, stream)
        _lib.call("mxs_fused_score_batch", _dev.dtype_code(D), _dev.ptr(Q), n_q, l_q, _dev.ptr(D), b, l_pad, d,
                  _dev.ptr(valid_lens), _dev.ptr(scores), _dev.ptr(argmax), _dev.ptr(rowmax), 1 if exact_path else 0,
                  _dev.stream_handle(stream, D.device))
    return scores, argmax, rowmax


def _stack_queries(queries):
    if isinstance(queries, torch.Tensor):
        if queries.dim() == 2:
            queries = queries[None]
        return _dev.to_device(queries)
    if isinstance(queries, EmbeddingMatrix) or hasattr(queries, "rows"):
        queries = [queries]
    if len(queries) == 0:
        raise ShapeMismatch("need at least one query")
    mats = [as_embedding(q) for q in queries]
    l_q = mats[0].rows
    for m in mats:
        if m.rows != l_q:
            raise ShapeMismatch("batched queries must share length; pack ragged queries separately")
    return torch.stack([m.data for m in mats])


def as_docbatch(docs) -> DocBatch:
    if isinstance(docs, DocBatch):
        return docs
    if isinstance(docs, torch.Tensor):
        return DocBatch.from_dense(docs)
    if hasattr(docs, "valid_lens") and hasattr(docs, "data"):
        return DocBatch.from_reference(docs)
    return DocBatch(docs)


def _account_dense(rep, n_q, l_q, b, l_pad, d, e, count_query):
    if count_query:
        rep.add_read(n_q * l_q * d * e)
    rep.add_read(n_q * b * l_pad * d * e)
    rep.add_macs(2 * n_q * b * l_q * l_pad * d)
    rep.add_write(8 * n_q * b)


def fused_score_batch(queries, docs, tile: TileConfig = DEFAULT_TILE, report: TrafficReport | None = None,
                      threads: int = 1, count_query: bool = True, exact: bool | None = None):
    """All-pairs scores for N_q queries vs B documents (maxsim/forward.py:221-265).

    `threads` is accepted for API parity; the device decides its own parallelism.
    Returns (ScoreMatrix, ArgmaxMap, TrafficReport).
    """
    if not isinstance(tile, TileConfig) and not all(hasattr(tile, a) for a in ("bq", "bd", "qchunk")):
        raise TypeError("tile must be a TileConfig")  # ours or the reference's (duck-typed)
    Q = _stack_queries(queries)
    docs = as_docbatch(docs)
    if Q.shape[-1] != docs.dim:
        from .errors import DimMismatch

        raise DimMismatch(int(Q.shape[-1]), docs.dim)
    rep = report if report is not None else TrafficReport()
    if Q.dtype != docs.data.dtype:
        Q = Q.to(docs.data.dtype)
    n_q, l_q, d = Q.shape
    scores, argmax, _ = score_dense(Q, docs.data, docs.valid_lens, exact=exact, validate=False)
    rep.alloc(n_q * docs.n_docs * l_q * 4)  # per-token maxima (registers / shared memory on the device)
    rep.release(n_q * docs.n_docs * l_q * 4)
    _account_dense(rep, n_q, l_q, docs.n_docs, docs.padded_len, d, _dev.itemsize(docs.data), count_query)
    am = ArgmaxMap(argmax, docs.valid_lens_host, padded_len=docs.padded_len, validate=False)
    return ScoreMatrix(scores, validate=False), am, rep


def fused_score_pair(query, doc, valid_len: int | None = None, tile: TileConfig = DEFAULT_TILE,
                     report: TrafficReport | None = None, exact: bool | None = None):
    """One (query, document) pair (maxsim/forward.py:158-185) -> (float score, int32 argmax [L_q], report)."""
    validate_pair(query, doc)
    q = as_embedding(query)
    dm = as_embedding(doc)
    if valid_len is None:
        valid_len = dm.rows
    if valid_len < 1:
        raise EmptyDocument(0)
    if valid_len > dm.rows:
        raise ShapeMismatch(f"valid_len {valid_len} exceeds document rows {dm.rows}")
    rep = report if report is not None else TrafficReport()
    D = dm.data[None]
    vl = torch.tensor([valid_len], dtype=torch.int32, device=D.device)
    Q = q.data[None].to(D.dtype)
    scores, argmax, _ = score_dense(Q, D, vl, exact=exact, validate=False)
    _account_dense(rep, 1, q.rows, 1, dm.rows, dm.dim, _dev.itemsize(D), True)
    return float(scores[0, 0].item()), argmax[0, 0], rep
