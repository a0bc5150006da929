"""Per-token symmetric INT8 scoring on the tcgen05 int8 path (mirror of maxsim/quant.py:1-231).

Quantisation (K4) is bit-exact with the reference: scale = fl32(maxabs / levels) (1e-12 for a
zero row), values rounded half-to-even and clamped to [-levels, levels].  Scoring (K3) runs
`tcgen05.mma.kind::i8` with exact int32 accumulation in TMEM; the epilogue applies
fl(fl(f32(acc) * s_q[i]) * s_d[j]) before the same masked online max as the float path, so
INT8 scores and argmax are bit-identical to the reference including ties.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib
from .errors import DimMismatch, EmptyDocument, KTooLarge, ShapeMismatch
from .instrument import TrafficReport
from .types import DEFAULT_TILE, ArgmaxMap, DocBatch, EmbeddingMatrix, ScoreMatrix, TileConfig

ZERO_ROW_SCALE = np.float32(1e-12)
MAX_INT8_DIM = 133_000


def _t(x, dtype):
    return _dev.to_device(x if isinstance(x, torch.Tensor) else np.asarray(x), dtype)


class QuantizedMatrix:
    """int8 token rows plus one positive scale per token (maxsim/quant.py:34-63)."""

    __slots__ = ("q", "scale")

    def __init__(self, q, scale, validate: bool = True):
        self.q = _t(q, torch.int8)
        self.scale = _t(scale, torch.float32)
        if self.q.dim() != 2:
            raise ShapeMismatch(f"quantized rows must be 2-D, got shape {tuple(self.q.shape)}")
        if tuple(self.scale.shape) != (self.q.shape[0],):
            raise ShapeMismatch("need exactly one scale per token row")
        if self.q.shape[1] > MAX_INT8_DIM:
            raise ShapeMismatch(f"dim {self.q.shape[1]} exceeds {MAX_INT8_DIM}; int32 dot accumulation could overflow")
        if validate and self.scale.numel() and float(self.scale.min()) <= 0.0:
            raise ShapeMismatch("token scales must be positive")

    @property
    def rows(self) -> int:
        return int(self.q.shape[0])

    @property
    def dim(self) -> int:
        return int(self.q.shape[1])


class QuantizedCorpus:
    """Uniform-length quantized corpus: (B, L, dim) int8 plus (B, L) scales (maxsim/quant.py:66-101)."""

    __slots__ = ("q", "scales")

    def __init__(self, q, scales):
        self.q = _t(q, torch.int8)
        self.scales = _t(scales, torch.float32)
        if self.q.dim() != 3 or tuple(self.scales.shape) != tuple(self.q.shape[:2]):
            raise ShapeMismatch("quantized corpus needs (B, L, dim) rows and (B, L) scales")

    @property
    def n_docs(self) -> int:
        return int(self.q.shape[0])

    @property
    def elem(self) -> str:
        return "i8"

    def doc(self, b: int) -> QuantizedMatrix:
        return QuantizedMatrix(self.q[b], self.scales[b], validate=False)

    def matrices(self):
        return [self.doc(b) for b in range(self.n_docs)]

    def __len__(self):
        return self.n_docs

    def __getitem__(self, b):
        return self.doc(b)

    @classmethod
    def from_matrices(cls, mats) -> "QuantizedCorpus":
        lens = {m.rows for m in mats}
        if len(lens) != 1:
            raise ShapeMismatch("quantized file layout requires uniform document length")
        return cls(q=torch.stack([_t(m.q, torch.int8) for m in mats]),
                   scales=torch.stack([_t(m.scale, torch.float32) for m in mats]))


def quantize_tensor(x: torch.Tensor, levels: int = 127, stream=None):
    """Device quantisation of any [..., dim] float tensor -> (q int8 [..., dim], scale f32 [...])."""
    if not 1 <= levels <= 127:
        raise ValueError(f"levels must be in [1, 127], got {levels}")
    x = x.contiguous()
    _dev.require_cuda(x)
    dim = x.shape[-1]
    rows = x.numel() // dim if dim else 0
    q = torch.empty(x.shape, dtype=torch.int8, device=x.device)
    s = torch.empty(x.shape[:-1], dtype=torch.float32, device=x.device)
    with _dev.on_device(x):
        _lib.call("mxs_quantize_per_token", _dev.dtype_code(x), _dev.ptr(x), rows, dim, levels, _dev.ptr(q),
                  _dev.ptr(s), _dev.stream_handle(stream, x.device))
    _dev.keep_alive(x, stream)
    return q, s


def quantize_per_token(x, levels: int = 127) -> QuantizedMatrix:
    """Symmetric per-token quantisation (maxsim/quant.py:104-120)."""
    data = x.data if isinstance(x, EmbeddingMatrix) or hasattr(x, "rows") else x
    t = _dev.to_device(data)
    if not t.is_floating_point():
        t = t.to(torch.float32)
    if t.dim() != 2:
        raise ShapeMismatch(f"expected 2-D token rows, got shape {tuple(t.shape)}")
    if not 1 <= levels <= 127:
        raise ValueError(f"levels must be in [1, 127], got {levels}")
    q, s = quantize_tensor(t, levels)
    return QuantizedMatrix(q, s, validate=False)


def quantize_corpus(docs, levels: int = 127) -> QuantizedCorpus:
    """Quantise a padded DocBatch / [B, L, d] tensor in one launch (padding rows get scale 1e-12)."""
    data = docs.data if isinstance(docs, DocBatch) else _dev.to_device(docs)
    q, s = quantize_tensor(data, levels)
    return QuantizedCorpus(q, s)


def dequantize(qm: QuantizedMatrix) -> torch.Tensor:
    """scale[t] * q[t] in float32 (maxsim/quant.py:123-125)."""
    return qm.scale[:, None] * qm.q.to(torch.float32)


def score_int8(q_q, q_s, d_q, d_s, valid_lens=None, want_argmax=True, stream=None, *, want_rowmax=False,
               validate=True):
    """Tensor-level batched INT8 forward: q_q [n_q, l_q, d] i8, q_s [n_q, l_q]; d_q [B, L, d], d_s [B, L].

    Returns (scores f64 [n_q, B], argmax or None, rowmax or None) -- see forward.score_dense.
    """
    _dev.require_cuda(q_q, d_q)
    n_q, l_q, dim = q_q.shape
    b, l_pad, d2 = d_q.shape
    if dim != d2:
        raise DimMismatch(int(dim), int(d2))
    if tuple(q_s.shape) != (n_q, l_q) or tuple(d_s.shape) != (b, l_pad):
        raise ShapeMismatch("need exactly one scale per token row")
    dev = d_q.device
    with _dev.on_device(d_q):
        q_q, q_s, d_q, d_s = (t.contiguous() for t in (q_q, q_s, d_q, d_s))
        if valid_lens is not None:
            valid_lens = valid_lens.to(device=dev, dtype=torch.int32).contiguous()
            if valid_lens.numel() != b:
                raise ShapeMismatch(f"valid_lens holds {valid_lens.numel()} entries for {b} documents")
            if validate:
                _dev.validate_lens(valid_lens, l_pad, stream)
        scores = torch.empty((n_q, b), dtype=torch.float64, device=dev)
        argmax = torch.empty((n_q, b, l_q), dtype=torch.int32, device=dev) if want_argmax else None
        rowmax = torch.empty((n_q, b, l_q), dtype=torch.float32, device=dev) if want_rowmax else None
        for t in (q_q, q_s, d_q, d_s, valid_lens):
            _dev.keep_alive(t, stream)
        _lib.call("mxs_fused_score_int8", _dev.ptr(q_q), _dev.ptr(q_s), n_q, l_q, _dev.ptr(d_q), _dev.ptr(d_s), b, l_pad,
                  dim, _dev.ptr(valid_lens), _dev.ptr(scores), _dev.ptr(argmax), _dev.ptr(rowmax),
                  _dev.stream_handle(stream, dev))
    return scores, argmax, rowmax


def fused_score_int8(q_quant: QuantizedMatrix, d_quant: QuantizedMatrix, valid_len: int | None = None,
                     tile: TileConfig = DEFAULT_TILE, report: TrafficReport | None = None):
    """INT8 x INT8 pair score (maxsim/quant.py:128-182) -> (float score, int32 argmax [L_q])."""
    if q_quant.dim != d_quant.dim:
        raise DimMismatch(q_quant.dim, d_quant.dim)
    if valid_len is None:
        valid_len = d_quant.rows
    if valid_len < 1:
        raise EmptyDocument(0)
    if valid_len > d_quant.rows:
        raise ShapeMismatch(f"valid_len {valid_len} exceeds document rows {d_quant.rows}")
    rep = report if report is not None else TrafficReport()
    qm = q_quant if isinstance(q_quant, QuantizedMatrix) else QuantizedMatrix(q_quant.q, q_quant.scale)
    dm = d_quant if isinstance(d_quant, QuantizedMatrix) else QuantizedMatrix(d_quant.q, d_quant.scale)
    vl = torch.tensor([valid_len], dtype=torch.int32, device=dm.q.device)
    scores, argmax, _ = score_int8(qm.q[None], qm.scale[None], dm.q[None], dm.scale[None], vl, validate=False)
    rep.add_read(qm.q.numel() + qm.scale.numel() * 4)
    rep.add_read(dm.rows * (dm.dim + 4))
    rep.add_macs(2 * qm.rows * dm.rows * dm.dim)
    rep.add_write(8)
    return float(scores[0, 0].item()), argmax[0, 0]


def fused_score_int8_batch(q_quant, corpus, valid_lens=None, report: TrafficReport | None = None):
    """Batched INT8 scoring of one or more quantised queries against a QuantizedCorpus.

    q_quant: QuantizedMatrix (one query) or (q [n_q, l_q, d] int8, scales [n_q, l_q]).
    Returns (ScoreMatrix, ArgmaxMap, TrafficReport).
    """
    rep = report if report is not None else TrafficReport()
    if isinstance(q_quant, QuantizedMatrix):
        qq, qs = q_quant.q[None], q_quant.scale[None]
    else:
        qq, qs = _t(q_quant[0], torch.int8), _t(q_quant[1], torch.float32)
    if not isinstance(corpus, QuantizedCorpus):
        corpus = QuantizedCorpus.from_matrices(corpus)
    b, l_pad, dim = corpus.q.shape
    if valid_lens is None:
        lens_host = np.full(b, l_pad, dtype=np.int32)
        vl = None
    else:
        lens_host = np.asarray(valid_lens.cpu() if isinstance(valid_lens, torch.Tensor) else valid_lens, np.int32)
        if (lens_host < 1).any():
            raise EmptyDocument(int(np.argmax(lens_host < 1)))
        vl = torch.from_numpy(lens_host).to(corpus.q.device)
    scores, argmax, _ = score_int8(qq, qs, corpus.q, corpus.scales, vl, validate=False)
    n_q, l_q, _ = qq.shape
    rep.add_read(n_q * l_q * (dim + 4))
    rep.add_read(n_q * b * l_pad * (dim + 4))
    rep.add_macs(2 * n_q * b * l_q * l_pad * dim)
    rep.add_write(8 * n_q * b)
    return ScoreMatrix(scores, validate=False), ArgmaxMap(argmax, lens_host, padded_len=l_pad, validate=False), rep


def _corpus_q_tensors(corpus_q):
    """QuantizedCorpus or a list of QuantizedMatrix (possibly ragged) -> (q, s, valid_lens)."""
    if isinstance(corpus_q, QuantizedCorpus):
        return corpus_q.q, corpus_q.scales, None
    mats = [m if isinstance(m, QuantizedMatrix) else QuantizedMatrix(m.q, m.scale) for m in corpus_q]
    lens = np.array([m.rows for m in mats], np.int32)
    L = int(lens.max())
    dim = mats[0].dim
    dev = mats[0].q.device
    q = torch.zeros((len(mats), L, dim), dtype=torch.int8, device=dev)
    s = torch.ones((len(mats), L), dtype=torch.float32, device=dev)
    for b, m in enumerate(mats):
        q[b, : m.rows] = m.q
        s[b, : m.rows] = m.scale
    return q, s, torch.from_numpy(lens).to(dev)


def two_stage_topk(query, corpus_q, corpus_full: DocBatch, k: int, shortlist_factor: int = 4,
                   tile: TileConfig = DEFAULT_TILE, report: TrafficReport | None = None):
    """Coarse INT8 scan, exact rescoring of a K * shortlist_factor shortlist (maxsim/quant.py:185-231).

    Returns [(doc id, full-precision score)] sorted by score desc, id asc.
    """
    from .forward import as_docbatch, score_dense
    from .topk import topk as device_topk

    if shortlist_factor < 1:
        raise ValueError(f"shortlist_factor must be >= 1, got {shortlist_factor}")
    corpus_full = as_docbatch(corpus_full)
    n_docs = corpus_q.n_docs if isinstance(corpus_q, QuantizedCorpus) else len(corpus_q)
    if corpus_full.n_docs != n_docs:
        raise ShapeMismatch("quantized and full-precision corpora are not aligned")
    if k > n_docs:
        raise KTooLarge(k, n_docs)
    if k == 0:
        return []
    rep = report if report is not None else TrafficReport()
    qm = query if isinstance(query, EmbeddingMatrix) else EmbeddingMatrix(query.data if hasattr(query, "rows") else query)
    qq, qs = quantize_tensor(qm.data)
    dq, ds, vl = _corpus_q_tensors(corpus_q)
    coarse, _, _ = score_int8(qq[None], qs[None], dq, ds, vl, want_argmax=False, validate=False)
    shortlist_n = min(k * shortlist_factor, n_docs)
    _, short_ids = device_topk(coarse[0], shortlist_n)
    short_ids, _ = torch.sort(short_ids)  # shortlist positions in id order: ties rank by lower id
    D = corpus_full.data.index_select(0, short_ids)
    vls = corpus_full.valid_lens.index_select(0, short_ids)
    fine, _, _ = score_dense(qm.data[None].to(D.dtype), D, vls, want_argmax=False, validate=False)
    top_s, top_pos = device_topk(fine[0], k)
    ids = short_ids.index_select(0, top_pos).cpu().tolist()
    rep.add_read(n_docs * dq.shape[1] * (dq.shape[2] + 4))
    return [(int(i), float(s)) for i, s in zip(ids, top_s.cpu().tolist())]
