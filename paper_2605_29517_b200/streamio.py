"""MXS1 embedding files and out-of-core streamed scoring (maxsim/streamio.py:1-395).

* `write_embeddings` writes the reference's little-endian "MXS1" format (header + payload,
  maxsim/streamio.py:57-88) from our device types, reference objects or numpy arrays.
* `CorpusReader` / `read_embeddings` parse it with the native reader of libmaxsim_b200.so
  (`mxs_mxs1_*`, pread straight into caller-owned -- here pinned -- host buffers); the error
  classes are the reference's (BadMagic, VersionUnsupported, TruncatedPayload, IoError).
* `stream_score_topk` scores a corpus that stays on disk (maxsim/streamio.py:265-322): two
  pinned staging buffers and two device buffers; the file read of block i+1 (a worker thread in
  the native reader, GIL released), the H2D copy of block i+1 (copy stream) and the kernels of
  block i (compute stream) overlap.  Every block's scores go through the device top-K and are
  merged into the running device top-K with the reference order (score desc, id asc), so the
  ranking equals exhaustive in-memory ranking, and GPU memory is two blocks + O(K) -- flat in
  corpus size.
"""

from __future__ import annotations

import ctypes
import struct
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .errors import KTooLarge, ShapeMismatch
from .instrument import TrafficReport
from .topk import TopKHeap, select_candidates, topk
from .types import DEFAULT_TILE, DocBatch, EmbeddingMatrix, TileConfig

MAGIC = b"MXS1"
VERSION = 1

_ELEM_CODES = {"f32": 0, "f16": 1, "i8": 2}
_ELEM_NAMES = {v: k for k, v in _ELEM_CODES.items()}
_ELEM_NP = {"f32": "<f4", "f16": "<f2", "i8": "i1"}
_ELEM_SIZE = {"f32": 4, "f16": 2, "i8": 1}
_ELEM_TORCH = {"f32": torch.float32, "f16": torch.float16, "i8": torch.int8}
_LAYOUT_CODES = {"dense": 0, "packed": 1, "quantized": 2}
_LAYOUT_NAMES = {v: k for k, v in _LAYOUT_CODES.items()}

_HEAD = struct.Struct("<4sHBB")
_U64 = struct.Struct("<Q")

__all__ = ["CorpusReader", "TopKHeap", "TrafficModel", "model_traffic", "read_embeddings", "stream_score_topk",
           "write_embeddings"]


# --------------------------------------------------------------------------- writing
def _host(x, dtype=None) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        x = x.detach().cpu().numpy()
    a = np.asarray(x)
    return a if dtype is None else a.astype(dtype)


def _elem_of(obj, elem):
    if elem is not None:
        return elem
    e = getattr(obj, "elem", None)
    if e in _ELEM_CODES:
        return e
    data = getattr(obj, "data", getattr(obj, "tokens", None))
    if isinstance(data, torch.Tensor) and data.dtype == torch.float16:
        return "f16"
    return "f32"


def write_embeddings(path, obj, elem: str | None = None) -> None:
    """Persist embeddings in the MXS1 format; the layout follows the object (maxsim/streamio.py:57).

    DocBatch (fully valid) / EmbeddingMatrix -> dense, PackedCorpus -> packed,
    QuantizedCorpus -> quantized.  Works for this package's device types and the reference's.
    """
    from .errors import IoError

    kind = type(obj).__name__
    if kind == "EmbeddingMatrix":
        data = _host(obj.data, np.float32)[None]
        obj_kind, lens = "dense", None
    elif kind == "DocBatch":
        data = _host(obj.data, np.float32)
        lens = _host(getattr(obj, "valid_lens_host", obj.valid_lens))
        obj_kind = "dense"
    elif kind == "PackedCorpus":
        obj_kind = "packed"
    elif kind == "QuantizedCorpus":
        obj_kind = "quantized"
    else:
        raise ShapeMismatch(f"cannot persist objects of type {kind}")
    try:
        fh = open(path, "wb")
    except OSError as exc:
        raise IoError(f"cannot write {path}: {exc}") from exc
    with fh:
        if obj_kind == "dense":
            tag = _elem_of(obj, elem)
            if tag == "i8":
                raise ShapeMismatch("raw int8 embeddings must use the quantized layout")
            if lens is not None and (np.asarray(lens) != data.shape[1]).any():
                raise ShapeMismatch("ragged batches lose their lengths in the dense layout; pack() them instead")
            fh.write(_HEAD.pack(MAGIC, VERSION, _ELEM_CODES[tag], _LAYOUT_CODES["dense"]))
            for v in data.shape:
                fh.write(_U64.pack(int(v)))
            fh.write(data.astype(_ELEM_NP[tag]).tobytes())
        elif obj_kind == "packed":
            tag = _elem_of(obj, elem)
            if tag == "i8":
                raise ShapeMismatch("raw int8 embeddings must use the quantized layout")
            toks = _host(obj.tokens, np.float32)
            cu = _host(obj.cu_seqlens, np.int64)
            fh.write(_HEAD.pack(MAGIC, VERSION, _ELEM_CODES[tag], _LAYOUT_CODES["packed"]))
            fh.write(_U64.pack(int(cu.size - 1)))
            fh.write(_U64.pack(int(toks.shape[1])))
            fh.write(cu.astype("<u8").tobytes())
            fh.write(toks.astype(_ELEM_NP[tag]).tobytes())
        else:
            q = _host(obj.q, np.int8)
            b, l, d = q.shape
            fh.write(_HEAD.pack(MAGIC, VERSION, _ELEM_CODES["i8"], _LAYOUT_CODES["quantized"]))
            for v in (b, l, d):
                fh.write(_U64.pack(int(v)))
            fh.write(q.tobytes())
            fh.write(_host(obj.scales, np.float32).astype("<f4").tobytes())


# --------------------------------------------------------------------------- reading (native)
class CorpusReader:
    """Block access to an MXS1 file through the native reader (maxsim/streamio.py:166-228).

    Only the header (and, for packed files, the offset table) stays resident.  `read_block_into`
    copies a block's raw elements into any host buffer (pinned for the streaming scorer);
    `read_block` returns it as device-resident DocBatch / PackedCorpus.
    """

    def __init__(self, path, _allow_quantized: bool = False):
        self.path = str(path)
        lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(lib.mxs_mxs1_open(self.path.encode(), ctypes.byref(h)), "")
        self._h = h
        elem, layout = ctypes.c_int32(), ctypes.c_int32()
        n, length, dim = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(lib.mxs_mxs1_info(h, ctypes.byref(elem), ctypes.byref(layout), ctypes.byref(n),
                                     ctypes.byref(length), ctypes.byref(dim)), "mxs_mxs1_info")
        self.elem = _ELEM_NAMES[elem.value]
        self.layout = _LAYOUT_NAMES[layout.value]
        self._n_docs, self.length, self._dim = n.value, length.value, dim.value
        self.cu_seqlens = None
        if self.layout == "packed":
            cu = np.empty(self._n_docs + 1, dtype=np.int64)
            _lib.check(lib.mxs_mxs1_cu_seqlens(h, cu.ctypes.data_as(ctypes.c_void_p)), "mxs_mxs1_cu_seqlens")
            self.cu_seqlens = cu
        if self.layout == "quantized" and not _allow_quantized:
            self.close()
            raise ShapeMismatch("streamed scoring reads dense or packed files; quantized files load whole")

    @property
    def n_docs(self) -> int:
        return int(self._n_docs)

    @property
    def dim(self) -> int:
        return int(self._dim)

    def close(self):
        if self._h is not None:
            _lib.load().mxs_mxs1_close(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def block_bytes(self, first: int, count: int) -> int:
        return int(_lib.load().mxs_mxs1_block_bytes(self._h, first, count))

    def block_shape(self, first: int, count: int):
        count = min(count, self.n_docs - first)
        if self.layout == "packed":
            t0, t1 = int(self.cu_seqlens[first]), int(self.cu_seqlens[first + count])
            return (t1 - t0, self.dim), (self.cu_seqlens[first:first + count + 1] - t0).astype(np.int64)
        return (count, self.length, self.dim), None

    def read_block_into(self, first: int, count: int, dst_ptr: int, dst_bytes: int) -> int:
        """Raw elements of documents [first, first + count) into host memory at dst_ptr."""
        nbytes = self.block_bytes(first, count)
        _lib.check(_lib.load().mxs_mxs1_read_block(self._h, first, count, ctypes.c_void_p(dst_ptr), dst_bytes),
                   "mxs_mxs1_read_block")
        return nbytes

    def read_block_host(self, first: int, count: int):
        """(elements numpy array in the file dtype, relative cu_seqlens or None)."""
        shape, rel = self.block_shape(first, count)
        out = np.empty(shape, dtype=_ELEM_NP[self.elem])
        self.read_block_into(first, count, out.ctypes.data, out.nbytes)
        return out, rel

    def read_block(self, first: int, count: int):
        """Documents [first, first + count) as a device batch (maxsim/streamio.py:209-228)."""
        from .varlen import PackedCorpus

        arr, rel = self.read_block_host(first, count)
        t = torch.from_numpy(arr).to(_dev.device())
        if self.layout == "packed":
            return PackedCorpus(t, rel, elem=self.elem)
        return DocBatch.from_dense(t, elem=self.elem)


def read_embeddings(path):
    """Load a whole file: DocBatch, PackedCorpus or QuantizedCorpus (maxsim/streamio.py:136-163)."""
    from .quant import QuantizedCorpus

    r = CorpusReader(path, _allow_quantized=True)
    try:
        if r.layout == "quantized":
            q = np.empty((r.n_docs, r.length, r.dim), dtype=np.int8)
            r.read_block_into(0, r.n_docs, q.ctypes.data, q.nbytes)
            s = np.empty((r.n_docs, r.length), dtype=np.float32)
            _lib.check(_lib.load().mxs_mxs1_read_scales(r._h, s.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                                        s.nbytes), "mxs_mxs1_read_scales")
            return QuantizedCorpus(q=torch.from_numpy(q).to(_dev.device()), scales=torch.from_numpy(s).to(_dev.device()))
        return r.read_block(0, r.n_docs)
    finally:
        r.close()


# --------------------------------------------------------------------------- streamed scoring
def stream_score_topk(query, corpus, block_docs: int, k: int, tile: TileConfig = DEFAULT_TILE,
                      report: TrafficReport | None = None, compute_dtype=None):
    """Top-K of a corpus too big to hold, streamed from its MXS1 file (maxsim/streamio.py:265).

    Returns (ranked [(doc id, score)], TrafficReport).  `compute_dtype` (e.g. torch.bfloat16)
    casts each block on the device before scoring; by default the file dtype is kept (f32 files
    take the bit-exact fp32 kernel, f16 files the fp16 tensor-core kernel).
    """
    del tile  # results are tile-invariant; the device kernels choose their own tiling
    if block_docs < 1:
        raise ValueError("block_docs must be >= 1")
    own = None
    if not isinstance(corpus, CorpusReader):
        own = CorpusReader(corpus)
        corpus = own
    try:
        return _stream(query, corpus, block_docs, k, report, compute_dtype)
    finally:
        if own is not None:
            own.close()


# Staging buffers (2 pinned host + 2 device) reused across stream_score_topk calls: allocating
# ~GB of pinned memory per call costs more than streaming a small corpus.  One cached set per
# (device, size); a call that finds it in use (concurrent callers) allocates its own.
_STAGING: dict = {}
_STAGING_LOCK = threading.Lock()


def _staging(dev, cap):
    key = (str(dev), int(cap))
    if _STAGING_LOCK.acquire(blocking=False):
        bufs = _STAGING.get(key)
        if bufs is None:
            _STAGING.clear()
            bufs = ([torch.empty(cap, dtype=torch.uint8, pin_memory=True) for _ in range(2)],
                    [torch.empty(cap, dtype=torch.uint8, device=dev) for _ in range(2)])
            _STAGING[key] = bufs
        return bufs, _STAGING_LOCK.release
    return ([torch.empty(cap, dtype=torch.uint8, pin_memory=True) for _ in range(2)],
            [torch.empty(cap, dtype=torch.uint8, device=dev) for _ in range(2)]), (lambda: None)


def _stream(query, reader: CorpusReader, block_docs: int, k: int, report, compute_dtype):
    from .varlen import score_varlen
    from .forward import score_dense

    n_docs = reader.n_docs
    if n_docs == 0:
        raise ShapeMismatch("corpus is empty")
    if k > n_docs:
        raise KTooLarge(k, n_docs)
    rep = report if report is not None else TrafficReport()
    dev = _dev.device()
    if isinstance(query, (torch.Tensor, np.ndarray)):
        q_src = query
    else:  # EmbeddingMatrix (ours or the reference's)
        q_src = query.data
    q = torch.as_tensor(np.asarray(q_src) if not isinstance(q_src, torch.Tensor) else q_src).to(dev)
    if q.dim() == 2:
        q = q[None]
    if q.shape[-1] != reader.dim:
        from .errors import DimMismatch

        raise DimMismatch(int(q.shape[-1]), reader.dim)
    file_dtype = _ELEM_TORCH[reader.elem]
    work_dtype = compute_dtype or file_dtype
    exact = work_dtype == torch.float32
    q = q.to(work_dtype).contiguous()
    blocks = [(f, min(block_docs, n_docs - f)) for f in range(0, n_docs, block_docs)]
    cap = max(reader.block_bytes(f, c) for f, c in blocks)
    (host, devb), release_staging = _staging(dev, cap)
    h2d_done = [None, None]
    dev_free = [None, None]
    copy_stream = torch.cuda.Stream(device=dev)
    comp = torch.cuda.current_stream(dev)
    run_s = run_i = None
    es = _ELEM_SIZE[reader.elem]
    rep.add_read(q.numel() * es)
    pool = ThreadPoolExecutor(max_workers=1)

    def load(i):
        f, c = blocks[i]
        return reader.read_block_into(f, c, host[i % 2].data_ptr(), cap)

    try:
        fut = pool.submit(load, 0)
        for i, (first, count) in enumerate(blocks):
            nbytes = fut.result()
            slot = i % 2
            # H2D of block i on the copy stream once its device buffer is free
            with torch.cuda.stream(copy_stream):
                if dev_free[slot] is not None:
                    copy_stream.wait_event(dev_free[slot])
                devb[slot][:nbytes].copy_(host[slot][:nbytes], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy_stream)
                h2d_done[slot] = ev
            if i + 1 < len(blocks):
                # the other staging buffer is reused once its own copy (block i-1) finished
                if h2d_done[1 - slot] is not None:
                    h2d_done[1 - slot].synchronize()
                fut = pool.submit(load, i + 1)
            comp.wait_event(h2d_done[slot])
            rep.alloc(nbytes)
            shape, rel = reader.block_shape(first, count)
            raw = devb[slot][:nbytes].view(file_dtype).view(*shape)
            data = raw if work_dtype == file_dtype else raw.to(work_dtype)
            if reader.layout == "packed":
                cu = torch.from_numpy(rel).to(dev, non_blocking=True)
                s, _, _ = score_varlen(q, data, cu, want_argmax=False, exact=exact, validate=False)
            else:
                s, _, _ = score_dense(q, data, exact=exact, want_argmax=False)
            rep.add_read(nbytes)
            rep.add_write(8 * count * q.shape[0])
            rep.add_macs(2 * q.shape[0] * q.shape[1] * (shape[0] if reader.layout == "packed" else count * shape[1])
                         * reader.dim)
            bs, bi = topk(s[0], min(k, count), id_offset=first)
            if run_s is None:
                run_s, run_i = bs, bi
            else:
                run_s, run_i = select_candidates(torch.cat([run_s, bs]), torch.cat([run_i, bi]), min(k, run_s.numel()
                                                                                                    + bs.numel()))
            ev_free = torch.cuda.Event()
            ev_free.record(comp)
            dev_free[slot] = ev_free
            rep.release(nbytes)
        ids = run_i.cpu().tolist()
        vals = run_s.cpu().tolist()
        return [(int(a), float(b)) for a, b in zip(ids, vals)][:k], rep
    finally:
        pool.shutdown(wait=True)
        torch.cuda.current_stream(dev).synchronize()  # staging buffers are idle before reuse
        release_staging()


def stream_score_host(query, docs_host: torch.Tensor, k: int, block_docs: int = 1000, valid_lens=None,
                      compute_dtype=None, want_scores: bool = True):
    """Score a corpus resident in (pinned) HOST memory: block i+1 is copied to the device on a
    copy stream while block i is scored, so the step costs ~max(H2D, compute) instead of their sum.

    docs_host [B, L, d] CPU tensor (pin it for overlap); returns (scores f64 [B] on the device or
    None, top_s f64 [k], top_id int64 [k]) -- ranking in the reference order (score desc, id asc).
    """
    from .forward import score_dense

    if docs_host.is_cuda:
        raise ShapeMismatch("stream_score_host expects host-resident documents")
    n_docs = int(docs_host.shape[0])
    if k > n_docs:
        raise KTooLarge(k, n_docs)
    dev = _dev.device()
    q = query if isinstance(query, torch.Tensor) else torch.as_tensor(np.asarray(getattr(query, "data", query)))
    q = q.to(dev)
    if q.dim() == 2:
        q = q[None]
    work_dtype = compute_dtype or docs_host.dtype
    q = q.to(work_dtype).contiguous()
    vl = None if valid_lens is None else torch.as_tensor(valid_lens).to(dev, torch.int32)
    blocks = [(f, min(block_docs, n_docs - f)) for f in range(0, n_docs, block_docs)]
    devb = [torch.empty((block_docs,) + tuple(docs_host.shape[1:]), dtype=docs_host.dtype, device=dev)
            for _ in range(2)]
    copy_stream = torch.cuda.Stream(device=dev)
    comp = torch.cuda.current_stream(dev)
    scores = torch.empty(n_docs, dtype=torch.float64, device=dev) if want_scores else None
    dev_free = [None, None]
    run_s = run_i = None
    h2d = [None] * len(blocks)

    def enqueue_copy(i):
        first, count = blocks[i]
        slot = i % 2
        with torch.cuda.stream(copy_stream):
            if dev_free[slot] is not None:  # the block that last used this buffer was scored
                copy_stream.wait_event(dev_free[slot])
            devb[slot][:count].copy_(docs_host[first:first + count], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy_stream)
            h2d[i] = ev

    enqueue_copy(0)
    for i, (first, count) in enumerate(blocks):
        slot = i % 2
        if i + 1 < len(blocks):
            enqueue_copy(i + 1)  # overlaps the scoring of block i
        comp.wait_event(h2d[i])
        data = devb[slot][:count]
        if work_dtype != data.dtype:
            data = data.to(work_dtype)
        s, _, _ = score_dense(q, data, None if vl is None else vl[first:first + count], want_argmax=False,
                              validate=False)
        if scores is not None:
            scores[first:first + count].copy_(s[0])
        bs, bi = topk(s[0], min(k, count), id_offset=first)
        if run_s is None:
            run_s, run_i = bs, bi
        else:
            run_s, run_i = select_candidates(torch.cat([run_s, bs]), torch.cat([run_i, bi]),
                                             min(k, run_s.numel() + bs.numel()))
        ev_free = torch.cuda.Event()
        ev_free.record(comp)
        dev_free[slot] = ev_free
    return scores, run_s[:k], run_i[:k]


# --------------------------------------------------------------------------- byte model
@dataclass(frozen=True)
class TrafficModel:
    """Predicted main-memory bytes for one scoring workload (maxsim/streamio.py:325-363)."""

    fused_read: int
    fused_write: int
    naive_read: int
    naive_write: int
    s_to_operand_ratio: float

    @property
    def fused_total(self) -> int:
        return self.fused_read + self.fused_write

    @property
    def naive_total(self) -> int:
        return self.naive_read + self.naive_write

    @property
    def naive_over_fused(self) -> float:
        return self.naive_total / self.fused_total

    def bytes(self, mode: str) -> int:
        if mode == "fused":
            return self.fused_total
        if mode == "naive":
            return self.naive_total
        raise ValueError(f"unknown mode {mode!r}")


def model_traffic(n_queries: int, n_docs: int, len_q: int, len_d: int, dim: int, elem_bytes: int = 4,
                  scalar_bytes: int = 8) -> TrafficModel:
    """Analytic byte model (maxsim/streamio.py:366-395); the fused counts are the roofline
    numerators the benchmarks divide by measured kernel time."""
    for v in (n_queries, n_docs, len_q, len_d, dim):
        if v < 1:
            raise ValueError("model_traffic expects positive shape values")
    q_bytes = n_queries * len_q * dim * elem_bytes
    d_bytes = n_queries * n_docs * len_d * dim * elem_bytes
    s_elems = n_queries * n_docs * len_q * len_d
    out_bytes = n_queries * n_docs * scalar_bytes
    return TrafficModel(
        fused_read=q_bytes + d_bytes,
        fused_write=out_bytes,
        naive_read=q_bytes + d_bytes + 2 * s_elems * elem_bytes,
        naive_write=s_elems * elem_bytes + out_bytes,
        s_to_operand_ratio=(len_q * len_d) / ((len_q + len_d) * dim),
    )
