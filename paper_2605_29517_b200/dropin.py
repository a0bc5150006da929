"""Drop-in binding for an existing `maxsim` installation (the reference package).

`install(maxsim)` rebinds the reference's hot-path entry points -- the forward scorers
(maxsim/forward.py:158 fused_score_pair, :221 fused_score_batch), the backward
(maxsim/backward.py:81 build_inverse_csr, :135 grad_docs_csr, :176 grad_docs_scatter, :218
grad_query, :258 backward_dispatch), INT8 (maxsim/quant.py:104 quantize_per_token, :128
fused_score_int8, :185 two_stage_topk), varlen (maxsim/varlen.py:88 fused_score_varlen) and
Chamfer (maxsim/chamfer.py:81 chamfer_forward, :153 chamfer_backward) -- to adapters that run
this package's sm_100a kernels and hand back the REFERENCE's own result types (numpy-backed
ScoreMatrix / ArgmaxMap / CsrInverse / QuantizedMatrix, float scores, numpy gradients).  The
reference's types, validation helpers, dense brute-force module, synth generators, streaming and
CLI stay the reference's; everything they call for scoring now runs on the GPU.  This is the
binding a maintainer adds to switch an application (or the reference's own test-suite) over:

    import maxsim, paper_2605_29517_b200.dropin as dropin
    dropin.install(maxsim)

Contract differences the adapters do not hide: bf16/fp16 inputs run on the tensor
cores (scores within 1e-3 of the fp32 oracle); gradients accumulate in fp32 (north_star: 1e-3
relative) where the reference accumulates float64 on float32 inputs; TileConfig is accepted and
ignored (the kernels choose their own tiling; results are tile-invariant).
"""

from __future__ import annotations

import functools
import sys

import numpy as np
import torch

from . import backward as _bw
from . import chamfer as _ch
from . import forward as _fw
from . import quant as _qt
from . import varlen as _vl

_INSTALLED = "_paper_2605_29517_b200_dropin"


def _np(x):
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    if hasattr(x, "numpy") and not isinstance(x, np.ndarray):
        return np.asarray(x.numpy())
    return np.asarray(x)


def _ref_argmax(ref, am):
    """Our ArgmaxMap -> the reference's (host int32 indices, doc lengths, padded_len)."""
    return ref.ArgmaxMap(_np(am.indices).astype(np.int32), np.asarray(am.doc_lens), padded_len=am.padded_len)


def _translating(ref, fn):
    """Re-raise this package's errors as the reference's classes of the same name (same message
    and fields), so `except maxsim.EmptyDocument` keeps working after the switch."""
    from . import errors as ours

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        except ours.MaxSimError as exc:
            cls = getattr(ref.errors, type(exc).__name__, None)
            if cls is None or not isinstance(cls, type):
                raise
            new = cls.__new__(cls)
            new.__dict__.update(getattr(exc, "__dict__", {}))
            new.args = exc.args
            raise new from exc

    return wrapped


def install(ref) -> None:
    """Rebind `ref` (an imported reference `maxsim` package) to the GPU kernels, idempotently."""
    if getattr(ref, _INSTALLED, False):
        return
    fwd, bwd, quant, varlen, chamfer = ref.forward, ref.backward, ref.quant, ref.varlen, ref.chamfer

    @functools.wraps(fwd.fused_score_pair)
    def fused_score_pair(query, doc, valid_len=None, tile=ref.DEFAULT_TILE, report=None):
        rep = report if report is not None else ref.TrafficReport()
        score, arg, _ = _fw.fused_score_pair(query, doc, valid_len=valid_len, tile=tile, report=rep)
        return float(score), _np(arg).astype(np.int32), rep

    @functools.wraps(fwd.fused_score_batch)
    def fused_score_batch(queries, docs, tile=ref.DEFAULT_TILE, report=None, threads=1, count_query=True):
        rep = report if report is not None else ref.TrafficReport()
        sc, am, _ = _fw.fused_score_batch(queries, docs, tile=tile, report=rep, threads=threads,
                                          count_query=count_query)
        return ref.ScoreMatrix(_np(sc)), _ref_argmax(ref, am), rep

    @functools.wraps(bwd.build_inverse_csr)
    def build_inverse_csr(argmax, report=None):
        csr = _bw.build_inverse_csr(argmax, report=report)
        rp, ci = csr.to_numpy()
        return bwd.CsrInverse(row_ptr=rp, col_idx=ci, n_dest=csr.n_dest, src_shape=tuple(csr.src_shape),
                              padded_len=csr.padded_len)

    def _our_csr(csr):
        return _bw.CsrInverse(row_ptr=torch.as_tensor(np.asarray(csr.row_ptr, np.int32)).cuda(),
                              col_idx=torch.as_tensor(np.asarray(csr.col_idx, np.int32)).cuda(),
                              n_dest=int(csr.n_dest), src_shape=tuple(csr.src_shape), padded_len=csr.padded_len)

    @functools.wraps(bwd.grad_docs_csr)
    def grad_docs_csr(csr, upstream, queries, report=None, out=None):
        c = _our_csr(csr) if not isinstance(csr, _bw.CsrInverse) else csr
        flat = _np(_bw.grad_docs_csr(c, upstream, queries, report=report)).astype(np.float64)
        if out is None:
            return flat
        out[...] = flat  # one store per destination row (the rows were each stored once on the device)
        return out

    @functools.wraps(bwd.grad_docs_scatter)
    def grad_docs_scatter(argmax, upstream, queries, report=None):
        return _np(_bw.grad_docs_scatter(argmax, upstream, queries, report=report)).astype(np.float64)

    @functools.wraps(bwd.grad_query)
    def grad_query(argmax, upstream, docs):
        return _np(_bw.grad_query(argmax, upstream, docs)).astype(np.float64)

    @functools.wraps(bwd.backward_dispatch)
    def backward_dispatch(argmax, upstream, queries, docs, threshold=bwd.DEFAULT_SCATTER_THRESHOLD, report=None):
        dq, dd = _bw.backward_dispatch(argmax, upstream, queries, docs, threshold=threshold, report=report)
        return _np(dq).astype(np.float64), _np(dd).astype(np.float64)

    @functools.wraps(quant.quantize_per_token)
    def quantize_per_token(x, levels=127):
        qm = _qt.quantize_per_token(x, levels=levels)
        return quant.QuantizedMatrix(q=_np(qm.q).astype(np.int8), scale=_np(qm.scale).astype(np.float32))

    @functools.wraps(quant.fused_score_int8)
    def fused_score_int8(q_quant, d_quant, valid_len=None, tile=ref.DEFAULT_TILE, report=None):
        score, arg = _qt.fused_score_int8(q_quant, d_quant, valid_len=valid_len, tile=tile, report=report)
        return float(score), _np(arg).astype(np.int32)

    @functools.wraps(quant.two_stage_topk)
    def two_stage_topk(query, corpus_q, corpus_full, k, shortlist_factor=4, tile=ref.DEFAULT_TILE, report=None):
        return _qt.two_stage_topk(query, corpus_q, corpus_full, k, shortlist_factor=shortlist_factor, tile=tile,
                                  report=report)

    @functools.wraps(varlen.fused_score_varlen)
    def fused_score_varlen(query, packed, tile=ref.DEFAULT_TILE, report=None, count_query=True):
        rep = report if report is not None else ref.TrafficReport()
        s, am, _ = _vl.fused_score_varlen(query, packed, tile=tile, report=rep, count_query=count_query)
        return _np(s).astype(np.float64), _ref_argmax(ref, am), rep

    @functools.wraps(chamfer.chamfer_forward)
    def chamfer_forward(p_set, s_set, tile=ref.DEFAULT_TILE, report=None):
        cd, a1, a2 = _ch.chamfer_forward(p_set, s_set, tile=tile, report=report)
        return float(cd), _np(a1).astype(np.int64), _np(a2).astype(np.int64)

    @functools.wraps(chamfer.chamfer_backward)
    def chamfer_backward(p_set, s_set, argmin_ps, argmin_sp, upstream=1.0, report=None):
        # the inversions go through the reference module's build_inverse_csr attribute, looked up at
        # call time (maxsim/chamfer.py:153-199 shares the one builder; after install() it is ours)
        d_p, d_s = _ch.chamfer_backward(p_set, s_set, argmin_ps, argmin_sp, upstream=upstream, report=report,
                                        csr_builder=lambda am: chamfer.build_inverse_csr(am))
        return _np(d_p), _np(d_s)

    table = {
        fwd: {"fused_score_pair": fused_score_pair, "fused_score_batch": fused_score_batch},
        bwd: {"build_inverse_csr": build_inverse_csr, "grad_docs_csr": grad_docs_csr,
              "grad_docs_scatter": grad_docs_scatter, "grad_query": grad_query,
              "backward_dispatch": backward_dispatch},
        quant: {"quantize_per_token": quantize_per_token, "fused_score_int8": fused_score_int8,
                "two_stage_topk": two_stage_topk},
        varlen: {"fused_score_varlen": fused_score_varlen},
        chamfer: {"chamfer_forward": chamfer_forward, "chamfer_backward": chamfer_backward},
    }
    # every module of the package that bound an original at import time (maxsim/__init__.py,
    # chamfer's `from .backward import build_inverse_csr`, the CLI ...) gets the GPU version too
    replace = {}
    for mod, fns in table.items():
        for name, fn in fns.items():
            replace[id(getattr(mod, name))] = _translating(ref, fn)
    prefix = ref.__name__ + "."
    for mname, mod in list(sys.modules.items()):
        if mod is None or not (mname == ref.__name__ or mname.startswith(prefix)):
            continue
        for attr, val in list(vars(mod).items()):
            if callable(val) and id(val) in replace:
                setattr(mod, attr, replace[id(val)])
    setattr(ref, _INSTALLED, True)
