"""Corpus / in-batch sharding across the GPUs of one node.

One process per GPU over torch.distributed.  The data path has no collective: each rank
scores its own contiguous document shard.  NCCL carries exactly three things:
  * rerank  : all_gather of each rank's K (score, global id) candidates -> identical global
              top-K (score desc, id asc) on every rank (k * 16 B per rank);
  * training: all_gather of the [N_q, B/W] local score blocks for the in-batch loss, and the
              all_reduce(sum) of the dQ partials (Q is replicated, dD stays shard-local).
Shards are balanced by token count (`shard_bounds`), so the varlen corpus splits evenly.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from .topk import merge_topk_across_ranks, topk


def shard_bounds(n_docs: int, world: int, rank: int, weights=None):
    """Contiguous [lo, hi) document range of `rank`, balanced by `weights` (doc lengths) if given."""
    if weights is None:
        lo = (n_docs * rank) // world
        hi = (n_docs * (rank + 1)) // world
        return lo, hi
    w = np.asarray(weights, dtype=np.int64)
    cum = np.concatenate([[0], np.cumsum(w)])
    total = cum[-1]
    lo = int(np.searchsorted(cum, total * rank / world, side="left"))
    hi = int(np.searchsorted(cum, total * (rank + 1) / world, side="left")) if rank + 1 < world else n_docs
    return min(lo, n_docs), min(hi, n_docs)


def sharded_topk(local_scores: torch.Tensor, k: int, doc_offset: int, group=None, select=None):
    """Global top-K of a doc-sharded score vector: device top-K per rank, then one all_gather."""
    kk = min(k, local_scores.numel())
    ts, ti = topk(local_scores, kk, id_offset=doc_offset)
    if kk < k:  # pad so every rank contributes k slots
        pad = k - kk
        ts = torch.cat([ts, torch.full((pad,), float("-inf"), dtype=ts.dtype, device=ts.device)])
        ti = torch.cat([ti, torch.full((pad,), -1, dtype=ti.dtype, device=ti.device)])
    return merge_topk_across_ranks(ts, ti, k, group=group, select=select)


def softmax_ce_device(scores: torch.Tensor, col0: int, ncols: int):
    """`softmax_ce` fused into one kernel (mxs_softmax_ce): returns (loss f64 0-d tensor, g f32
    [n_q, ncols] = columns [col0, col0 + ncols) of the score gradient), on the scores' device."""
    from . import _dev, _lib

    s = scores.to(torch.float64).contiguous()
    n_q, b = s.shape
    loss = torch.empty((), dtype=torch.float64, device=s.device)
    g = torch.empty((n_q, ncols), dtype=torch.float32, device=s.device)
    with _dev.on_device(s):
        _lib.call("mxs_softmax_ce", _dev.ptr(s), n_q, b, col0, ncols, _dev.ptr(loss), _dev.ptr(g),
                  _dev.stream_handle(None, s.device))
    return loss, g


def softmax_ce(scores: torch.Tensor):
    """In-batch contrastive loss with positives on the diagonal (maxsim/cli.py:198-206), float64."""
    s = scores.to(torch.float64)
    b = s.shape[0]
    mx = s.max(dim=1, keepdim=True).values
    lse = torch.log(torch.exp(s - mx).sum(dim=1)) + mx[:, 0]
    loss = torch.mean(lse - torch.diagonal(s))
    probs = torch.exp(s - lse[:, None])
    grad = (probs - torch.eye(b, dtype=s.dtype, device=s.device)) / b
    return loss, grad


_OFFSETS = {}


def _doc_offsets(b_local: int, l_pad: int, device):
    """Cached (row offset, length) tensors of b_local equal-length documents (read-only; saves the
    arange / full launches of every step)."""
    key = (b_local, l_pad, torch.device(device))
    if key not in _OFFSETS:
        off = torch.arange(b_local, dtype=torch.int64, device=device) * l_pad
        _OFFSETS[key] = (off, torch.full((b_local,), l_pad, dtype=torch.int64, device=device))
    return _OFFSETS[key]


class DeviceKernels:
    """The sm_100a kernels used by inbatch_step (tests substitute an oracle-backed twin)."""

    @staticmethod
    def score(Q, D, valid_lens):
        from .forward import score_dense

        scores, argmax, _ = score_dense(Q, D, valid_lens)
        return scores, argmax

    @staticmethod
    def grad_docs(Q, argmax, g, l_pad):
        from .autograd import _grad_docs

        b_local = argmax.shape[1]
        off, lens = _doc_offsets(b_local, l_pad, Q.device)
        return _grad_docs(Q, argmax, g, off, lens, b_local * l_pad, l_pad, Q.shape[-1])

    @staticmethod
    def grad_query(D, argmax, g):
        from .autograd import _grad_query

        b_local, l_pad, dim = D.shape
        off, _ = _doc_offsets(b_local, l_pad, D.device)
        return _grad_query(D.reshape(b_local * l_pad, dim).contiguous(), off, argmax, g, dim)

    @staticmethod
    def csr(argmax, l_pad):
        """The inverse CSR of the saved argmax alone (K6), so it can run beside the loss and dQ."""
        from .backward import csr_tensors

        b_local = argmax.shape[1]
        off, lens = _doc_offsets(b_local, l_pad, argmax.device)
        row_ptr, col_idx, _ = csr_tensors(argmax, off, lens, b_local * l_pad, l_pad)
        return row_ptr, col_idx

    @staticmethod
    def grad_docs_csr(Q, argmax, g, csr, l_pad):
        """dD from a prebuilt CSR (K7)."""
        from .autograd import _grad_docs_from_csr

        return _grad_docs_from_csr(Q, argmax, g, csr, argmax.shape[1] * l_pad, Q.shape[-1])


def inbatch_step(Q: torch.Tensor, D_local: torch.Tensor, doc_offset: int, group=None, valid_lens=None,
                 kernels=DeviceKernels):
    """One in-batch-negatives training step with B sharded over ranks (C3 at N GPUs).

    Q [N_q, L_q, d] replicated; D_local [B/W, L, d] this rank's documents starting at global
    doc `doc_offset`.  Returns (loss, scores [N_q, B], dQ [N_q, L_q, d] fp32 all-reduced,
    dD_local [B/W, L, d] fp32).  Collectives: one all_gather of the local score blocks, one
    all_reduce(sum) of dQ issued asynchronously and overlapped with the dD kernel; dD never
    leaves its rank.
    """
    import torch.distributed as dist

    scores_local, argmax = kernels.score(Q, D_local, valid_lens)
    b_local, l_pad, dim = D_local.shape
    # the inverse CSR needs only the argmax: build it on a side stream while the loss and dQ run
    # (a latency-bound kernel next to two bandwidth-bound ones)
    csr = None
    if hasattr(kernels, "csr") and argmax.is_cuda and os.environ.get("MXS_C3_OVERLAP", "1") != "0":
        from .autograd import _side_stream

        main, side = torch.cuda.current_stream(argmax.device), _side_stream(argmax.device)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            csr = kernels.csr(argmax, l_pad)
        argmax.record_stream(side)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world > 1:
        parts = [torch.empty_like(scores_local) for _ in range(world)]
        dist.all_gather(parts, scores_local.contiguous(), group=group)
        scores = torch.cat(parts, dim=1)
    else:
        scores = scores_local
    if scores.is_cuda and hasattr(kernels, "csr"):  # device kernels: one fused loss launch
        loss, g = softmax_ce_device(scores, doc_offset, b_local)
    else:
        loss, g_full = softmax_ce(scores)
        g = g_full[:, doc_offset : doc_offset + b_local].to(torch.float32).contiguous()
    dD = None
    if csr is not None and os.environ.get("MXS_C3_CONCURRENT", "1") != "0":
        # dD on the side stream right behind its CSR, concurrent with dQ on the main stream: the
        # two L2 gathers share the GPU instead of each paying its own tail
        side.wait_stream(main)  # g (the loss) is ready
        with torch.cuda.stream(side):
            dD = kernels.grad_docs_csr(Q.to(D_local.dtype).contiguous(), argmax, g, csr, l_pad)
        g.record_stream(side)
        Q.record_stream(side)
    # dQ first: its all_reduce (NCCL, async) crosses NVLink while the dD gather kernel runs
    dQ = kernels.grad_query(D_local, argmax, g)
    work = dist.all_reduce(dQ, group=group, async_op=True) if world > 1 else None
    if dD is not None:
        main.wait_stream(side)
        dD.record_stream(main)
    elif csr is not None:
        main.wait_stream(side)
        for t in csr:
            t.record_stream(main)
        dD = kernels.grad_docs_csr(Q.to(D_local.dtype).contiguous(), argmax, g, csr, l_pad)
    else:
        dD = kernels.grad_docs(Q.to(D_local.dtype).contiguous(), argmax, g, l_pad)
    if work is not None:
        work.wait()
    return loss, scores, dQ, dD.reshape(b_local, l_pad, dim)


class InBatchStepGraph:
    """`inbatch_step` captured once into a CUDA graph and replayed (single process).

    A training loop updates Q and D in place between steps; the graph reads those same buffers,
    so every replay is one launch of the whole step (forward kernel, f64 score fold, loss,
    device CSR, the two gather kernels) with no per-kernel host launch cost.  Outputs are the
    graph's static tensors (copy them if they must survive the next replay).
    """

    def __init__(self, Q: torch.Tensor, D: torch.Tensor, warmup: int = 2):
        import torch.distributed as dist

        if dist.is_initialized() and dist.get_world_size() > 1:
            raise ValueError("InBatchStepGraph is the single-GPU step; use inbatch_step across ranks")
        self.Q, self.D = Q, D
        side = torch.cuda.Stream(device=Q.device)
        side.wait_stream(torch.cuda.current_stream(Q.device))
        with torch.cuda.stream(side):
            for _ in range(warmup):  # allocator warm-up outside the capture
                inbatch_step(Q, D, 0)
        torch.cuda.current_stream(Q.device).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.out = inbatch_step(Q, D, 0)

    def __call__(self):
        """Replay: returns (loss, scores, dQ, dD) -- the graph's static output tensors."""
        self.graph.replay()
        return self.out


class ShardedInBatchStepGraph:
    """`inbatch_step` with B sharded over ranks, as CUDA graphs around EAGER collectives.

    The local work is captured in three graphs -- G1: forward (scores + argmax); G2: loss, score
    gradient, inverse CSR (side stream) and dQ; G3: dD -- and the two NCCL collectives run eagerly
    between replays on static buffers (nothing collective is captured): the score all_gather
    between G1 and G2, and the dQ all_reduce issued asynchronously right after G2 so that it
    crosses NVLink while G3 (dD) runs.  A step is then 3 graph launches + 2 collectives instead
    of ~20 kernel launches from Python.  With world == 1 the collectives are skipped and the
    result equals `inbatch_step` (tests/test_gpu_parity.py).  Q / D_local are read in place.
    """

    def __init__(self, Q: torch.Tensor, D_local: torch.Tensor, doc_offset: int, group=None, warmup: int = 2):
        import torch.distributed as dist

        from .autograd import _side_stream

        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.Q, self.D = Q, D_local
        self.doc_offset = doc_offset
        k = DeviceKernels
        b_local, l_pad, dim = D_local.shape
        n_q = Q.shape[0]
        dev = Q.device
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(warmup):  # allocator warm-up (and the cached offsets) outside the captures
                inbatch_step(Q, D_local, 0 if self.world == 1 else doc_offset, group)
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self.scores_full = torch.empty((n_q, b_local * self.world), dtype=torch.float64, device=dev)
        self.gathered = torch.empty((self.world, n_q, b_local), dtype=torch.float64, device=dev)
        self.g1, self.g2, self.g3 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g1):
            self.scores_local, self.argmax = k.score(Q, D_local, None)
        with torch.cuda.graph(self.g2):
            if self.world > 1:  # the all-gathered [world, n_q, b_local] blocks -> [n_q, B]
                self.scores_full.copy_(self.gathered.permute(1, 0, 2).reshape(n_q, -1))
            else:
                self.scores_full.copy_(self.scores_local)
            main, sidec = torch.cuda.current_stream(dev), _side_stream(dev)
            sidec.wait_stream(main)
            with torch.cuda.stream(sidec):
                self.csr = k.csr(self.argmax, l_pad)
            self.loss, self.g = softmax_ce_device(self.scores_full, doc_offset if self.world > 1 else 0, b_local)
            self.dQ = k.grad_query(D_local, self.argmax, self.g)
            main.wait_stream(sidec)
        with torch.cuda.graph(self.g3):
            self.dD = k.grad_docs_csr(Q.to(D_local.dtype).contiguous(), self.argmax, self.g, self.csr,
                                      l_pad).reshape(b_local, l_pad, dim)

    def __call__(self):
        """One step: returns (loss, scores [N_q, B], dQ all-reduced, dD_local) -- static tensors."""
        import torch.distributed as dist

        self.g1.replay()
        if self.world > 1:
            dist.all_gather(list(self.gathered.unbind(0)), self.scores_local.contiguous(), group=self.group)
        self.g2.replay()
        work = dist.all_reduce(self.dQ, group=self.group, async_op=True) if self.world > 1 else None
        self.g3.replay()
        if work is not None:
            work.wait()
        return self.loss, self.scores_full, self.dQ, self.dD
