"""Top-K ranking with the reference tie rule: score descending, document id ascending.

* `TopKHeap` mirrors maxsim/streamio.py:230-262 on the host (small, streaming merges).
* `topk` runs the device selection kernel (K9) over an f64 score vector.
* `merge_topk_across_ranks` all-gathers each rank's (score, global id) candidates over
  torch.distributed (NCCL) and re-selects them on the device with the same ordering, so a
  sharded corpus ranks exactly like the unsharded one.
"""

from __future__ import annotations

import heapq

import torch

from . import _dev, _lib
from .errors import KTooLarge


class TopKHeap:
    """Bounded min-heap keeping the K best (doc id, score) pairs (maxsim/streamio.py:230-262)."""

    __slots__ = ("capacity", "_heap")

    def __init__(self, capacity: int):
        if capacity < 0:
            raise ValueError("capacity must be >= 0")
        self.capacity = capacity
        self._heap = []

    def __len__(self):
        return len(self._heap)

    def offer(self, doc_id: int, score: float) -> None:
        if self.capacity == 0:
            return
        key = (float(score), -int(doc_id))
        if len(self._heap) < self.capacity:
            heapq.heappush(self._heap, key)
        elif key > self._heap[0]:
            heapq.heapreplace(self._heap, key)

    def offer_many(self, ids, scores) -> None:
        for i, s in zip(ids, scores):
            self.offer(int(i), float(s))

    def merge(self, other: "TopKHeap") -> None:
        for score, neg_id in other._heap:
            self.offer(-neg_id, score)

    def ranked(self):
        return [(-neg_id, score) for score, neg_id in sorted(self._heap, key=lambda t: (-t[0], -t[1]))]


def topk(scores: torch.Tensor, k: int, id_offset: int = 0, stream=None):
    """Device top-K of a 1-D f64 score vector -> (top_s f64 [k], top_id int64 [k]) on the device."""
    s = scores.reshape(-1).to(torch.float64).contiguous()
    _dev.require_cuda(s)
    n = s.numel()
    if k > n:
        raise KTooLarge(k, n)
    top_s = torch.empty(k, dtype=torch.float64, device=s.device)
    top_id = torch.empty(k, dtype=torch.int64, device=s.device)
    if k == 0:
        return top_s, top_id
    ws_bytes = int(_lib.load().mxs_topk_workspace_bytes(n, k))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=s.device)
    with _dev.on_device(s):
        _lib.call("mxs_topk", _dev.ptr(s), n, k, id_offset, _dev.ptr(top_s), _dev.ptr(top_id), _dev.ptr(ws), ws_bytes,
                  _dev.stream_handle(stream, s.device))
    for t in (s, ws):
        _dev.keep_alive(t, stream)
    return top_s, top_id


def ranked(scores, k: int | None = None):
    """[[id, score], ...] in reference order (maxsim/cli.py:88-92 _ranked)."""
    s = scores if isinstance(scores, torch.Tensor) else torch.as_tensor(scores)
    s = _dev.to_device(s.reshape(-1), torch.float64)
    kk = s.numel() if k is None else k
    ts, ti = topk(s, kk)
    return [[int(i), float(v)] for i, v in zip(ti.cpu().tolist(), ts.cpu().tolist())]


def select_candidates(scores: torch.Tensor, ids: torch.Tensor, k: int, stream=None):
    """Top-K among (score, id) candidates with explicit ids (ids < 0 are empty slots): one
    single-block selection kernel on the device (no host path)."""
    s = scores.reshape(-1).to(torch.float64).contiguous()
    i = ids.reshape(-1).to(torch.int64).contiguous()
    _dev.require_cuda(s, i)
    top_s = torch.empty(k, dtype=torch.float64, device=s.device)
    top_i = torch.empty(k, dtype=torch.int64, device=s.device)
    with _dev.on_device(s):
        _lib.call("mxs_topk_candidates", _dev.ptr(s), _dev.ptr(i), s.numel(), k, _dev.ptr(top_s), _dev.ptr(top_i),
                  _dev.stream_handle(stream, s.device))
    for t in (s, i):
        _dev.keep_alive(t, stream)
    return top_s, top_i


def merge_topk_across_ranks(top_s: torch.Tensor, top_id: torch.Tensor, k: int, group=None, select=None):
    """All-gather every rank's K candidates and re-select the global top-K (same tie rule).

    The payload is k * 16 bytes per rank; with NCCL it is one all_gather of device tensors
    straight into the device selection kernel.  `select` replaces that kernel (the CPU gloo tests
    pass an oracle-backed twin; the product path always uses `select_candidates`).
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    gs = [torch.empty_like(top_s) for _ in range(world)]
    gi = [torch.empty_like(top_id) for _ in range(world)]
    dist.all_gather(gs, top_s.contiguous(), group=group)
    dist.all_gather(gi, top_id.contiguous(), group=group)
    return (select or select_candidates)(torch.cat(gs), torch.cat(gi), k)
