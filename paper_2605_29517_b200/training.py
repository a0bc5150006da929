"""In-batch contrastive training helpers (maxsim/cli.py:198-252), on the device.

* `softmax_ce`: the C3 loss, positives on the diagonal, float64 (maxsim/cli.py:198-206).
* `dense_score_backward`: the materializing reference path (the full [L_q, L_d] similarity
  tensor per pair, float64 on the device) -- the "dense" side of the drift check.
* `contrastive_drift`: trains the same toy objective through the fused sm_100a path (forward
  kernel, device CSR, destination-owned gathers) and through the dense path, returning the loss
  trajectories and their max relative drift (maxsim/cli.py:209-252; reference acceptance
  criterion c11 asks for <= 1e-4 over 200 steps).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev
from .parallel import softmax_ce

__all__ = ["softmax_ce", "dense_score_backward", "contrastive_drift"]


def dense_score_backward(Q: torch.Tensor, D: torch.Tensor, g: torch.Tensor):
    """Dense reference: scores [N, B] f64, argmax, dQ, dD (f64) from the materialized similarities."""
    S = torch.einsum("qid,bjd->qbij", Q.double(), D.double())
    best, arg = S.max(dim=3)
    scores = best.sum(dim=2)
    w = g.double()[:, :, None].expand_as(best)                       # [N, B, L_q]
    Db = D.double()
    gathered = Db[torch.arange(D.shape[0], device=D.device)[None, :, None], arg]  # [N, B, L_q, d]
    dQ = (w[..., None] * gathered).sum(dim=1)
    dD = torch.zeros_like(Db)
    for b in range(D.shape[0]):
        idx = arg[:, b, :].reshape(-1)
        src = (w[:, b, :, None] * Q.double()).reshape(-1, Q.shape[-1])
        dD[b].index_add_(0, idx, src)
    return scores, arg, dQ, dD


def contrastive_drift(n_docs: int, len_q: int, len_d: int, dim: int, steps: int, seed: int,
                      lr: float = 0.05) -> dict:
    """Same toy objective through the fused device path and the dense path (maxsim/cli.py:209)."""
    from .autograd import maxsim

    rng = np.random.default_rng(seed)
    q0 = rng.standard_normal((n_docs, len_q, dim)).astype(np.float32)
    d0 = rng.standard_normal((n_docs, len_d, dim)).astype(np.float32)
    dev = _dev.device()
    params = {"fused": (torch.from_numpy(q0).to(dev), torch.from_numpy(d0).to(dev)),
              "dense": (torch.from_numpy(q0).to(dev), torch.from_numpy(d0).to(dev))}
    losses = {"fused": [], "dense": []}
    for _ in range(steps):
        for path in ("fused", "dense"):
            q, d = params[path]
            if path == "fused":
                Q = q.clone().requires_grad_(True)
                D = d.clone().requires_grad_(True)
                s = maxsim(Q, D)
                loss, g = softmax_ce(s.detach())
                (s * g).sum().backward()
                d_q, d_d = Q.grad.double(), D.grad.double()
            else:
                s, _, _, _ = dense_score_backward(q, d, torch.zeros(n_docs, n_docs, device=dev))
                loss, g = softmax_ce(s)
                _, _, d_q, d_d = dense_score_backward(q, d, g)
            losses[path].append(float(loss))
            params[path] = ((q.double() - lr * d_q).float(), (d.double() - lr * d_d).float())
    fused = np.array(losses["fused"])
    dense = np.array(losses["dense"])
    drift = float(np.max(np.abs(fused - dense) / np.maximum(np.abs(dense), 1e-300)))
    return {"steps": steps, "loss_first": float(dense[0]), "loss_last_dense": float(dense[-1]),
            "loss_last_fused": float(fused[-1]), "max_rel_drift": drift}
