"""Varlen tensor-core path vs the exact kernel and the oracle on ragged packed corpora."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx
from oracle import oracle as orc

def run(n_docs, lo, hi, l_q, n_q=1, dim=128, seed=0):
    rng = np.random.default_rng(seed)
    lens = rng.integers(lo, hi + 1, n_docs)
    cu = np.concatenate([[0], np.cumsum(lens)])
    g = torch.Generator(device="cuda").manual_seed(seed)
    T = torch.randn(int(cu[-1]), dim, device="cuda", generator=g)
    T = (T / T.norm(dim=-1, keepdim=True)).bfloat16()
    Q = torch.randn(n_q, l_q, dim, device="cuda", generator=g)
    Q = (Q / Q.norm(dim=-1, keepdim=True)).bfloat16()
    cud = torch.from_numpy(cu).cuda()
    s_tc, a_tc, r_tc = mx.score_varlen(Q, T, cud)
    s_ex, a_ex, r_ex = mx.score_varlen(Q, T, cud, exact=True)
    rel = ((s_tc - s_ex).abs() / s_ex.abs()).max().item()
    agree = (a_tc == a_ex).float().mean().item()
    rdiff = (r_tc - r_ex).abs().max().item()
    ok = rel < 1e-3 and agree > 0.998
    print(f"[varlen n={n_docs} L=[{lo},{hi}] l_q={l_q} n_q={n_q}] {'OK ' if ok else 'BAD'} rel={rel:.2e} rowmax_diff={rdiff:.2e} argmax_agree={agree:.5f}")
    return ok

ok = True
ok &= run(300, 32, 512, 32)
ok &= run(1000, 1, 20, 32)       # many docs per tile, 1-token docs
ok &= run(50, 100, 2000, 32)     # docs spanning many tiles
ok &= run(200, 1, 300, 16, n_q=4) # multi-query columns (64 cols)
ok &= run(100, 5, 200, 128)       # 128 columns, 4 chunks
ok &= run(7, 1, 3, 32)            # fewer docs than SMs / tiny
print("VARLEN_ALL_OK" if ok else "VARLEN_SOME_BAD")
