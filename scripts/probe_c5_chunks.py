"""C5 full size (1M docs): one varlen launch over the whole 69.7 GB vs K launches over contiguous
document chunks (same kernels, same scores) -- does the per-launch span matter?"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx

g = torch.Generator(device="cuda").manual_seed(0)
rng = np.random.default_rng(0)
n = 1_000_000
lens = rng.integers(32, 513, n)
cu_h = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
T = int(cu_h[-1])
cu = torch.from_numpy(cu_h).cuda()
toks = torch.empty(T, 128, dtype=torch.bfloat16, device="cuda")
for i in range(0, T, 8_000_000):
    x = torch.randn(min(8_000_000, T - i), 128, device="cuda", generator=g)
    toks[i:i + x.shape[0]] = (x / x.norm(dim=-1, keepdim=True)).bfloat16()
    del x
q = torch.randn(1, 32, 128, device="cuda", generator=g)
q = (q / q.norm(dim=-1, keepdim=True)).bfloat16()
ref, _, _ = mx.score_varlen(q, toks, cu, want_argmax=False)
for K in (1, 2, 4, 8, 16):
    bounds = [(n * i) // K for i in range(K + 1)]
    parts = [(toks[int(cu_h[a]):int(cu_h[b])], (cu[a:b + 1] - cu[a]).contiguous()) for a, b in zip(bounds, bounds[1:])]
    out = torch.empty(1, n, dtype=torch.float64, device="cuda")
    def run():
        for (tk, c), a, b in zip(parts, bounds, bounds[1:]):
            s, _, _ = mx.score_varlen(q, tk, c, want_argmax=False)
            out[:, a:b].copy_(s)
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[2]
    print(f"K={K:2d} launches: {ms:.2f} ms  {n / ms / 1e3:.1f} M docs/s  {T * 256 / ms / 1e6:.0f} GB/s  "
          f"identical={bool(torch.equal(out, ref))}")
