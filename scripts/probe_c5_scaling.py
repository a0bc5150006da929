"""Varlen kernel throughput vs corpus size (same process, same clocks): 100K .. 1M documents."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
rng = np.random.default_rng(0)
n = 1_000_000
lens = rng.integers(32, 513, n)
cu_h = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
T = int(cu_h[-1])
toks = torch.empty(T, 128, dtype=torch.bfloat16, device="cuda")
for i in range(0, T, 8_000_000):
    x = torch.randn(min(8_000_000, T - i), 128, device="cuda", generator=g)
    toks[i:i + x.shape[0]] = (x / x.norm(dim=-1, keepdim=True)).bfloat16()
    del x
q = torch.randn(1, 32, 128, device="cuda", generator=g)
q = (q / q.norm(dim=-1, keepdim=True)).bfloat16()
for nd in (100_000, 300_000, 1_000_000, 100_000):
    cu = torch.from_numpy(cu_h[:nd + 1]).cuda()
    t = toks[: int(cu_h[nd])]
    for _ in range(2):
        mx.score_varlen(q, t, cu, want_argmax=False)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mx.score_varlen(q, t, cu, want_argmax=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[2]
    print(f"{nd} docs: {ms:.3f} ms  {int(cu_h[nd]) * 256 / ms / 1e6:.0f} GB/s")
