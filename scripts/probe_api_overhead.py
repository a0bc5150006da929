"""Public-API call overhead (validation + scratch) at C1 and a C5 sample, validate on / off."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


g = torch.Generator(device="cuda").manual_seed(0)
q1 = torch.randn(1, 32, 128, device="cuda", generator=g)
d1 = torch.randn(1000, 180, 128, device="cuda", generator=g)
vl1 = torch.full((1000,), 180, dtype=torch.int32, device="cuda")
print(f"C1 score_dense fp32: {timeit(lambda: mx.score_dense(q1, d1, want_argmax=False)):.3f} ms; "
      f"with valid_lens: {timeit(lambda: mx.score_dense(q1, d1, vl1, want_argmax=False)):.3f} ms; "
      f"no validation: {timeit(lambda: mx.score_dense(q1, d1, vl1, want_argmax=False, validate=False)):.3f} ms")
rng = np.random.default_rng(0)
lens = rng.integers(32, 513, 100000)
cu = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)])).cuda()
toks = torch.randn(int(cu[-1]), 128, device="cuda", generator=g).bfloat16()
q5 = torch.randn(1, 32, 128, device="cuda", generator=g).bfloat16()
print(f"C5 100K score_varlen: {timeit(lambda: mx.score_varlen(q5, toks, cu, want_argmax=False)):.3f} ms; "
      f"no validation: {timeit(lambda: mx.score_varlen(q5, toks, cu, want_argmax=False, validate=False)):.3f} ms")
