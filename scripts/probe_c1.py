"""C1 only (cut from probe_configs.py): Time the non-headline configs: C3 (fwd+bwd), C4 (INT8), C5 (varlen, scaled down), top-K."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx
from paper_2605_29517_b200 import _dev, _lib
from paper_2605_29517_b200.parallel import inbatch_step

def timeit(fn, reps=5, warm=2):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]

g = torch.Generator(device="cuda").manual_seed(0)
def unit(*shape):
    x = torch.randn(*shape, device="cuda", generator=g)
    return (x / x.norm(dim=-1, keepdim=True)).bfloat16()

# C1: ColBERT rerank, 1 query L_q=32 vs 1000 docs L_d=180, d=128, FP32 -> the bit-exact fp32 kernel
q1 = torch.randn(1, 32, 128, device="cuda", generator=g)
q1 = q1 / q1.norm(dim=-1, keepdim=True)
d1 = torch.randn(1000, 180, 128, device="cuda", generator=g)
d1 = d1 / d1.norm(dim=-1, keepdim=True)
t_c1 = timeit(lambda: mx.score_dense(q1, d1))
print(f"C1 fp32 exact {t_c1:.3f} ms ({1000 / t_c1 * 1e3 / 1e6:.2f} M docs/s, {1.47456e9 / t_c1 / 1e9:.2f} TFLOP/s fp32)")

