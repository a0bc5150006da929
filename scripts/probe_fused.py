"""A/B on one box: fused epilogue S4 sum (rowmax = NULL, one launch) vs materialised row maxima +
separate rowsum pass, interleaved, medians of REPS launches.  C2 bf16 (rerank / +argmax), C4 INT8
rerank, 100K-doc varlen sample."""
import ctypes
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_29517_b200 import _lib  # noqa: E402
from paper_2605_29517_b200.quant import quantize_tensor  # noqa: E402

REPS = int(os.environ.get("REPS", "20"))
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def P(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def timeit(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def ab(name, fns):
    for f in fns.values():
        for _ in range(3):
            f()
    torch.cuda.synchronize()
    ts = {k: [] for k in fns}
    for _ in range(REPS):
        for k, f in fns.items():
            ts[k].append(timeit(f))
    print(name + ": " + ", ".join(f"{k} {statistics.median(v):.4f} ms" for k, v in ts.items()), flush=True)


g = torch.Generator(device="cuda").manual_seed(1)
nb = 10000
Q = torch.randn(1, 1024, 128, device="cuda", generator=g)
Q = (Q / Q.norm(dim=-1, keepdim=True)).bfloat16()
D = torch.randn(nb, 1024, 128, device="cuda", generator=g)
D = (D / D.norm(dim=-1, keepdim=True)).bfloat16()
scores = torch.empty(1, nb, dtype=torch.float64, device="cuda")
am = torch.empty(1, nb, 1024, dtype=torch.int32, device="cuda")
rm = torch.empty(1, nb, 1024, dtype=torch.float32, device="cuda")


def dense(argmax, rowmax):
    return lambda: _lib.call("mxs_fused_score_batch", _lib.MXS_BF16, P(Q), 1, 1024, P(D), nb, 1024, 128, None,
                             P(scores), P(argmax), P(rowmax), 0, st)


ab("C2 rerank", {"fused": dense(None, None), "rowmax+rowsum": dense(None, rm)})
ab("C2 +argmax", {"fused": dense(am, None), "rowmax+rowsum": dense(am, rm)})

qq, qs = quantize_tensor(Q.float())
dq, ds = quantize_tensor(D)


def int8(rowmax):
    return lambda: _lib.call("mxs_fused_score_int8", P(qq), P(qs), 1, 1024, P(dq), P(ds), nb, 1024, 128, None,
                             P(scores), None, P(rowmax), st)


ab("C4 INT8 rerank", {"fused": int8(None), "rowmax+rowsum": int8(rm)})
del qq, qs, dq, ds

n = 100_000
lens = np.random.default_rng(5).integers(32, 513, n)
cu = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)])).cuda()
T = int(lens.sum())
toks = torch.randn(T, 128, device="cuda", generator=g)
toks = (toks / toks.norm(dim=-1, keepdim=True)).bfloat16()
q5 = Q[:, :32].contiguous()
s5 = torch.empty(1, n, dtype=torch.float64, device="cuda")
r5 = torch.empty(1, n, 32, dtype=torch.float32, device="cuda")


def varlen(rowmax):
    return lambda: _lib.call("mxs_fused_score_varlen", _lib.MXS_BF16, P(q5), 1, 32, P(toks), P(cu), n, T, 128,
                             P(s5), None, P(rowmax), 0, st)


ab("C5 100K varlen", {"fused": varlen(None), "rowmax+rowsum": varlen(r5)})
