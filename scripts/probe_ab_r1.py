"""A/B on one box: the current library vs the round-1 library (scripts/old_lib/libmaxsim_r1.so,
built from commit 91d5b66), interleaved launches, medians.  Old entry points always need rowmax."""
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
new = _lib.load()
old = ctypes.CDLL(os.path.join("scripts", "old_lib", "libmaxsim_r1.so"))
for lib in (new, old):
    for name in ("mxs_fused_score_batch", "mxs_fused_score_int8", "mxs_fused_score_varlen"):
        getattr(lib, name).argtypes = _lib._SIGNATURES[name]
        getattr(lib, name).restype = ctypes.c_int
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def P(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def chk(r):
    assert r == 0, r


def timeit(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def ab(name, fns):
    import random

    for f in fns.values():
        for _ in range(3):
            f()
    torch.cuda.synchronize()
    ts = {k: [] for k in fns}
    rnd = random.Random(1)
    for _ in range(REPS):
        order = list(fns.items())
        rnd.shuffle(order)
        for k, f in order:
            ts[k].append(timeit(f))
    print(name + ": " + ", ".join(f"{k} {statistics.median(v):.4f} (min {min(v):.4f})" for k, v in ts.items()),
          flush=True)


def unit(shape):
    x = torch.randn(*shape, device="cuda", generator=g)
    return (x / x.norm(dim=-1, keepdim=True)).bfloat16()


g = torch.Generator(device="cuda").manual_seed(1)
for (nq, nb) in ((1, 10000), (64, 64)):
    Q = unit((nq, 1024, 128))
    D = unit((nb, 1024, 128))
    scores = torch.empty(nq, nb, dtype=torch.float64, device="cuda")
    am = torch.empty(nq, nb, 1024, dtype=torch.int32, device="cuda")
    rm = torch.empty(nq, nb, 1024, dtype=torch.float32, device="cuda")

    def dense(lib, argmax, rowmax):
        return lambda: chk(lib.mxs_fused_score_batch(_lib.MXS_BF16, P(Q), nq, 1024, P(D), nb, 1024, 128, None,
                                                     P(scores), P(argmax), P(rowmax), 0, st))

    tag = "C2" if nq == 1 else "C3 fwd"
    ab(f"{tag} rerank", {"new": dense(new, None, None), "r1": dense(old, None, rm)})
    ab(f"{tag} +argmax", {"new": dense(new, am, None), "new+rowmax": dense(new, am, rm), "r1": dense(old, am, rm)})
    if nq == 1:
        qq, qs = quantize_tensor(Q.float())
        dq, ds = quantize_tensor(D)

        def int8(lib, argmax, rowmax):
            return lambda: chk(lib.mxs_fused_score_int8(P(qq), P(qs), 1, 1024, P(dq), P(ds), nb, 1024, 128, None,
                                                        P(scores), P(argmax), P(rowmax), st))

        ab("C4 INT8 rerank", {"new": int8(new, None, None), "new+rowmax": int8(new, None, rm), "r1": int8(old, None, rm)})
        ab("C4 INT8 +argmax", {"new": int8(new, am, None), "new+rowmax": int8(new, am, rm), "r1": int8(old, am, rm)})
        del qq, qs, dq, ds
    del Q, D, scores, am, rm

n = 100_000
lens = np.random.default_rng(5).integers(32, 513, n)
cu = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)])).cuda()
T = int(lens.sum())
toks = unit((T, 128))
q5 = unit((1, 32, 128))
s5 = torch.empty(1, n, dtype=torch.float64, device="cuda")
r5 = torch.empty(1, n, 32, dtype=torch.float32, device="cuda")
a5 = torch.empty(1, n, 32, dtype=torch.int32, device="cuda")


def varlen(lib, argmax, rowmax):
    return lambda: chk(lib.mxs_fused_score_varlen(_lib.MXS_BF16, P(q5), 1, 32, P(toks), P(cu), n, T, 128, P(s5),
                                                  P(argmax), P(rowmax), 0, st))


ab("C5 100K varlen", {"new": varlen(new, None, None), "new+rowmax": varlen(new, None, r5), "r1": varlen(old, None, r5)})
ab("C5 100K varlen +argmax", {"new": varlen(new, a5, None), "r1": varlen(old, a5, r5)})
