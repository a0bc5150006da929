"""fwd_ts / fwd_i8r with and without the fused S4 epilogue (MXS_FWD_FUSE toggled in-process) vs the
round-1 library, randomized interleaving: C4 INT8 (+argmax / rerank), C2 bf16 (+argmax / rerank)."""
import ctypes
import os
import random
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_29517_b200 import _lib  # noqa: E402
from paper_2605_29517_b200.quant import quantize_tensor  # noqa: E402

REPS = int(os.environ.get("REPS", "30"))
new = _lib.load()
old = ctypes.CDLL(os.path.join("scripts", "old_lib", "libmaxsim_r1.so"))
for lib in (new, old):
    for name in ("mxs_fused_score_batch", "mxs_fused_score_int8"):
        getattr(lib, name).argtypes = _lib._SIGNATURES[name]
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())  # noqa: E731
g = torch.Generator(device="cuda").manual_seed(1)


def unit(shape):
    x = torch.randn(*shape, device="cuda", generator=g)
    return (x / x.norm(dim=-1, keepdim=True)).bfloat16()


nb = 10000
Q, D = unit((1, 1024, 128)), unit((nb, 1024, 128))
qq, qs = quantize_tensor(Q.float())
dq, ds = quantize_tensor(D)
sc = torch.empty(1, nb, dtype=torch.float64, device="cuda")
am = torch.empty(1, nb, 1024, dtype=torch.int32, device="cuda")
rm = torch.empty(1, nb, 1024, dtype=torch.float32, device="cuda")


def i8(lib, argmax, fuse):
    def f():
        os.environ["MXS_FWD_FUSE"] = "1" if fuse else "0"
        r = lib.mxs_fused_score_int8(P(qq), P(qs), 1, 1024, P(dq), P(ds), nb, 1024, 128, None, P(sc), P(argmax), P(rm), st)
        assert r == 0
    return f


def bf(lib, argmax, fuse):
    def f():
        os.environ["MXS_FWD_FUSE"] = "1" if fuse else "0"
        r = lib.mxs_fused_score_batch(_lib.MXS_BF16, P(Q), 1, 1024, P(D), nb, 1024, 128, None, P(sc), P(argmax), P(rm), 0, st)
        assert r == 0
    return f


def ab(name, fns):
    for f in fns.values():
        f()
    torch.cuda.synchronize()
    ts = {k: [] for k in fns}
    rnd = random.Random(2)
    for _ in range(REPS):
        order = list(fns.items())
        rnd.shuffle(order)
        for k, f in order:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            torch.cuda.synchronize()
            ts[k].append(e0.elapsed_time(e1))
    print(name + ": " + ", ".join(f"{k} {statistics.median(v):.4f} (min {min(v):.4f})" for k, v in ts.items()), flush=True)


for a, tag in ((am, "+argmax"), (None, "rerank")):
    ab(f"C4 INT8 {tag}", {"fused": i8(new, a, True), "unfused": i8(new, a, False), "r1": i8(old, a, True)})
    ab(f"C2 bf16 {tag}", {"fused": bf(new, a, True), "unfused": bf(new, a, False), "r1": bf(old, a, True)})
