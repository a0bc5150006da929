"""One C4 INT8 launch and one C5-shape varlen launch (for ncu -k regex)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx
g = torch.Generator(device="cuda").manual_seed(0)
def unit(*shape):
    x = torch.randn(*shape, device="cuda", generator=g)
    return (x / x.norm(dim=-1, keepdim=True)).bfloat16()
which = os.environ.get("WHICH", "both")
if which in ("both", "int8"):
    nb = 2000
    qq, qs = mx.quant.quantize_tensor(unit(1, 1024, 128))
    dq, ds = mx.quant.quantize_tensor(unit(nb, 1024, 128))
    for _ in range(3):
        mx.score_int8(qq, qs, dq, ds, want_argmax=os.environ.get("ARGMAX", "1") == "1")
if which in ("both", "varlen"):
    rng = np.random.default_rng(0)
    lens = rng.integers(32, 513, 50000)
    cu = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)])).cuda()
    toks = unit(int(cu[-1]), 128)
    q = unit(1, 32, 128)
    for _ in range(3):
        mx.score_varlen(q, toks, cu)
torch.cuda.synchronize()
