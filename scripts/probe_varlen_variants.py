"""Varlen kernel variants (scripts/old_lib/*.so) timed interleaved on one box: 100K-doc C5 sample."""
import ctypes
import glob
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_29517_b200 import _lib  # noqa: E402

libs = {"current": _lib.load()}
for p in sorted(glob.glob("scripts/old_lib/*.so")):
    libs[os.path.basename(p)] = ctypes.CDLL(p)
for lib in libs.values():
    lib.mxs_fused_score_varlen.argtypes = _lib._SIGNATURES["mxs_fused_score_varlen"]
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())  # noqa: E731
g = torch.Generator(device="cuda").manual_seed(1)
n = 100_000
lens = np.random.default_rng(5).integers(32, 513, n)
cu = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)])).cuda()
T = int(lens.sum())
toks = torch.randn(T, 128, device="cuda", generator=g).bfloat16()
q5 = torch.randn(1, 32, 128, device="cuda", generator=g).bfloat16()
s5 = torch.empty(1, n, dtype=torch.float64, device="cuda")
r5 = torch.empty(1, n, 32, dtype=torch.float32, device="cuda")
runs = [(k, lib, r5) for k, lib in libs.items()] + [("current fused (rowmax NULL)", libs["current"], None)]
if os.environ.get("MXS_VARLEN_FUSE") == "0":
    runs = [(k + " [MXS_VARLEN_FUSE=0]", lib, rm) for k, lib, rm in runs]
ts = {k: [] for k, _, _ in runs}
import random
rnd = random.Random(0)
for it in range(40):
    order = list(runs)
    rnd.shuffle(order)
    for k, lib, rm in order:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = lib.mxs_fused_score_varlen(_lib.MXS_BF16, P(q5), 1, 32, P(toks), P(cu), n, T, 128, P(s5), None, P(rm), 0, st)
        e1.record()
        torch.cuda.synchronize()
        assert r == 0
        if it >= 3:
            ts[k].append(e0.elapsed_time(e1))
for k, v in ts.items():
    print(f"{k}: median {statistics.median(v):.4f} ms  min {min(v):.4f}  max {max(v):.4f}")
