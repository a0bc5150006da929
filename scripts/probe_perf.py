"""C2 timing under debug knobs (MXS_DEBUG: 0 = full, 1 = TMEM load only, 2 = no epilogue)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_29517_b200 import _lib  # noqa: E402

nb = int(os.environ.get("NB", "10000"))
lq = int(os.environ.get("LQ", "1024"))
g = torch.Generator(device="cuda").manual_seed(1)
Q = torch.randn(1, lq, 128, device="cuda", generator=g).bfloat16()
D = torch.randn(nb, 1024, 128, device="cuda", generator=g).bfloat16()
scores = torch.empty(1, nb, dtype=torch.float64, device="cuda")
am = torch.empty(1, nb, lq, dtype=torch.int32, device="cuda")
rm = torch.empty(1, nb, lq, dtype=torch.float32, device="cuda")
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def P(t):
    return ctypes.c_void_p(t.data_ptr())


WANT_ARGMAX = os.environ.get("ARGMAX", "1") == "1"
WANT_ROWMAX = os.environ.get("ROWMAX", "1") == "1"  # 0: fused score only (the bench's rerank call)


def go():
    _lib.call("mxs_fused_score_batch", _lib.MXS_BF16, P(Q), 1, lq, P(D), nb, 1024, 128, None, P(scores),
              P(am) if WANT_ARGMAX else None, P(rm) if WANT_ROWMAX else None, 0, st)


for _ in range(3):
    go()
torch.cuda.synchronize()
ts = []
for _ in range(int(os.environ.get("REPS", "10"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    go()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t = sorted(ts)[len(ts) // 2]
fl = 2 * lq * 1024 * 128 * nb
print(f"debug={os.environ.get('MXS_DEBUG', '0')} argmax={int(WANT_ARGMAX)} nb={nb} lq={lq}: {t:.3f} ms "
      f"{fl / t / 1e9:.0f} TFLOP/s")
