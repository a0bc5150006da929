"""C4 INT8 rerank timing (10K docs) under the MXS_DEBUG knobs (2 = slots released unread)."""
import os, sys
import torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx

g = torch.Generator(device="cuda").manual_seed(0)
nb = int(os.environ.get("NB", "10000"))
WA = os.environ.get("ARGMAX", "0") == "1"
x = torch.randn(1, 1024, 128, device="cuda", generator=g)
qq, qs = mx.quant.quantize_tensor(x)
dq = torch.randint(-127, 128, (nb, 1024, 128), dtype=torch.int8, device="cuda", generator=g)
ds = torch.rand(nb, 1024, device="cuda", generator=g) * 0.01 + 0.001
for _ in range(3):
    mx.score_int8(qq, qs, dq, ds, want_argmax=WA)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mx.score_int8(qq, qs, dq, ds, want_argmax=WA)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t = sorted(ts)[len(ts) // 2]
print(f"int8 argmax={int(WA)} debug={os.environ.get('MXS_DEBUG', '0')} nb={nb}: {t:.3f} ms ({2 * 1024 * 1024 * 128 * nb / t / 1e9:.0f} TOP/s)")
