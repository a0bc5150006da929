# varlen C5 sample (500K docs): integer fixed-point sum warp vs the previous FP64 one, same box
cat > /tmp/v.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx
g = torch.Generator(device="cuda").manual_seed(0)
rng = np.random.default_rng(0)
import os
n = int(os.environ.get("NDOCS", "500000"))
lens = rng.integers(32, 513, n)
cu = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)])).cuda()
T = int(cu[-1])
toks = torch.empty(T, 128, dtype=torch.bfloat16, device="cuda")
for i in range(0, T, 4_000_000):
    toks[i:i + 4_000_000] = torch.randn(min(4_000_000, T - i), 128, device="cuda", generator=g).bfloat16()
q = torch.randn(1, 32, 128, device="cuda", generator=g).bfloat16()
def t(f):
    for _ in range(3): f()
    torch.cuda.synchronize(); ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[5]
ms = t(lambda: mx.score_varlen(q, toks, cu, want_argmax=False, validate=False))
print(f"varlen {n} docs: {ms:.3f} ms {T * 256 / ms / 1e6:.0f} GB/s")
PY
for n in 250000 500000 1000000 500000; do NDOCS=$n timeout 600 python /tmp/v.py; done
