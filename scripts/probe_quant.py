"""C4 corpus quantisation (10K x 1024 x 128 bf16 -> INT8 + per-token scales): CUDA-event time and
HBM rate (3 B per element + 4 B per row)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(10_000 * 1024, 128, device="cuda", generator=g).bfloat16()
for _ in range(3):
    q, s = mx.quant.quantize_tensor(x)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mx.quant.quantize_tensor(x)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t = statistics.median(ts)
nbytes = x.numel() * 3 + x.shape[0] * 4
print(f"quantize 10.24M rows: {t:.3f} ms  {nbytes / t / 1e6:.0f} GB/s  checksum {int(q.to(torch.int64).sum())} {float(s.double().sum()):.6f}")
