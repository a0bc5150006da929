"""top-K latency at the bench's shapes (k = 20 of 10K, 100K, 1M scores)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx
g = torch.Generator(device="cuda").manual_seed(0)
for n in (10000, 100000, 1000000):
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    for _ in range(3):
        mx.topk(x, 20)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); mx.topk(x, 20); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"topk 20 of {n}: {sorted(ts)[10] * 1e3:.1f} us")
