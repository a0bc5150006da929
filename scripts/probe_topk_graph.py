"""Device time of one top-K call (k = 20) at the bench shapes, CUDA-graph timed (no host overhead)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
for n in (10000, 100000, 1000000):
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    for _ in range(3):
        mx.topk(x, 20)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(20):
            mx.topk(x, 20)
    gr.replay()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / 20)
    print(f"topk 20 of {n}: {statistics.median(ts):.1f} us per call (graph)")
