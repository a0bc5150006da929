import sys, statistics, torch
sys.path.insert(0, ".")
from paper_2605_29517_b200.parallel import ShardedInBatchStepGraph, InBatchStepGraph, inbatch_step
g = torch.Generator(device="cuda").manual_seed(0)
def unit(*sh):
    x = torch.randn(*sh, device="cuda", generator=g); return (x / x.norm(dim=-1, keepdim=True)).bfloat16()
Q = unit(64, 1024, 128); D = unit(64, 1024, 128)
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
sg = ShardedInBatchStepGraph(Q, D, 0); fg = InBatchStepGraph(Q, D)
for _ in range(2):
    print(f"eager {t(lambda: inbatch_step(Q, D, 0)):.3f} ms | segmented graphs {t(sg):.3f} ms | whole-step graph {t(fg):.3f} ms")
# the 8-rank shard size (8 docs per rank) on one GPU: host-overhead regime
D8 = D[:8].contiguous(); Q8 = Q[:8].contiguous()
sg8 = ShardedInBatchStepGraph(Q8, D8, 0)
print(f"B=8 shard: eager {t(lambda: inbatch_step(Q8, D8, 0)):.3f} ms | segmented graphs {t(sg8):.3f} ms")
