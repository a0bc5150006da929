import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx
g = torch.Generator(device="cuda").manual_seed(1)
n = 100_000
lens = np.random.default_rng(5).integers(32, 513, n)
cu = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)])).cuda()
toks = torch.randn(int(lens.sum()), 128, device="cuda", generator=g).bfloat16()
q = torch.randn(1, 32, 128, device="cuda", generator=g).bfloat16()
for _ in range(2):
    mx.score_varlen(q, toks, cu, want_argmax=False, validate=False)
torch.cuda.synchronize()
