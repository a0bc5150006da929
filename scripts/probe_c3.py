"""C3 in-batch step (N_q = B = 64, ColPali shape, bf16): run a few steps (for ncu launch lists)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_29517_b200.parallel import inbatch_step  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)


def unit(*shape):
    x = torch.randn(*shape, device="cuda", generator=g)
    return (x / x.norm(dim=-1, keepdim=True)).bfloat16()


Q = unit(64, 1024, 128)
D = unit(64, 1024, 128)
for _ in range(3):
    inbatch_step(Q, D, 0)
torch.cuda.synchronize()
