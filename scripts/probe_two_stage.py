"""Breakdown of two_stage_topk at the C4 shape (host wall time per phase, synchronised)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx
from paper_2605_29517_b200 import quant
from paper_2605_29517_b200.forward import score_dense
from paper_2605_29517_b200.topk import topk as device_topk

g = torch.Generator(device="cuda").manual_seed(0)
nb = 10000
def unit(*shape):
    x = torch.randn(*shape, device="cuda", generator=g)
    return (x / x.norm(dim=-1, keepdim=True)).bfloat16()
Q = unit(1024, 128)
D = torch.empty(nb, 1024, 128, dtype=torch.bfloat16, device="cuda")
for i in range(0, nb, 1000): D[i:i + 1000] = unit(1000, 1024, 128)
dq, ds = quant.quantize_tensor(D)
cq = mx.QuantizedCorpus(dq, ds)
full = mx.DocBatch.from_dense(D)

def T(name, fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): out = fn()
    torch.cuda.synchronize()
    print(f"{name:28s} {(time.perf_counter() - t0) / reps * 1e3:8.3f} ms")
    return out

T("two_stage_topk total", lambda: mx.two_stage_topk(Q, cq, full, k=20))
T("EmbeddingMatrix(query)", lambda: mx.EmbeddingMatrix(Q))
qq, qs = T("quantize query", lambda: quant.quantize_tensor(Q))
coarse = T("score_int8 10K", lambda: quant.score_int8(qq[None], qs[None], dq, ds, None, want_argmax=False)[0])
ids = T("topk 80", lambda: device_topk(coarse[0], 80)[1])
sid = T("sort ids", lambda: torch.sort(ids)[0])
Dsel = T("index_select 80 docs", lambda: full.data.index_select(0, sid))
vls = full.valid_lens.index_select(0, sid)
fine = T("score_dense 80", lambda: score_dense(Q[None], Dsel, vls, want_argmax=False)[0])
T("topk 20 + .cpu()", lambda: [t.cpu() for t in device_topk(fine[0], 20)])
