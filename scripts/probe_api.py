"""Public-API overhead at the C2 shape: reference-facing calls vs the raw forward kernel."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx

g = torch.Generator(device="cuda").manual_seed(0)
nb = 10000
def unit(*shape):
    x = torch.randn(*shape, device="cuda", generator=g)
    return (x / x.norm(dim=-1, keepdim=True)).bfloat16()
Q = unit(1, 1024, 128)
D = torch.empty(nb, 1024, 128, dtype=torch.bfloat16, device="cuda")
for i in range(0, nb, 1000): D[i:i + 1000] = unit(1000, 1024, 128)
docs = mx.DocBatch.from_dense(D)

def T(name, fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    print(f"{name:44s} {(time.perf_counter() - t0) / reps * 1e3:8.3f} ms")

T("score_dense rerank (tensor API)", lambda: mx.score_dense(Q, D, want_argmax=False))
T("score_dense + argmax (tensor API)", lambda: mx.score_dense(Q, D))
T("score_dense + argmax + valid_lens", lambda: mx.score_dense(Q, docs.data, docs.valid_lens))
T("score_dense + argmax, D = docs.data", lambda: mx.score_dense(Q, docs.data))
print("docs.data is D:", docs.data.data_ptr() == D.data_ptr(), docs.data.dtype, docs.data.is_contiguous())
T("fused_score_batch(Q, DocBatch) (reference API)", lambda: mx.fused_score_batch(Q, docs))
T("fused_score_batch + scores.numpy()", lambda: mx.fused_score_batch(Q, docs)[0].numpy())
T("maxsim autograd forward", lambda: mx.maxsim(Q, D))
