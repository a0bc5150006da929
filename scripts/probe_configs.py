"""Time the non-headline configs: C3 (fwd+bwd), C4 (INT8), C5 (varlen, scaled down), top-K."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx
from paper_2605_29517_b200 import _dev, _lib
from paper_2605_29517_b200.parallel import inbatch_step

def timeit(fn, reps=5, warm=2):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]

g = torch.Generator(device="cuda").manual_seed(0)
def unit(*shape):
    x = torch.randn(*shape, device="cuda", generator=g)
    return (x / x.norm(dim=-1, keepdim=True)).bfloat16()

# C1: ColBERT rerank, 1 query L_q=32 vs 1000 docs L_d=180, d=128, FP32 -> the bit-exact fp32 kernel
q1 = torch.randn(1, 32, 128, device="cuda", generator=g)
q1 = q1 / q1.norm(dim=-1, keepdim=True)
d1 = torch.randn(1000, 180, 128, device="cuda", generator=g)
d1 = d1 / d1.norm(dim=-1, keepdim=True)
t_c1 = timeit(lambda: mx.score_dense(q1, d1))
print(f"C1 fp32 exact {t_c1:.3f} ms ({1000 / t_c1 * 1e3 / 1e6:.2f} M docs/s, {1.47456e9 / t_c1 / 1e9:.2f} TFLOP/s fp32)")

# C3: in-batch 64 x 64 ColPali shape
Q = unit(64, 1024, 128); D = unit(64, 1024, 128)
t_fwd = timeit(lambda: mx.score_dense(Q, D))
_, am, _ = mx.score_dense(Q, D)
gq = torch.randn(64, 64, device="cuda", generator=g).float()
off = torch.arange(64, dtype=torch.int64, device="cuda") * 1024
lens = torch.full((64,), 1024, dtype=torch.int64, device="cuda")
from paper_2605_29517_b200.backward import csr_tensors
from paper_2605_29517_b200.autograd import _grad_docs, _grad_query
t_csr = timeit(lambda: csr_tensors(am, off, lens, 65536, 1024))
t_dd = timeit(lambda: _grad_docs(Q, am, gq, off, lens, 65536, 1024, 128))
t_dq = timeit(lambda: _grad_query(D.reshape(-1, 128), off, am, gq, 128))
t_step = timeit(lambda: inbatch_step(Q, D, 0))
from paper_2605_29517_b200.parallel import InBatchStepGraph
gstep = InBatchStepGraph(Q, D)
t_gstep = timeit(gstep)
print(f"C3 fwd {t_fwd:.3f} ms ({1.0995e12 / t_fwd / 1e9:.0f} TF/s) | csr {t_csr:.3f} | csr+dD {t_dd:.3f} | dQ {t_dq:.3f} | full step {t_step:.3f} ms | graph step {t_gstep:.3f} ms")

# C4: INT8 10K docs
nb = 10000
Qf = unit(1, 1024, 128); Df = torch.empty(nb, 1024, 128, dtype=torch.bfloat16, device="cuda")
for i in range(0, nb, 1000): Df[i:i + 1000] = unit(1000, 1024, 128)
t_q = timeit(lambda: mx.quant.quantize_tensor(Df))
dq, ds = mx.quant.quantize_tensor(Df); qq, qs = mx.quant.quantize_tensor(Qf)
t_i8 = timeit(lambda: mx.score_int8(qq, qs, dq, ds, want_argmax=False))
t_i8a = timeit(lambda: mx.score_int8(qq, qs, dq, ds))
t_bf = timeit(lambda: mx.score_dense(Qf, Df, want_argmax=False))
t_bfa = timeit(lambda: mx.score_dense(Qf, Df))
print(f"C4 int8 rerank {t_i8:.3f} ms ({nb / t_i8 * 1e3 / 1e6:.2f} M docs/s, {2.684e12 / t_i8 / 1e9:.0f} TOP/s), "
      f"+argmax {t_i8a:.3f} ms | bf16 rerank {t_bf:.3f} ms, +argmax {t_bfa:.3f} ms | quantize corpus {t_q:.3f} ms")
# measured INT8 dense peak (torch._int_mm at 8192^3, the cuBLASLt s8 x s8 -> s32 GEMM)
a8 = torch.randint(-127, 128, (8192, 8192), dtype=torch.int8, device="cuda")
b8 = torch.randint(-127, 128, (8192, 8192), dtype=torch.int8, device="cuda").t()
t_mm = timeit(lambda: torch._int_mm(a8, b8), reps=10, warm=3)
peak8 = 2 * 8192 ** 3 / t_mm / 1e9
print(f"C4 roofline: int8 peak (torch._int_mm 8192^3) {peak8:.0f} TOP/s; rerank kernel {2.684e12 / t_i8 / 1e9:.0f} TOP/s "
      f"= {2.684e12 / t_i8 / 1e9 / peak8:.1%} of measured, {2.684e12 / t_i8 / 1e9 / 4500:.1%} of 4.5 POPS spec")
del a8, b8
# two-stage top-20 (INT8 scan of all 10K docs, bf16 rescoring of the 80-doc shortlist), public API
corpus_q = mx.QuantizedCorpus(dq, ds) if hasattr(mx, "QuantizedCorpus") else None
full = mx.DocBatch.from_dense(Df)
try:
    t_2s = timeit(lambda: mx.two_stage_topk(Qf[0], corpus_q, full, k=20), reps=5, warm=2)
    print(f"C4 two-stage top-20 of {nb}: {t_2s:.3f} ms ({nb / t_2s * 1e3 / 1e6:.2f} M docs/s) incl. host result list")
except Exception as e:  # report, do not abort the probe
    print(f"C4 two-stage: {type(e).__name__}: {e}")
del Df, dq

# C5 scaled: varlen 100K docs L in [32, 512], L_q = 32
rng = np.random.default_rng(0)
n5 = int(os.environ.get("N5", "100000"))
lens5 = rng.integers(32, 513, n5)
cu = torch.from_numpy(np.concatenate([[0], np.cumsum(lens5)])).cuda()
T = int(cu[-1])
toks = torch.empty(T, 128, dtype=torch.bfloat16, device="cuda")
for i in range(0, T, 4_000_000): toks[i:i + 4_000_000] = unit(min(4_000_000, T - i), 128)
q5 = unit(1, 32, 128)
t_v = timeit(lambda: mx.score_varlen(q5, toks, cu, want_argmax=False), reps=3, warm=1)
t_va = timeit(lambda: mx.score_varlen(q5, toks, cu), reps=3, warm=1)
byt = T * 256
print(f"C5 varlen {n5} docs ({T} tokens): rerank {t_v:.3f} ms ({n5 / t_v * 1e3 / 1e6:.2f} M docs/s, {byt / t_v / 1e6:.0f} GB/s), +argmax {t_va:.3f} ms")
sc, _, _ = mx.score_varlen(q5, toks, cu)
t_k = timeit(lambda: mx.topk(sc[0], 20))
print(f"topk 20 of {n5}: {t_k:.3f} ms")
