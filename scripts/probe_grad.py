"""C3-shape backward gathers (N_q = B = 64, L = 1024, d = 128, bf16): CUDA-graph-timed dD
(grad_docs_csr) and dQ (grad_query) kernels, and their effective L2 gather rate."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx  # noqa: E402
from paper_2605_29517_b200.backward import csr_tensors  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
Q = torch.randn(64, 1024, 128, device="cuda", generator=g).bfloat16()
D = torch.randn(64, 1024, 128, device="cuda", generator=g).bfloat16()
idx = torch.randint(0, 1024, (64, 64, 1024), device="cuda", generator=g, dtype=torch.int32)
up = torch.randn(64, 64, device="cuda", generator=g, dtype=torch.float64)
off = torch.arange(64, device="cuda", dtype=torch.int64) * 1024
lens = torch.full((64,), 1024, device="cuda", dtype=torch.int64)
rp, ci, _ = csr_tensors(idx, off, lens, 65536, 1024)
csr = mx.CsrInverse(row_ptr=rp, col_idx=ci, n_dest=65536, src_shape=(64, 64, 1024), padded_len=1024)
am = mx.ArgmaxMap(idx, [1024] * 64, padded_len=1024)
out_d = torch.empty(65536, 128, device="cuda")


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(reps):
            fn()
    gr.replay()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    return statistics.median(ts)


docs = mx.DocBatch.from_dense(D)
gbytes = 64 * 64 * 1024 * 256  # gathered row bytes per kernel
for name, fn in (("dD grad_docs_csr", lambda: mx.grad_docs_csr(csr, up, Q, out=out_d)),
                 ("dQ grad_query", lambda: mx.grad_query(am, up, docs))):
    us = timed(fn)
    print(f"{name:18s} {us:7.1f} us   gathered rows {gbytes / us / 1e6:6.1f} TB/s", flush=True)
