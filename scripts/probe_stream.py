"""Out-of-core top-K: an MXS1 file of ColPali-shape fp16 documents streamed through
stream_score_topk (native pread into pinned buffers, H2D of block i+1 under the scoring of block i,
device top-K merge).  The file was just written, so it is page-cache resident: this measures the
host-memory -> PCIe -> tensor-core pipeline, not the disk."""
import os, sys, time
import torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx

nb = int(os.environ.get("NB", "12000"))
g = torch.Generator(device="cuda").manual_seed(0)
def unit(*shape):
    x = torch.randn(*shape, device="cuda", generator=g)
    return (x / x.norm(dim=-1, keepdim=True)).half()
D = torch.empty(nb, 1024, 128, dtype=torch.float16, device="cuda")
for i in range(0, nb, 500): D[i:i + 500] = unit(min(500, nb - i), 1024, 128)
q = unit(1024, 128)
path = "/tmp/mxs_stream_probe.mxs1"
t0 = time.perf_counter()
mx.write_embeddings(path, mx.DocBatch.from_dense(D), elem="f16")
print(f"wrote {os.path.getsize(path) / 1e9:.2f} GB in {time.perf_counter() - t0:.1f} s")
del D
torch.cuda.empty_cache()
for bd in (1000, 2000):
    mx.stream_score_topk(q, path, block_docs=bd, k=20)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        ranked, rep = mx.stream_score_topk(q, path, block_docs=bd, k=20)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    print(f"stream_score_topk block_docs={bd}: {t * 1e3:.1f} ms for {nb} docs = {nb / t:,.0f} docs/s "
          f"({os.path.getsize(path) / t / 1e9:.1f} GB/s file -> scores)")
os.remove(path)
