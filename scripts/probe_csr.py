"""C3-shape inverse CSR (64 x 64 x 1024 argmax, 65,536 destination rows): CUDA-event time of
mxs_build_inverse_csr per builder / warp-range size (MXS_CSR_IMPL, MXS_CSR_SRC_PER_WARP)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx  # noqa: E402
from paper_2605_29517_b200.backward import csr_tensors  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
idx = torch.randint(0, 1024, (64, 64, 1024), device="cuda", generator=g, dtype=torch.int32)
off = torch.arange(64, device="cuda", dtype=torch.int64) * 1024
lens = torch.full((64,), 1024, device="cuda", dtype=torch.int64)
ref = None
CONFIGS = [("doc", "512"), ("doc", "1024"), ("doc", "2048"), ("doc", "4096")]
if os.environ.get("CONFIGS"):  # e.g. CONFIGS=doc:1024,sort:0
    CONFIGS = [tuple(c.split(":")) for c in os.environ["CONFIGS"].split(",")]
for impl, pw in CONFIGS:
    os.environ["MXS_CSR_IMPL"] = impl
    os.environ["MXS_CSR_SRC_PER_WARP"] = pw
    for _ in range(3):
        rp, ci, _ = csr_tensors(idx, off, lens, 65536, 1024)
    torch.cuda.synchronize()
    if ref is None:
        ref = (rp.clone(), ci.clone())
    assert torch.equal(rp, ref[0]) and torch.equal(ci, ref[1]), (impl, pw)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(10):
            csr_tensors(idx, off, lens, 65536, 1024)
    gr.replay()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / 10)
    print(f"{impl:5s} per_warp={pw:5s} median {statistics.median(ts):7.1f} us  min {min(ts):7.1f} us", flush=True)
