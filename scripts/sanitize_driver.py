"""Small invocations of every device kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): fwd_ts (bf16 with argmax, rerank fused S4), fwd_pair (CTA pairs, QB = 4 / 2),
fwd_i8r + fwd_ts INT8,
varlen_rows (bf16, ragged across 128-token tiles), exact fp32, quantiser, CSR (cluster kernel +
radix-sort path), dD / dQ gathers, top-K, Chamfer.  WHICH=a,b,... selects families."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29517_b200 as mx  # noqa: E402
from paper_2605_29517_b200.backward import csr_tensors  # noqa: E402

WHICH = set(os.environ.get("WHICH", "fwd,pair,int8,varlen,exact,quant,csr,grad,topk,chamfer").split(","))
g = torch.Generator(device="cuda").manual_seed(0)


def unit(*shape, dtype=torch.bfloat16):
    x = torch.randn(*shape, device="cuda", generator=g)
    return (x / x.norm(dim=-1, keepdim=True)).to(dtype)


Q = unit(2, 256, 128)
D = unit(6, 384, 128)
vl = torch.tensor([384, 1, 200, 129, 255, 384], dtype=torch.int32, device="cuda")
if "fwd" in WHICH:
    s, a, _ = mx.score_dense(Q, D, vl)
    s2, _, _ = mx.score_dense(Q, D, vl, want_argmax=False)
    torch.cuda.synchronize()
    print("fwd ok", float(s.sum()), float(s2.sum()))
if "pair" in WHICH:  # CTA-pair forward: QB = 4 (L_q = 700: TMEM + SS blocks) and QB = 2 (L_q = 384)
    for lq in (700, 384):
        Qp = unit(2, lq, 128)
        sp, ap, _ = mx.score_dense(Qp, D, vl)
        sp2, _, _ = mx.score_dense(Qp, D, vl, want_argmax=False)
        torch.cuda.synchronize()
        print("pair ok", lq, float(sp.sum()), float(sp2.sum()))
if "int8" in WHICH:
    qq, qs = mx.quant.quantize_tensor(Q.float())
    dq, ds = mx.quant.quantize_tensor(D.float())
    s8, a8, _ = mx.score_int8(qq, qs, dq, ds, vl)
    r8, _, _ = mx.score_int8(qq, qs, dq, ds, vl, want_argmax=False)
    torch.cuda.synchronize()
    print("int8 ok", float(s8.sum()), float(r8.sum()))
if "varlen" in WHICH:
    lens = [1, 130, 127, 300, 64, 257]
    toks = unit(sum(lens), 128)
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int64, device="cuda")
    sv, av, _ = mx.score_varlen(Q[:1, :32], toks, cu)
    torch.cuda.synchronize()
    print("varlen ok", float(sv.sum()))
if "exact" in WHICH:
    se, ae, _ = mx.score_dense(Q.float()[:, :32], D.float()[:, :100], torch.clamp(vl, max=100))
    torch.cuda.synchronize()
    print("exact ok", float(se.sum()))
if "quant" in WHICH:
    q8, sc = mx.quant.quantize_tensor(D.reshape(-1, 128))
    torch.cuda.synchronize()
    print("quant ok", int(q8.float().sum()))
if "csr" in WHICH or "grad" in WHICH:
    _, a, _ = mx.score_dense(Q, D, vl)
    off = torch.arange(6, device="cuda", dtype=torch.int64) * 384
    lens = torch.full((6,), 384, device="cuda", dtype=torch.int64)
    for impl in ("doc", "sort"):
        os.environ["MXS_CSR_IMPL"] = impl
        rp, ci, _ = csr_tensors(a, off, lens, 6 * 384, 384)
    os.environ.pop("MXS_CSR_IMPL")
    torch.cuda.synchronize()
    print("csr ok", int(rp[-1]))
    if "grad" in WHICH:
        Qg = Q.clone().requires_grad_(True)
        Dg = D.clone().requires_grad_(True)
        sc = mx.maxsim(Qg, Dg, vl)
        sc.sum().backward()
        torch.cuda.synchronize()
        print("grad ok", float(Qg.grad.float().sum()), float(Dg.grad.float().sum()))
if "topk" in WHICH:
    x = torch.randn(50000, dtype=torch.float64, device="cuda", generator=g)
    ts, ti = mx.topk(x, 20)
    ts2, ti2 = mx.topk(x, 300)
    torch.cuda.synchronize()
    print("topk ok", int(ti[0]), int(ti2[0]))
if "chamfer" in WHICH:
    p = torch.randn(500, 3, device="cuda", generator=g)
    q = torch.randn(400, 3, device="cuda", generator=g)
    cd, a1, a2 = mx.chamfer_forward(p, q)
    dp, dq_ = mx.chamfer_backward(p, q, a1, a2)
    torch.cuda.synchronize()
    print("chamfer ok", cd)
