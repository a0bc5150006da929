"""GPU probe: tensor-core / exact forward vs a torch fp32 reference, plus a C2 timing."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2605_29517_b200 import _lib  # noqa: E402

L = _lib.load()
print(L.mxs_version().decode(), "SMs", L.mxs_device_sm_count())


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def unit(shape, dtype, gen):
    x = torch.randn(*shape, device="cuda", generator=gen)
    x = x / x.norm(dim=-1, keepdim=True)
    return x.to(dtype)


def torch_ref(Q, D, vl):
    Qf, Df = Q.float(), D.float()
    S = torch.einsum("qid,bjd->qbij", Qf, Df)
    j = torch.arange(D.shape[1], device="cuda")
    S = S.masked_fill(j[None, None, None, :] >= vl[None, :, None, None], float("-inf"))
    m, a = S.max(dim=-1)
    top2 = S.topk(2, dim=-1).values if D.shape[1] > 1 else None
    gap = (top2[..., 0] - top2[..., 1]) if top2 is not None else torch.full_like(m, 1.0)
    return m, a.int(), gap, m.double().sum(-1)


def run(Q, D, vl, exact=0, dtype=_lib.MXS_BF16):
    nq, lq, d = Q.shape
    nb, lp, _ = D.shape
    scores = torch.empty(nq, nb, dtype=torch.float64, device="cuda")
    am = torch.empty(nq, nb, lq, dtype=torch.int32, device="cuda")
    rm = torch.empty(nq, nb, lq, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("mxs_fused_score_batch", dtype, ptr(Q), nq, lq, ptr(D), nb, lp, d, ptr(vl), ptr(scores), ptr(am),
              ptr(rm), exact, ctypes.c_void_p(st))
    torch.cuda.synchronize()
    return scores, am, rm


def check(name, nq, lq, nb, lp, d, dtype=torch.bfloat16, ragged=True, exact=0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    Q = unit((nq, lq, d), dtype, g)
    D = unit((nb, lp, d), dtype, g)
    if ragged:
        vl = torch.randint(1, lp + 1, (nb,), device="cuda", generator=g, dtype=torch.int32)
        vl[0] = lp
    else:
        vl = torch.full((nb,), lp, dtype=torch.int32, device="cuda")
    # zero padding like DocBatch
    j = torch.arange(lp, device="cuda")
    D = D.masked_fill((j[None, :] >= vl[:, None])[..., None], 0)
    mxdt = {torch.bfloat16: _lib.MXS_BF16, torch.float16: _lib.MXS_F16, torch.float32: _lib.MXS_F32}[dtype]
    try:
        s, a, r = run(Q, D, vl, exact=exact, dtype=mxdt)
    except Exception as e:  # noqa: BLE001
        print(f"[{name}] ERROR {type(e).__name__}: {e}")
        return False
    m, ra, gap, rs = torch_ref(Q, D, vl)
    rel = ((s - rs).abs() / rs.abs().clamp_min(1e-30)).max().item()
    mdiff = (r - m).abs().max().item()
    safe = gap > 1e-5
    mism = ((a != ra) & safe).sum().item()
    ok = rel < 1e-3 and mism == 0
    print(f"[{name}] {'OK ' if ok else 'BAD'} score_rel={rel:.2e} rowmax_absdiff={mdiff:.2e} argmax_mism={mism} "
          f"(excluded near-ties {(~safe).sum().item()}/{safe.numel()})")
    return ok


allok = True
allok &= check("exact f32 small", 2, 32, 16, 180, 128, torch.float32, exact=1)
allok &= check("tc bf16 tiny", 1, 128, 4, 128, 128)
allok &= check("tc bf16 lq1024", 1, 1024, 24, 1024, 128)
allok &= check("tc bf16 multi-q", 4, 300, 40, 260, 128)
allok &= check("tc bf16 lq32 lp180", 3, 32, 50, 180, 128)
allok &= check("tc f16 d64", 2, 200, 30, 333, 64, torch.float16)
allok &= check("tc bf16 d256", 2, 520, 20, 400, 256)
allok &= check("tc bf16 d96", 1, 130, 10, 129, 96)
allok &= check("exact bf16", 2, 40, 10, 77, 128, torch.bfloat16, exact=1)
print("ALL_OK" if allok else "SOME_BAD")

# ---- C2 timing
g = torch.Generator(device="cuda").manual_seed(1)
nb = 10000
Q = unit((1, 1024, 128), torch.bfloat16, g)
D = torch.empty(nb, 1024, 128, dtype=torch.bfloat16, device="cuda")
for i in range(0, nb, 1000):
    D[i:i + 1000] = unit((1000, 1024, 128), torch.bfloat16, g)
scores = torch.empty(1, nb, dtype=torch.float64, device="cuda")
am = torch.empty(1, nb, 1024, dtype=torch.int32, device="cuda")
rm = torch.empty(1, nb, 1024, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def go(with_arg=True):
    _lib.call("mxs_fused_score_batch", _lib.MXS_BF16, ptr(Q), 1, 1024, ptr(D), nb, 1024, 128, None, ptr(scores),
              ptr(am) if with_arg else None, ptr(rm), 0, ctypes.c_void_p(st))


for _ in range(3):
    go()
torch.cuda.synchronize()
for wa in (True, False):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        e0.record()
        go(wa)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[len(ts) // 2]
    flops = 2 * 1024 * 1024 * 128 * nb
    print(f"C2 argmax={wa}: {t:.3f} ms  {nb / t * 1e3 / 1e6:.3f} M docs/s  {flops / t / 1e9:.1f} TFLOP/s "
          f"({flops / t / 1e9 / 1625.7 * 100:.1f}% of measured bf16 peak)")
# spot check C2 sample
m, ra, gap, rs = torch_ref(Q, D[:64], torch.full((64,), 1024, dtype=torch.int32, device="cuda"))
go()
torch.cuda.synchronize()
print("C2 sample score rel", ((scores[:, :64] - rs).abs() / rs.abs()).max().item(),
      "argmax mism", ((am[:, :64] != ra) & (gap > 1e-5)).sum().item())
