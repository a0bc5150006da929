"""CTA-pair forward (MXS_FWD_IMPL=pair) vs fwd_ts: agreement on a few shapes, then C2 timings
(rerank = fused score only, +argmax) under the MXS_DEBUG knobs."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_29517_b200 import _lib  # noqa: E402

st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731


def run(Q, D, vl, argmax, impl, rowmax=False):
    os.environ["MXS_FWD_IMPL"] = impl
    nq, lq, d = Q.shape
    nb, lp, _ = D.shape
    s = torch.empty(nq, nb, dtype=torch.float64, device="cuda")
    am = torch.empty(nq, nb, lq, dtype=torch.int32, device="cuda") if argmax else None
    rm = torch.empty(nq, nb, lq, dtype=torch.float32, device="cuda") if rowmax else None
    _lib.call("mxs_fused_score_batch", _lib.MXS_BF16 if Q.dtype == torch.bfloat16 else _lib.MXS_F16, P(Q), nq, lq,
              P(D), nb, lp, d, P(vl), P(s), P(am), P(rm), 0, st)
    return s, am, rm


g = torch.Generator(device="cuda").manual_seed(0)
ok = True
for (nq, lq, nb, lp, d, dt) in [(1, 1024, 50, 1024, 128, torch.bfloat16), (3, 1000, 37, 300, 128, torch.bfloat16),
                                 (2, 512, 20, 256, 128, torch.float16), (2, 700, 9, 130, 64, torch.bfloat16),
                                 (4, 384, 33, 1024, 96, torch.bfloat16)]:
    Q = torch.randn(nq, lq, d, device="cuda", generator=g).to(dt)
    D = torch.randn(nb, lp, d, device="cuda", generator=g).to(dt)
    vl = torch.randint(1, lp + 1, (nb,), device="cuda", generator=g, dtype=torch.int32)
    vl[0] = lp
    for am_ in (False, True):
        s0, a0, r0 = run(Q, D, vl, am_, "ts", rowmax=True)
        s1, a1, r1 = run(Q, D, vl, am_, "pair", rowmax=True)
        torch.cuda.synchronize()
        rel = ((s1 - s0).abs() / s0.abs().clamp_min(1e-9)).max().item()
        same_rm = torch.equal(r0, r1)
        same_am = torch.equal(a0, a1) if am_ else True
        good = rel < 1e-6 and same_rm and same_am
        ok &= good
        print(f"shape nq={nq} lq={lq} nb={nb} lp={lp} d={d} {dt} argmax={am_}: rel={rel:.2e} rowmax_eq={same_rm} "
              f"argmax_eq={same_am} {'OK' if good else 'MISMATCH'}")
print("AGREE" if ok else "DISAGREE")

nb = 10000
Q = torch.randn(1, 1024, 128, device="cuda", generator=g).bfloat16()
D = torch.randn(nb, 1024, 128, device="cuda", generator=g).bfloat16()
fl = 2 * 1024 * 1024 * 128 * nb


def timeit(f, reps=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


Q5 = torch.randn(1, 512, 128, device="cuda", generator=g).bfloat16()
for impl in ("ts", "pair"):
    for am_ in (False, True):
        t = timeit(lambda: run(Q5, D, None, am_, impl))
        print(f"L_q=512 {impl:4s} argmax={int(am_)}: {t:.3f} ms {fl / 2 / t / 1e9:.0f} TFLOP/s")
os.environ["MXS_PAIR_CL"] = "4"
for am_ in (False, True):
    t = timeit(lambda: run(Q, D, None, am_, "pair"))
    print(f"C2 pair(2 pairs/cluster, CL=4) argmax={int(am_)}: {t:.3f} ms {fl / t / 1e9:.0f} TFLOP/s")
os.environ["MXS_PAIR_CL"] = "2"
for impl in ("ts", "pair"):
    for dbg in (("0",) if os.environ.get("QUICK") else ("0", "2", "3")):
        os.environ["MXS_DEBUG"] = dbg
        for am_ in (False, True):
            if dbg == "3" and am_:
                continue
            t = timeit(lambda: run(Q, D, None, am_, impl))
            print(f"C2 {impl:4s} debug={dbg} argmax={int(am_)}: {t:.3f} ms {fl / t / 1e9:.0f} TFLOP/s")
os.environ["MXS_DEBUG"] = "0"
