"""C5 varlen: is the full-corpus bandwidth drop a footprint (TLB / page) effect or a sustained-power
effect?  Answer (profiles/r2_c5_power_probe_gap*.log): power.  With 0.3 s idle before each
measurement every mode runs at ~6.2 TB/s (full 1M-doc launch 6228 GB/s median); back to back
every mode drops to ~5.1-5.4 TB/s.  An in-kernel token-window split (one launch per <= 8 GB) was
also measured: identical per-launch rates under ncu, no gain back to back (not kept).  Same 1M-doc corpus, same total work per timed region (10 launches of 100K docs each):
  same   -- the same 100K-doc slice 10x (7 GB footprint, 13 ms of load)
  chunks -- the 10 consecutive 100K-doc slices (70 GB footprint, 13 ms)
  full   -- one launch over all 1M docs
Prints GB/s for each, interleaved over 3 rounds."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx

g = torch.Generator(device="cuda").manual_seed(0)
rng = np.random.default_rng(0)
n = 1_000_000
lens = rng.integers(32, 513, n)
cu_h = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
T = int(cu_h[-1])
toks = torch.empty(T, 128, dtype=torch.bfloat16, device="cuda")
for i in range(0, T, 8_000_000):
    toks[i:i + 8_000_000] = torch.randn(min(8_000_000, T - i), 128, device="cuda", generator=g).bfloat16()
q = torch.randn(1, 32, 128, device="cuda", generator=g).bfloat16()
cu = torch.from_numpy(cu_h).cuda()
slices = []
for k in range(10):
    d0, d1 = k * 100_000, (k + 1) * 100_000
    t0, t1 = int(cu_h[d0]), int(cu_h[d1])
    slices.append((toks[t0:t1], (cu[d0:d1 + 1] - t0).contiguous(), t1 - t0))


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def run_same():
    tk, c, _ = slices[3]
    for _ in range(10):
        mx.score_varlen(q, tk, c, want_argmax=False, validate=False)


def run_chunks():
    for tk, c, _ in slices:
        mx.score_varlen(q, tk, c, want_argmax=False, validate=False)


def run_full():
    mx.score_varlen(q, toks, cu, want_argmax=False, validate=False)




def run_halves():
    for h in range(2):
        d0, d1 = h * 500_000, (h + 1) * 500_000
        t0 = int(cu_h[d0])
        mx.score_varlen(q, toks[t0:int(cu_h[d1])], (cu[d0:d1 + 1] - t0), want_argmax=False, validate=False)


res = {}
modes = [("same", run_same, 10 * slices[3][2] * 256), ("chunks", run_chunks, T * 256),
         ("full", run_full, T * 256)]
gap = float(os.environ.get("GAP_S", "0.3"))
for r in range(int(os.environ.get("ROUNDS", "3"))):
    k = r % len(modes)
    for name, fn, nbytes in modes[k:] + modes[:k]:  # rotated order: no mode always runs first
        time.sleep(gap)
        ms = timed(fn)
        res.setdefault(name, []).append(nbytes / ms / 1e6)
        print(f"round {r} {name:6s}: {ms:7.3f} ms  {nbytes / ms / 1e6:6.0f} GB/s", flush=True)
for k, v in res.items():
    print(f"{k:6s}: median {np.median(v):6.0f} GB/s  min {min(v):6.0f}  max {max(v):6.0f}")
