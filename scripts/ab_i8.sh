# fwd_ts padded argmax stash: INT8 +argmax and bf16 (L_q = 256, fwd_ts) timings vs the previous build; parity
timeout 900 python -m pytest tests -m gpu -q -x -k "int8 or argmax or fused or alternate or acceptance or c3" 2>&1 | tail -1
cat > /tmp/t.py <<'PY'
import os, sys, torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(1, 1024, 128, device="cuda", generator=g)
qq, qs = mx.quant.quantize_tensor(x)
dq = torch.randint(-127, 128, (10000, 1024, 128), dtype=torch.int8, device="cuda", generator=g)
ds = torch.rand(10000, 1024, device="cuda", generator=g) * 0.01 + 0.001
Q2 = torch.randn(8, 256, 128, device="cuda", generator=g).bfloat16()
D2 = torch.randn(5000, 1024, 128, device="cuda", generator=g).bfloat16()
def t(f):
    for _ in range(3): f()
    torch.cuda.synchronize(); ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[5]
print(f"int8 +argmax {t(lambda: mx.score_int8(qq, qs, dq, ds, want_argmax=True)):.3f} ms | bf16 L_q=256 +argmax {t(lambda: mx.score_dense(Q2, D2)):.3f} ms")
PY
for i in 1 2; do
timeout 120 python /tmp/t.py | sed "s/^/new /"
MXS_LIB_PATH=scripts/old_lib/v_pre_tspad.so timeout 120 python /tmp/t.py | sed "s/^/old /"
done
