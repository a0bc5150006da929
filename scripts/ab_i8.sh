# fwd_ts INT8 with three accumulator slots: parity, then +argmax and rerank (MXS_I8_IMPL=ts) vs i8r
timeout 900 python -m pytest tests -m gpu -q -x -k "int8 or i8 or quant or two_stage" > /tmp/t.log 2>&1; tail -1 /tmp/t.log
MXS_I8_IMPL=ts timeout 900 python -m pytest tests -m gpu -q -x -k "int8 or i8" > /tmp/t2.log 2>&1; tail -1 /tmp/t2.log
cat > /tmp/t.py <<'PY'
import os, sys, torch
sys.path.insert(0, ".")
import paper_2605_29517_b200 as mx
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(1, 1024, 128, device="cuda", generator=g)
qq, qs = mx.quant.quantize_tensor(x)
dq = torch.randint(-127, 128, (10000, 1024, 128), dtype=torch.int8, device="cuda", generator=g)
ds = torch.rand(10000, 1024, device="cuda", generator=g) * 0.01 + 0.001
def t(f):
    for _ in range(3): f()
    torch.cuda.synchronize(); ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[5]
print(f"int8 +argmax {t(lambda: mx.score_int8(qq, qs, dq, ds, want_argmax=True)):.3f} ms | rerank {t(lambda: mx.score_int8(qq, qs, dq, ds, want_argmax=False)):.3f} ms")
PY
for i in 1 2; do
timeout 120 python /tmp/t.py | sed "s/^/3slot /"
MXS_TS_SLOTS=2 timeout 120 python /tmp/t.py | sed "s/^/2slot /"
MXS_I8_IMPL=ts timeout 120 python /tmp/t.py | sed "s/^/ts-rerank-3slot /"
done
