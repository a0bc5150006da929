import torch, time
n = 2_621_440_000 // 2
h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
def run(nstreams, chunks):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    per = n // chunks
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for c in range(chunks):
        s = ss[c % nstreams]
        s.wait_event(e0)
        with torch.cuda.stream(s):
            d[c * per:(c + 1) * per].copy_(h[c * per:(c + 1) * per], non_blocking=True)
    for s in ss:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return n * 2 / e0.elapsed_time(e1) / 1e6
for cfg in [(1, 10), (2, 10), (4, 20), (1, 1), (2, 2)]:
    print(cfg, [round(run(*cfg), 1) for _ in range(3)], "GB/s")
