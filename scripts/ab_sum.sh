# integer fixed-point S4 sums: parity suite, then timings of every fused-sum kernel
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2
for i in 1 2; do
ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/pair /"
MXS_FWD_FUSE=0 ARGMAX=0 ROWMAX=1 timeout 60 python scripts/probe_perf.py | sed "s/^/pair-rowmax+rowsum /"
MXS_FWD_IMPL=ts ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/ts /"
timeout 60 python scripts/probe_i8.py
MXS_FWD_FUSE=0 timeout 60 python scripts/probe_i8.py | sed "s/^/rowmax+rowsum /"
done
timeout 120 python scripts/probe_api_overhead.py | tail -1
