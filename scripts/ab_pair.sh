# +argmax paths after dropping the warp vote: parity (argmax everywhere) and timings
timeout 900 python -m pytest tests -m gpu -q -x -k "argmax or alternate or c3 or acceptance or fused or int8 or varlen or grad or csr" 2>&1 | tail -1
for i in 1 2; do
ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/pair /"
MXS_FWD_IMPL=ts ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/ts /"
done
timeout 120 python scripts/probe_configs.py 2>&1 | grep -E "^C3|^C4 int8"
