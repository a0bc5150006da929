# C2 +argmax forward: padded stash (immediate offsets) -- parity, then timing
timeout 200 python scripts/probe_pair.py 2>&1 | grep -E "AGREE|MISMATCH"
timeout 600 python -m pytest tests -m gpu -q -x -k "argmax or acceptance or alternate or c3 or fused" 2>&1 | tail -1
for i in 1 2; do
ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/pair /"
MXS_FWD_IMPL=ts ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/ts /"
ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/pair /"
done
timeout 120 python scripts/probe_configs.py 2>&1 | grep "^C3"
