# split-Q pair mode (two independent cluster groups, TMEM-only pairs) vs the hybrid pair
MXS_PAIR_SPLIT=1 timeout 200 python scripts/probe_pair.py 2>&1 | grep -E "AGREE|MISMATCH"
MXS_PAIR_SPLIT=1 timeout 600 python -m pytest tests -m gpu -q -x -k "fused or acceptance or alternate or certificate or c3" 2>&1 | tail -1
for i in 1 2; do
ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/hybrid /"
MXS_PAIR_SPLIT=1 ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/split /"
ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/hybrid /"
MXS_PAIR_SPLIT=1 ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/split /"
done
