# fwd_pair: both accumulators of a set and tile in one drain pipeline (MXS_PAIR_XPIPE=1) vs default; C2 +argmax, C3, C2 rerank
for i in 1 2 3; do
ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/base /"
MXS_LIB_PATH=scripts/old_lib/v_xpipe.so ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/xpipe /"
done
timeout 120 python scripts/probe_configs.py 2>&1 | grep "^C3" | sed "s/^/base /"
MXS_LIB_PATH=scripts/old_lib/v_xpipe.so timeout 120 python scripts/probe_configs.py 2>&1 | grep "^C3" | sed "s/^/xpipe /"
MXS_LIB_PATH=scripts/old_lib/v_xpipe.so timeout 600 python -m pytest tests -m gpu -q -x -k "pair or argmax or c2 or c3 or dense or golden or alternate" 2>&1 | tail -1
for i in 1 2 3; do
ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/base /"
MXS_LIB_PATH=scripts/old_lib/v_xpipe.so ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/xpipe /"
done
