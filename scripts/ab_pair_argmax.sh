# C2 +argmax and C3 forward: software-pipelined argmax drain in fwd_pair (MXS_PAIR_ARGMAX_PIPE=1) vs default
for i in 1 2 3; do
ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/base /"
MXS_LIB_PATH=scripts/old_lib/v_apipe.so ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/pipe /"
done
timeout 120 python scripts/probe_configs.py 2>&1 | grep "^C3" | sed "s/^/base /"
MXS_LIB_PATH=scripts/old_lib/v_apipe.so timeout 120 python scripts/probe_configs.py 2>&1 | grep "^C3" | sed "s/^/pipe /"
MXS_LIB_PATH=scripts/old_lib/v_apipe.so timeout 600 python -m pytest tests -m gpu -q -x -k "pair or argmax or c2 or c3 or dense or golden or alternate" 2>&1 | tail -1
