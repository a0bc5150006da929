# C2 rerank: software-pipelined drain in fwd_pair (MXS_PAIR_RERANK_PIPE=1) vs default
for i in 1 2 3 4; do
ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/base /"
MXS_LIB_PATH=scripts/old_lib/v_rpipe.so ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/pipe /"
done
