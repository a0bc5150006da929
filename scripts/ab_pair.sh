# C2 +argmax forward: hybrid pair (QB=4, 2 SS blocks) vs TMEM-only pairs (4-CTA clusters, 132 SMs) vs fwd_ts
for i in 1 2; do
ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/pair-hybrid /"
MXS_PAIR_CL=4 ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/pair-cl4 /"
MXS_FWD_IMPL=ts ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/ts /"
MXS_PAIR_CL=4 ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/pair-cl4 /"
done
