# CTA-pair forward at C2 (rerank, fused score only): knob A/B
for i in 1 2; do
MXS_FWD_IMPL=ts ARGMAX=0 ROWMAX=0 python scripts/probe_perf.py | sed "s/^/ts /"
ARGMAX=0 ROWMAX=0 python scripts/probe_perf.py | sed "s/^/pair /"
MXS_MMA_SPIN=1 ARGMAX=0 ROWMAX=0 python scripts/probe_perf.py | sed "s/^/pair-spin /"
ARGMAX=1 ROWMAX=0 python scripts/probe_perf.py | sed "s/^/pair /"
MXS_FWD_IMPL=ts ARGMAX=1 ROWMAX=0 python scripts/probe_perf.py | sed "s/^/ts /"
done
