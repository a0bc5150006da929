# C2 forward: distributed certified partial sums
for i in 1 2; do
ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/partials /"
MXS_DEBUG=6 ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/no-handoff /"
ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/partials /"
done
timeout 600 python -m pytest tests -m gpu -q -x -k "fused or rerank or acceptance or alternate or certificate" 2>&1 | tail -2
timeout 200 python scripts/probe_pair.py 2>&1 | grep -E "AGREE|MISMATCH"
