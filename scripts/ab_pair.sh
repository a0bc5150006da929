# C2 forward, same box: integer partials deferred vs at document end
for i in 1 2; do
ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/deferred /"
MXS_LIB_PATH=scripts/old_lib/v_nodefer.so ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/doc-end /"
MXS_DEBUG=9 ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/no-partial /"
ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/deferred /"
MXS_LIB_PATH=scripts/old_lib/v_nodefer.so ARGMAX=1 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/doc-end /"
done
