# INT8 rerank: rolled drain loop (value selects) vs per-case unrolled drains
for i in 1 2; do
timeout 60 python scripts/probe_i8.py | sed "s/^/rolled /"
MXS_LIB_PATH=scripts/old_lib/v_i8unroll.so timeout 60 python scripts/probe_i8.py | sed "s/^/unrolled /"
done
MXS_LIB_PATH=scripts/old_lib/v_i8unroll.so timeout 300 python -m pytest tests -m gpu -q -x -k "int8 or i8" 2>&1 | tail -1
