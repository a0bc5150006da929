# C4 INT8 +argmax (fwd_ts): software-pipelined drain (MXS_TS_I8_PIPE=1) vs default
for i in 1 2 3; do
ARGMAX=1 timeout 60 python scripts/probe_i8.py | sed "s/^/base /"
ARGMAX=1 MXS_LIB_PATH=scripts/old_lib/v_i8pipe.so timeout 60 python scripts/probe_i8.py | sed "s/^/pipe /"
done
MXS_LIB_PATH=scripts/old_lib/v_i8pipe.so timeout 300 python -m pytest tests -m gpu -q -x -k "int8 or i8" 2>&1 | tail -1
