# INT8 rerank A/B: bias written by a kind::f16 MMA (default) vs by the epilogue's tcgen05.st (MXS_I8_ST_BIAS=1)
for i in 1 2 3; do
timeout 60 python scripts/probe_i8.py | sed "s/^/mma-bias /"
MXS_LIB_PATH=scripts/old_lib/v_stbias.so timeout 60 python scripts/probe_i8.py | sed "s/^/st-bias /"
done
MXS_DEBUG=2 timeout 60 python scripts/probe_i8.py | sed "s/^/mma-bias /"
MXS_DEBUG=2 MXS_LIB_PATH=scripts/old_lib/v_stbias.so timeout 60 python scripts/probe_i8.py | sed "s/^/st-bias /"
MXS_LIB_PATH=scripts/old_lib/v_stbias.so timeout 300 python -m pytest tests -m gpu -q -x -k "int8 or i8" 2>&1 | tail -1
