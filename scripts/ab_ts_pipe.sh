# fwd_ts bf16 (L_q <= 256; and MXS_FWD_IMPL=ts at L_q = 1024): software-pipelined drain (MXS_TS_PIPE=1) vs default
for i in 1 2 3; do
for a in 0 1; do
LQ=256 ARGMAX=$a ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/base /"
LQ=256 ARGMAX=$a ROWMAX=0 MXS_LIB_PATH=scripts/old_lib/v_tspipe.so timeout 60 python scripts/probe_perf.py | sed "s/^/pipe /"
MXS_FWD_IMPL=ts ARGMAX=$a ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/base-ts1024 /"
MXS_FWD_IMPL=ts ARGMAX=$a ROWMAX=0 MXS_LIB_PATH=scripts/old_lib/v_tspipe.so timeout 60 python scripts/probe_perf.py | sed "s/^/pipe-ts1024 /"
done
done
MXS_LIB_PATH=scripts/old_lib/v_tspipe.so timeout 600 python -m pytest tests -m gpu -q -x -k "dense or alternate or golden or c2 or argmax" 2>&1 | tail -1
