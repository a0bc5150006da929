# INT8 rerank / fwd_ts: HEAD (old DSMEM hand-off in i8r) vs bulk-copy hand-off
for i in 1 2; do
for v in head i8bulk; do
MXS_LIB_PATH=scripts/old_lib/v_$v.so timeout 60 python scripts/probe_i8.py | sed "s/^/$v /"
MXS_LIB_PATH=scripts/old_lib/v_$v.so MXS_FWD_IMPL=ts ARGMAX=0 ROWMAX=0 timeout 60 python scripts/probe_perf.py | sed "s/^/$v ts /"
done
done
