# C3 backward gathers: row-load cache hints and rows in flight per lane group, same box
for i in 1 2; do
timeout 120 python scripts/probe_grad.py | sed "s/^/base /"
for v in gl1 gl2 gl3 gu16 gu4; do MXS_LIB_PATH=scripts/old_lib/v_$v.so timeout 120 python scripts/probe_grad.py | sed "s/^/$v /"; done
done
