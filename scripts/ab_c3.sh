# C3 step (CUDA graph): CSR build overlapped on a side stream vs sequential
for i in 1 2 3; do
timeout 120 python scripts/probe_configs.py 2>&1 | grep "^C3" | sed "s/^/overlap /"
MXS_C3_OVERLAP=0 timeout 120 python scripts/probe_configs.py 2>&1 | grep "^C3" | sed "s/^/sequential /"
done
