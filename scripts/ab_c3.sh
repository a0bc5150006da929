# C3 step + autograd backward with the side-stream CSR; parity of the autograd / C3 paths
timeout 900 python -m pytest tests -m gpu -q -x -k "autograd or maxsim or backward or c3 or inbatch or grad or graph" 2>&1 | tail -1
for i in 1 2; do
timeout 120 python scripts/probe_configs.py 2>&1 | grep "^C3" | sed "s/^/overlap /"
MXS_C3_OVERLAP=0 timeout 120 python scripts/probe_configs.py 2>&1 | grep "^C3" | sed "s/^/sequential /"
done
