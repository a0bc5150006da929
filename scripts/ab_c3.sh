# C3 step: dD on the side stream concurrent with dQ (default) vs dD after dQ (MXS_C3_CONCURRENT=0)
timeout 900 python -m pytest tests -m gpu -q -x -k "autograd or maxsim or backward or c3 or inbatch or grad or graph" 2>&1 | tail -1
for i in 1 2 3; do
timeout 120 python scripts/probe_configs.py 2>&1 | grep "^C3" | sed "s/^/concurrent /"
MXS_C3_CONCURRENT=0 timeout 120 python scripts/probe_configs.py 2>&1 | grep "^C3" | sed "s/^/sequential /"
done
