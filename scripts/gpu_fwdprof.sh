set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_ts -s 3 -c 1 -o /tmp/fwd -f python scripts/probe_perf.py > gpurun_out/ncu_fwd.log 2>&1
python scripts/ncu_hotlines.py /tmp/fwd.ncu-rep 80 > gpurun_out/fwd_hot.txt 2>&1
ncu -i /tmp/fwd.ncu-rep --page source --csv --print-source sass > gpurun_out/fwd_src.csv 2>/dev/null
ls -la gpurun_out/fwd_src.csv
