set -x
mkdir -p gpurun_out
WHICH=varlen timeout 900 ncu --set full --clock-control none --import-source on -k regex:varlen -s 2 -c 1 -o /tmp/vl -f python scripts/probe_int8_varlen.py > gpurun_out/ncu_vl.log 2>&1
python scripts/ncu_hotlines.py /tmp/vl.ncu-rep 40 > gpurun_out/vl_hot.txt 2>&1
ncu -i /tmp/vl.ncu-rep --page source --csv --print-source sass > gpurun_out/vl_src.csv 2>/dev/null
