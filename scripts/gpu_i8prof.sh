set -x
mkdir -p gpurun_out
ARGMAX=0 WHICH=int8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_i8 -s 2 -c 1 -o gpurun_out/i8 -f python scripts/probe_int8_varlen.py > gpurun_out/ncu_i8.log 2>&1
python scripts/ncu_hotlines.py gpurun_out/i8.ncu-rep 40 > gpurun_out/i8_hot.txt 2>&1
python scripts/ncu_summary.py gpurun_out/i8.ncu-rep gpurun_out/ncu_i8r.json "int8 rerank (fwd_i8r)" > /dev/null 2>&1
ncu -i gpurun_out/i8.ncu-rep --page details > gpurun_out/ncu_i8r_details.txt 2>/dev/null
