# ncu of the CTA-pair forward (rerank, C2 shape) + its cluster count
mkdir -p gpurun_out
MXS_PRINT_GRID=1 MXS_FWD_IMPL=pair ARGMAX=0 NB=2000 REPS=2 python scripts/probe_perf.py 2>&1 | tail -3
MXS_FWD_IMPL=pair ARGMAX=0 NB=2000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_pair -s 2 -c 1 -o gpurun_out/pair -f python scripts/probe_perf.py > gpurun_out/ncu_pair.log 2>&1
python scripts/ncu_hotlines.py gpurun_out/pair.ncu-rep 40 > gpurun_out/pair_hot.txt 2>&1
python scripts/ncu_summary.py gpurun_out/pair.ncu-rep gpurun_out/ncu_pair.json "pair fwd" > /dev/null 2>&1
ncu -i gpurun_out/pair.ncu-rep --page details > gpurun_out/ncu_pair_details.txt 2>/dev/null
