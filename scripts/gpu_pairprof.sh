# ncu of the CTA-pair forward (rerank, C2 shape): full kernel vs raw pipeline (MXS_DEBUG=3)
mkdir -p gpurun_out
for d in 0 2 3; do
MXS_DEBUG=$d ARGMAX=0 ROWMAX=0 NB=2000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_pair -s 2 -c 1 -o gpurun_out/pair_d$d -f python scripts/probe_perf.py > gpurun_out/ncu_pair_d$d.log 2>&1
python scripts/ncu_summary.py gpurun_out/pair_d$d.ncu-rep gpurun_out/ncu_pair_d$d.json "pair fwd debug=$d" > /dev/null 2>&1
done
