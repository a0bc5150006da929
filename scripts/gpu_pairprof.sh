# ncu of the CTA-pair forward at the C2 shape (2000 docs): rerank vs +argmax
mkdir -p gpurun_out
for a in 0 1; do
ARGMAX=$a ROWMAX=0 NB=2000 timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_pair -s 2 -c 1 -o gpurun_out/pair_a$a -f python scripts/probe_perf.py > gpurun_out/ncu_pair_a$a.log 2>&1
python scripts/ncu_summary.py gpurun_out/pair_a$a.ncu-rep gpurun_out/ncu_pair_a$a.json "pair fwd argmax=$a" > /dev/null 2>&1
done
