# ncu --set full of the final CTA-pair forward at C2 (10K docs): rerank (fused score) and +argmax
mkdir -p gpurun_out
for a in 0 1; do
ARGMAX=$a ROWMAX=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_pair -s 3 -c 1 -o gpurun_out/fwd_a$a -f python scripts/probe_perf.py > gpurun_out/ncu_fwd_a$a.log 2>&1
python scripts/ncu_summary.py gpurun_out/fwd_a$a.ncu-rep gpurun_out/ncu_fwd_a$a.json "ARGMAX=$a ROWMAX=0 ncu --set full --clock-control none -k regex:fwd_pair -s 3 -c 1 python scripts/probe_perf.py" > /dev/null 2>&1
ncu -i gpurun_out/fwd_a$a.ncu-rep --page details > gpurun_out/ncu_fwd_a${a}_details.txt 2>&1
done
python -c "
import json
for a in (0, 1):
    d = json.load(open(f'gpurun_out/ncu_fwd_a{a}.json'))
    print(a, d['gpu__time_duration_us'], d['sm_clock_ghz'], d['tensor_pipe_active_pct'], d['dram_bytes_read'], d['issue_active_pct'])
"
