# ncu --set full of the final quantiser and backward gathers
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quantize128 -s 2 -c 1 -o gpurun_out/quant_final -f python scripts/probe_quant.py > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/quant_final.ncu-rep gpurun_out/r2_ncu_quant.json "ncu --set full -k regex:quantize128 -s 2 -c 1 python scripts/probe_quant.py" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grad_ -s 2 -c 2 -o gpurun_out/grad_final -f python scripts/probe_grad.py > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/grad_final.ncu-rep gpurun_out/r2_ncu_grad_final.json "ncu --set full -k regex:grad_ -s 2 -c 2 python scripts/probe_grad.py" > /dev/null 2>&1
python -c "
import json
for f in ('gpurun_out/r2_ncu_quant.json', 'gpurun_out/r2_ncu_grad_final.json'):
    d = json.load(open(f))
    ds = d if isinstance(d, list) else [d]
    for x in ds:
        print(f, x.get('kernel','?')[:60], x.get('gpu__time_duration_us'), x.get('dram_bytes_read'), x.get('dram_bytes_write'), x.get('l2_hit_rate_pct'))
"
