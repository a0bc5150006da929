# INT8 rerank A/B: parity tests, then the C4 kernel with each implementation / debug knob
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "int8 or i8 or quant or two_stage or rerank" 2>&1 | tail -2
for i in 1 2; do
MXS_I8_IMPL=r3 python scripts/probe_i8.py
for d in 0 2 3 4; do MXS_DEBUG=$d python scripts/probe_i8.py; done
done
