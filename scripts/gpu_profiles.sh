# Refresh the committed evidence: bench line, launch lists, ncu --set full of each hot kernel,
# condensed ON THE BOX (summary JSON + details page) so gpurun_out stays far below 64 MiB.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python scripts/probe_c3.py > /dev/null 2>&1
prof() {  # name, kernel regex, skip, env, command...
  name=$1; rx=$2; skip=$3; shift 3
  timeout 900 env "$@" > gpurun_out/ncu_$name.log 2>&1
  python scripts/ncu_summary.py /tmp/$name.ncu-rep gpurun_out/ncu_$name.json "$*" > /dev/null 2>&1
  ncu -i /tmp/$name.ncu-rep --page details > gpurun_out/ncu_${name}_details.txt 2>/dev/null
  rm -f /tmp/$name.ncu-rep
}
prof fwd fwd_pair 3 ARGMAX=0 ROWMAX=0 ncu --set full --clock-control none -k regex:fwd_pair -s 3 -c 1 -o /tmp/fwd -f python scripts/probe_perf.py
prof fwd_argmax fwd_pair 3 ARGMAX=1 ROWMAX=0 ncu --set full --clock-control none -k regex:fwd_pair -s 3 -c 1 -o /tmp/fwd_argmax -f python scripts/probe_perf.py
prof int8 fwd_i8r 2 ARGMAX=0 WHICH=int8 ncu --set full --clock-control none -k regex:fwd_i8r -s 2 -c 1 -o /tmp/int8 -f python scripts/probe_int8_varlen.py
prof varlen varlen 2 WHICH=varlen ncu --set full --clock-control none -k regex:varlen -s 2 -c 1 -o /tmp/varlen -f python scripts/probe_int8_varlen.py
prof bwd_dd grad_docs 2 ncu --set full --clock-control none -k regex:grad_docs -s 2 -c 1 -o /tmp/bwd_dd -f python scripts/probe_c3.py
prof bwd_dq grad_query 2 ncu --set full --clock-control none -k regex:grad_query -s 2 -c 1 -o /tmp/bwd_dq -f python scripts/probe_c3.py
prof csr csr_doc 2 ncu --set full --clock-control none -k regex:csr_doc -s 2 -c 1 -o /tmp/csr -f python scripts/probe_c3.py
ls -la gpurun_out
