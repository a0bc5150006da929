# one gpurun call: GPU parity suite, bench, config probes, ncu captures (args select parts)
set -x
mkdir -p gpurun_out
PARTS="${PARTS:-tests bench probe}"
for p in $PARTS; do
case $p in
tests) timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gpu_tests.log; cat gpurun_out/gpu_tests.log ;;
smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log ;;
bench) timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err ;;
ref) timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json ;;
probe) timeout 600 python scripts/probe_configs.py > gpurun_out/probe_configs.log 2>&1; cat gpurun_out/probe_configs.log ;;
launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1; tail -3 gpurun_out/b_ncu.log ;;
ncu_int8) WHICH=int8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_ts -s 2 -c 1 -o gpurun_out/int8 -f python scripts/probe_int8_varlen.py > gpurun_out/ncu_int8.log 2>&1; tail -3 gpurun_out/ncu_int8.log ;;
ncu_varlen) WHICH=varlen timeout 900 ncu --set full --clock-control none --import-source on -k regex:varlen -s 2 -c 1 -o gpurun_out/varlen -f python scripts/probe_int8_varlen.py > gpurun_out/ncu_varlen.log 2>&1; tail -3 gpurun_out/ncu_varlen.log ;;
ncu_fwd) timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_ts -s 3 -c 1 -o gpurun_out/fwd -f python scripts/probe_perf.py > gpurun_out/ncu_fwd.log 2>&1; tail -3 gpurun_out/ncu_fwd.log ;;
ncu_bwd) timeout 900 ncu --set full --clock-control none --import-source on -k regex:grad -s 2 -c 2 -o gpurun_out/bwd -f python scripts/probe_configs.py > gpurun_out/ncu_bwd.log 2>&1; tail -3 gpurun_out/ncu_bwd.log ;;
*) eval "$p" ;;
esac
done
