# final evidence at HEAD: GPU tests, bench line, its launch list, config probes, C3 launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1
timeout 600 python scripts/probe_configs.py > gpurun_out/probe_configs.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python scripts/probe_c3.py > gpurun_out/c3_ncu.log 2>&1
cat gpurun_out/gpu_tests.log; head -c 600 gpurun_out/bench.json; echo; tail -12 gpurun_out/probe_configs.log
