# compute-sanitizer over scripts/sanitize_driver.py, one tool at a time; logs -> gpurun_out/sanitize_*.log
mkdir -p gpurun_out; rm -f gpurun_out/sanitize_summary.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    --kernel-name kns=mxs \
    python scripts/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.log
  tail -4 gpurun_out/sanitize_$tool.log
done
