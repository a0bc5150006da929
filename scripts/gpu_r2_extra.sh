# sanitizers on the forward families (CTA-pair kernel incl. fused score hand-off, fwd_ts, INT8, varlen)
mkdir -p gpurun_out; rm -f gpurun_out/sanitize_pair_summary.log
for tool in memcheck racecheck synccheck; do
  WHICH=fwd,pair,int8,varlen,grad timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 --kernel-name kns=mxs \
    python scripts/sanitize_driver.py > gpurun_out/sanitize_pair_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_pair_summary.log
done
