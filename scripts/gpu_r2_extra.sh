# sanitizers on the forward family (CTA-pair kernel) + the CSR ncu capture
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  WHICH=pair timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 --kernel-name kns=mxs \
    python scripts/sanitize_driver.py > gpurun_out/sanitize_pair_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_pair_summary.log
done
# timeout 900 ncu --set full --clock-control none -k regex:csr_doc -s 2 -c 1 -o /tmp/csr -f python scripts/probe_c3.py > gpurun_out/ncu_csr.log 2>&1
# python scripts/ncu_summary.py /tmp/csr.ncu-rep gpurun_out/ncu_csr.json "ncu --set full -k regex:csr_doc probe_c3.py" > /dev/null 2>&1
# ncu -i /tmp/csr.ncu-rep --page details > gpurun_out/ncu_csr_details.txt 2>/dev/null
