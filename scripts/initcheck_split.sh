# compute-sanitizer initcheck per kernel family (error counts)
for w in fwd int8 varlen exact quant csr grad topk chamfer; do
  WHICH=$w timeout 600 compute-sanitizer --tool initcheck --print-limit 3 --kernel-name kns=mxs python scripts/sanitize_driver.py > /tmp/ic_$w.log 2>&1
  echo "$w: $(grep 'ERROR SUMMARY' /tmp/ic_$w.log | head -1) $(grep -m1 'Device Frame' /tmp/ic_$w.log)"
done
