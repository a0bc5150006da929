"""Top SASS lines by stall samples from an .ncu-rep (source page), with per-line stall reasons,
plus samples grouped by execution count (a proxy for warp role / loop level)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = rows[2:]
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
S = "Warp Stall Sampling (All Samples)"
tot = sum(int(r[idx[S]] or 0) for r in data) or 1
print(f"total samples {tot}")
groups = collections.defaultdict(collections.Counter)
for r in data:
    e = int(r[idx["Instructions Executed"]] or 0)
    for k in reasons:
        groups[e][k[6:]] += int(r[idx[k]] or 0)
print("by execution count:")
for e, c in sorted(groups.items(), key=lambda x: -sum(x[1].values()))[:12]:
    s = sum(c.values())
    print(f"  exec {e:>10d}: {s / tot:6.1%}  " + ", ".join(f"{k}={v}" for k, v in c.most_common(4)))
print("top lines:")
for r in sorted(data, key=lambda r: -int(r[idx[S]] or 0))[:n]:
    c = collections.Counter({k[6:]: int(r[idx[k]] or 0) for k in reasons})
    print(f"  {r[idx['Address']][-5:]} {int(r[idx[S]]):6d} {int(r[idx['Instructions Executed']] or 0):>10d}  "
          f"{r[idx['Source']].strip()[:70]:70s} {c.most_common(2)}")
