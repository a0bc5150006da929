"""Summarise an ncu --metrics gpu__time_duration.sum launch list: count, mean us, share per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
d = collections.defaultdict(list)
for r in rows[i + 1:]:
    rr = dict(zip(h, r))
    if rr.get("Metric Name") == "gpu__time_duration.sum":
        name = rr["Kernel Name"]
        if "mxs" not in name and "--all" not in sys.argv:
            continue
        d[name[:90]].append(float(rr["Metric Value"]) / 1e3)
tot = sum(sum(v) for v in d.values())
print(f"{'n':>4} {'mean_us':>10} {'share':>6}  kernel")
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{len(v):>4} {sum(v) / len(v):>10.1f} {sum(v) / tot:>6.3f}  {k}")
