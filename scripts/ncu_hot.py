"""Hot SASS lines of an ncu source page CSV (--page source --csv --print-source sass)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = rows[2:]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
inst = sum(int(r[idx["Instructions Executed"]] or 0) for r in data)
print("total samples", tot, "warp-instructions", inst)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
if "--mix" in sys.argv:
    import collections
    c = collections.Counter()
    for r in data:
        op = r[idx["Source"]].split()[0] if r[idx["Source"]].split() else "?"
        if op.startswith("@"):
            op = r[idx["Source"]].split()[1]
        c[op.split(".")[0]] += int(r[idx["Instructions Executed"]] or 0)
    for k, x in c.most_common(30):
        print(f"{k:12s} {x:>12d} {x / inst:6.1%}")
    sys.exit()
top = sorted(data, key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))[:n]
for r in top:
    print(f"{r[idx['Address']][-5:]} {int(r[idx['Warp Stall Sampling (All Samples)']]):6d} "
          f"{int(r[idx['Instructions Executed']] or 0):9d}  {r[idx['Source']].strip()[:90]}")
