"""Instruction mix of an .ncu-rep source page: executed warp-instructions grouped by execution
count (a proxy for loop level / warp role), and the SASS of one group in address order.
Usage: python scripts/ncu_execmix.py REP [EXEC_COUNT]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
pick = int(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = rows[2:]
tot = sum(int(r[idx["Instructions Executed"]] or 0) for r in data)
g = collections.Counter()
n = collections.Counter()
for r in data:
    e = int(r[idx["Instructions Executed"]] or 0)
    g[e] += e
    n[e] += 1
print(f"total executed warp-instructions {tot}")
for e, s in g.most_common(20):
    print(f"  exec {e:>10d} x {n[e]:5d} lines = {s / tot:6.1%}")
if pick is not None:
    ops = collections.Counter()
    for r in data:
        if int(r[idx["Instructions Executed"]] or 0) == pick:
            src = r[idx["Source"]].strip()
            print(f"  {r[idx['Address']][-5:]} {src[:90]}")
            op = src.split()[1] if src.startswith("@") else src.split()[0]
            ops[op.split(".")[0]] += 1
    print(ops.most_common())
