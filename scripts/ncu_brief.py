"""Key counters of an .ncu-rep (first kernel): duration, clocks, pipes, issue, stalls, DRAM."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, v = r[0], r[2]
d = dict(zip(h, v))
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for k in keys:
    for kk in d:
        if kk.startswith(k):
            print(f"{kk:80s} {d[kk]}")
            break
st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(x)) for k, x in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and x.replace('.', '', 1).isdigit()]
tot = sum(x for _, x in st) or 1
print("stalls:", ", ".join(f"{k} {x / tot:.0%}" for k, x in sorted(st, key=lambda t: -t[1])[:8]))
