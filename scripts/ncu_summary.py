"""Condense an .ncu-rep (first profiled kernel) into a JSON summary for profiles/.

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep profiles/r1_x_ncu.json "what was run"
"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
cmd = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
d = dict(zip(h, v))


def num(k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None


summary = {
    "kernel": d.get("Kernel Name"),
    "command": cmd,
    "report": rep.split("/")[-1],
    "gpu__time_duration_us": num("gpu__time_duration.sum"),
    "sm_clock_ghz": num("sm__cycles_elapsed.avg.per_second"),
    "registers_per_thread": num("launch__registers_per_thread"),
    "grid": d.get("launch__grid_size"),
    "block": d.get("launch__block_size"),
    "dram_bytes_read": num("dram__bytes_read.sum"),
    "dram_bytes_write": num("dram__bytes_write.sum"),
    "dram_throughput_pct": num("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    "tensor_pipe_active_pct": num("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "pipe_alu_pct": num("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    "pipe_fma_pct": num("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    "pipe_lsu_pct": num("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    "pipe_xu_pct": num("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    "l2_hit_rate_pct": num("lts__t_sector_hit_rate.pct"),
}
# dram byte units: ncu reports in the unit of the column header row 1
units = dict(zip(h, rows[1]))
for k in ("dram_bytes_read", "dram_bytes_write"):
    key = "dram__bytes_read.sum" if k.endswith("read") else "dram__bytes_write.sum"
    u = units.get(key, "byte")
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
    if summary[k] is not None:
        summary[k] *= mult
tunit = units.get("gpu__time_duration.sum", "ns")
if summary["gpu__time_duration_us"] is not None:
    summary["gpu__time_duration_us"] *= {"ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(tunit, 1e-3)
stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(x) for k, x in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
          and x.replace(".", "", 1).isdigit()}
tot = sum(stalls.values()) or 1.0
summary["stall_share"] = {k: round(x / tot, 3) for k, x in sorted(stalls.items(), key=lambda t: -t[1])[:8]}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary, indent=1))
