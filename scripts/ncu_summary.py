"""Summarise one kernel of an ncu --set full report: time, occupancy, issue, pipes, stalls.
Usage: python scripts/ncu_summary.py report.ncu-rep [kernel-regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "raw", "--csv"]
if len(sys.argv) > 2:
    args += ["-k", "regex:" + sys.argv[2]]
rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
hdr, vals = rows[0], rows[2]
d = dict(zip(hdr, vals))
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "launch__occupancy_limit_registers"]
for k in keys:
    print(f"{k:60s} {d.get(k)}")
st = [(float(vals[i].replace(",", "")), h) for i, h in enumerate(hdr)
      if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued") and vals[i] not in ("", "n/a")]
st.sort(reverse=True)
tot = sum(v for v, _ in st) or 1
print("stalls:", ", ".join(f"{h[33:]} {100 * v / tot:.1f}%" for v, h in st[:7]))
