"""One-paragraph summary per kernel of an ncu --set full report (the lines
kept in profiles/r1_ncu_kernels_summary.txt).
usage: python tools/ncu_summary.py REPORT "LABEL" [KERNEL_REGEX]"""
import csv
import io
import subprocess
import sys

rep, label = sys.argv[1], sys.argv[2]
args = ["ncu", "-i", rep, "--page", "raw", "--csv"]
if len(sys.argv) > 3:
    args += ["--kernel-name", "regex:" + sys.argv[3]]
rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
h = rows[0]
M = {"time": "gpu__time_duration.sum", "regs": "launch__registers_per_thread",
     "warps_active_%": "sm__warps_active.avg.pct_of_peak_sustained_active",
     "issue_active_%": "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "threads_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
     "warp_inst": "smsp__inst_executed.sum", "fp64_pipe_%": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
     "dram_read": "dram__bytes_read.sum", "dram_write": "dram__bytes_write.sum",
     "dram_%": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"}
ST = ["no_instructions", "wait", "branch_resolving", "long_scoreboard", "selected", "not_selected",
      "math_pipe_throttle", "barrier"]
print(f"== {label}")
for v in rows[2:]:
    g = lambda k: v[h.index(k)] if k in h else "-"
    print(f"  kernel: {g('Kernel Name')[:80]}")
    print("    " + ", ".join(f"{k}={g(m)}" for k, m in M.items()))
    st = [f"{s}={g('smsp__pcsamp_warps_issue_stalled_' + s)}" for s in ST]
    print("    stall samples: " + ", ".join(st))
