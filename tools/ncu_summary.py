"""Compact per-kernel summary of an `ncu --set full` report (profiles/*.txt):
python tools/ncu_summary.py report.ncu-rep [title]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
KEYS = {
    "gpu__time_duration.sum": "time_us",
    "dram__bytes_read.sum": "dram_read_MB",
    "dram__bytes_write.sum": "dram_write_MB",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
}
UNIT = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
units = rows[1]
print(f"{title}\n")
for r in rows[2:]:
    name = r[h.index("Kernel Name")][:70]
    vals = {}
    for k, short in KEYS.items():
        if k in h:
            i = h.index(k)
            try:
                vals[short] = float(r[i].replace(",", "")) * UNIT.get(units[i], 1.0)
            except ValueError:
                pass
    stalls = {}
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(r[i])
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
    print(name)
    print("  " + ", ".join(f"{k}={v:.1f}" for k, v in vals.items()))
    print("  stalls (cycles/issue): " + ", ".join(f"{k} {v:.2f} ({v / tot:.0%})" for k, v in top) + "\n")
