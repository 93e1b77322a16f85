"""Key metrics of an ncu report (dev aid): python scripts/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__block_size", "launch__grid_size",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "local_load", "sm__cycles_active.avg"]
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, v = rows[0], rows[1], rows[2]
    print("==", rep)
    for name, unit, val in zip(h, u, v):
        if name in KEYS or ("stall" in name and name.endswith("_per_issue_active.ratio") and
                            name.startswith("smsp__average_warps_issue_stalled") and float(val or 0) > 0.2) or \
                ("inst_executed_pipe" in name and name.endswith("avg.pct_of_peak_sustained_active") and float(val or 0) > 5):
            print(f"  {name:75s} {val} {unit}")
