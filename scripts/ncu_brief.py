"""Brief of an ncu raw CSV (scripts/gpu_prof.sh): key utilisations + top stalls.
usage: python scripts/ncu_brief.py gpurun_out/raw_c5a.csv [...]"""
import csv
import io
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]
for f in sys.argv[1:]:
    r = list(csv.reader(io.StringIO(open(f).read())))
    h, u, v = r[0], r[1], r[2]
    d = {n: (val, un) for n, un, val in zip(h, u, v)}
    print("==", f, d.get("Kernel Name", ("?",))[0][:100])
    for k in KEYS:
        if k in d:
            print(f"  {k:70s} {d[k][0]} {d[k][1]}")
    st = sorted(((float(val or 0), n) for n, (val, un) in d.items()
                 if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")),
                reverse=True)[:9]
    print("  stalls: " + ", ".join(f"{n.split('stalled_')[1].split('_per')[0]} {x:.2f}" for x, n in st))
