"""Summarise ncu reports + the launch list into profiles/<tag>_summary.md.
usage: python scripts/make_profile_summary.py TAG launches.csv rep1.ncu-rep [rep2 ...]"""
import collections
import csv
import io
import subprocess
import sys
from pathlib import Path

tag, launches, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
out = [f"# ncu summaries, round {tag}", "",
       "Captured on one B200 (sm_100a, driver 580.159) through `gpurun` with "
       "`ncu --set full --clock-control none --import-source on -k 'regex:dfg_w3_kernel|dfg_fast_kernel' -s 3 -c 1` on "
       "`python bench.py --config <c> --steps 1 --warmup 3 --no-cpu --no-parity --no-table` (the 4th launch: after the 3 warm-up steps), "
       "and the launch list with `--metrics gpu__time_duration.sum,... --clock-control none -c 400` on the default "
       "bench command (`scripts/gpu_profiles.sh`). "
       "Durations under ncu are cold-cache and serialised; the bench numbers come from CUDA events without ncu.", ""]

# launch list shares
rows = list(csv.reader(l for l in open(launches) if not l.startswith("==")))
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    agg[r[ki]][r[mi]].append(float(r[vi].replace(",", "")))
tot = sum(sum(m["gpu__time_duration.sum"]) for m in agg.values())
out += ["## Launch list of the default bench command (C5a: ddf:exact:window=7, 8192x8192)", "",
        "| kernel | launches | mean time (us) | share of GPU time | warp instructions | registers | DRAM read+write per launch |",
        "|---|---|---|---|---|---|---|"]
for k, m in sorted(agg.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
    t = m["gpu__time_duration.sum"]
    dr = (sum(m.get("dram__bytes_read.sum", [0])) + sum(m.get("dram__bytes_write.sum", [0]))) / max(1, len(t))
    out.append(f"| `{k[:90]}` | {len(t)} | {sum(t) / len(t) / 1e3:.1f} | {100 * sum(t) / tot:.1f}% | "
               f"{sum(m.get('smsp__inst_executed.sum', [0])) / len(t):.3g} | "
               f"{m.get('launch__registers_per_thread', ['-'])[0]} | {dr / 1e6:.2f} MB |")
out.append("")
out.append("(`at::vectorized_elementwise_kernel` is bench.py's 256 MiB L2 flush between timed steps, "
           "outside the timed events; `spin_kernel` is the device-side sleep that precedes each start event so the host launch path stays off the measured interval.)")
out.append("")

KEYS = [("gpu__time_duration.sum", "duration"), ("smsp__inst_executed.sum", "warp instructions"),
        ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % of 64"),
        ("launch__registers_per_thread", "registers/thread"), ("launch__block_size", "block"),
        ("launch__grid_size", "grid"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe busy %"),
        ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
        ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1/shared data pipe %"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank-conflict wavefronts"),
        ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write")]
traffic = {}
for rep in reps:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    hh, uu, vv = r[0], r[1], r[2]
    d = {n: (v, u) for n, u, v in zip(hh, uu, vv)}
    name = d.get("Kernel Name", ("?", ""))[0]
    out += [f"## `{Path(rep).stem}`: `{name[:110]}`", "", "| metric | value |", "|---|---|"]
    for k, label in KEYS:
        if k in d:
            out.append(f"| {label} (`{k}`) | {d[k][0]} {d[k][1]} |")
    stalls = sorted(((float(v or 0), n) for n, (v, u) in d.items()
                     if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")),
                    reverse=True)[:6]
    out.append("| top stall reasons (warps per issue) | " +
               ", ".join(f"{n.split('stalled_')[1].split('_per')[0]} {v:.2f}" for v, n in stalls) + " |")
    out.append("")
    try:
        def num(k):
            v, u = d[k]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3,
                     "nsecond": 1e-9, "second": 1, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1, "%": 1}.get(u.strip(), 1)
            return float(v.replace(",", "")) * scale
        traffic[Path(rep).stem.replace("prof_", "")] = {
            "kernel": name, "dram_bytes": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
            "duration_s": num("gpu__time_duration.sum"),
            "fma_pipe_cycles_active_pct": num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "fma_pipe_inst_pct": num("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
            "xu_pipe_inst_pct": num("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active")}
    except (KeyError, ValueError):
        pass
Path(f"profiles/{tag}_summary.md").write_text("\n".join(out) + "\n")
import json  # noqa: E402
Path(f"profiles/{tag}_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
print(f"profiles/{tag}_summary.md", f"profiles/{tag}_traffic.json")
