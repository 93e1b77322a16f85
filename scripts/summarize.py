"""Print one line per gpurun_out/bench_*.json (development helper)."""
import glob
import json

for f in sorted(glob.glob("gpurun_out/bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    r = d["roofline"]
    print(f"{d['config']['workload']:16s} {d['config']['spec']:24s} {d['value']:10.0f} Mpx/s  "
          f"{d['ms_per_step']:9.3f} ms  frac {r['frac']:.3f}  redecided {d['redecided_px_per_step']:6d}  "
          f"e2e {(d['e2e'] or {}).get('value')}  cpu {(d['cpu_baseline'] or {}).get('value')}  "
          f"clk {d['clocks']['sm_mhz']}")
