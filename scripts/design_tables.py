"""Regenerate DESIGN.md's measurement tables from gpurun_out/bench_<c>.json
(+ cpu_<c>.json CPU baselines, profiles/r01_traffic.json DRAM bytes)."""
import json
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
G = ROOT / "gpurun_out"


def load(f):
    return json.loads((G / f).read_text().strip().splitlines()[-1])


def f(x):
    return f"{x:,.0f}".replace(",", " ")


p = ROOT / "DESIGN.md"
s = p.read_text()
t = json.loads((ROOT / "profiles/r01_traffic.json").read_text())
alg = {"c1": 512 * 512 * 6, "c2": 1024 * 1024 * 6, "c3": 2048 * 2048 * 6, "c5a": 8192 * 8192 * 6,
       "c5b": 64 * 1920 * 1080 * 6}
rows = [("c1", "C1 512²", "bvdf:exact"), ("c2", "**C2 1024²**", "**ddf:exact**"), ("c3", "C3 2048²", "acwddf:exact:window=5"),
        ("c4_bvdf_minimax", "C4 4096²", "bvdf:minimax:window=5"), ("c4_bvdf_rgb", "C4", "bvdf:rgb:window=5"),
        ("c4_ddf_minimax", "C4", "ddf:minimax:window=5"), ("c4_ddf_rgb", "C4", "ddf:rgb:window=5"),
        ("c5a", "C5a 8192²", "ddf:exact:window=7"), ("c5b", "C5b 64×1080p", "acwddf:exact")]
i0 = s.index("| config | spec | Mpx/s | frac of FP32 roofline | e2e Mpx/s | sync Mpx/s |")
i1 = s.index("CPU baseline beside every config")
L = ["| config | spec | Mpx/s | frac of FP32 roofline | e2e Mpx/s | sync Mpx/s | re-decided px/step | DRAM B/launch (ncu) vs algorithmic |",
     "|---|---|---|---|---|---|---|---|"]
for c, name, spec in rows:
    d = load(f"bench_{c}.json")
    e = d.get("e2e") or {}
    sc = (e.get("sync_call") or {}).get("value")
    v, fr, ev = f(d["value"]), f"{d['roofline']['frac']:.3f}", f(e["value"])
    if c == "c2":
        v, fr, ev = f"**{v}**", f"**{fr}**", f"**{ev}**"
    tt = t[c]
    dr = f"{tt['dram_bytes'] / 1e6:.2f} MB / {alg.get(c, 4096 * 4096 * 6) / 1e6:.2f} MB"
    L.append(f"| {name} | {spec} | {v} | {fr} | {ev} | {f(sc) if sc else '—'} | {d['redecided_px_per_step']} | {dr} |")
s = s[:i0] + "\n".join(L) + "\n\n" + s[i1:]
j0 = s.index("| config | CPU Mpx/s (16 threads) |")
j1 = s.index("Run-to-run spread on fresh boxes this round:")
L = ["| config | CPU Mpx/s (16 threads) | device Mpx/s | e2e Mpx/s | device ÷ CPU | e2e ÷ CPU |", "|---|---|---|---|---|---|"]
for c, name, _ in rows:
    name = name.replace("*", "").split(" ")[0] + ("" if not c.startswith("c4") else " " + c[3:].replace("_", ":"))
    cpu = (load("bench_c2.json") if c == "c2" else load(f"cpu_{c}.json"))["cpu_baseline"]["value"]
    m = load(f"bench_{c}.json")
    v, e = m["value"], m["e2e"]["value"]
    L.append(f"| {name} | {cpu:.2f} | {f(v)} | {f(e)} | {f(v / cpu)}× | {f(e / cpu)}× |")
s = s[:j0] + "\n".join(L) + "\n\n" + s[j1:]
p.write_text(s)
print("ok")
