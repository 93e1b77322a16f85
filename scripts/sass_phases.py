"""Attribute a kernel's dynamic instructions and stall samples to the
barrier-delimited regions of its SASS (barrier waits to the region the
barrier ends -- see the note at stall_barrier below) (ncu source page CSV, scripts/gpu_prof.sh).
usage: python scripts/sass_phases.py src_c5a.csv.gz [units]"""
import collections
import csv
import gzip
import io
import re
import sys

f = sys.argv[1]
txt = gzip.open(f, "rt").read() if f.endswith(".gz") else open(f).read()
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
seg = 0
segs = collections.defaultdict(lambda: {"n": 0, "s": 0, "ops": collections.Counter(), "st": collections.Counter(),
                                        "first": None})
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    m = re.match(r'(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?', src)
    op = (m.group(2) + (m.group(3) or "")) if m else src[:12]
    d = segs[seg]
    if d["first"] is None:
        d["first"] = r[ix["Address"]]
    d["n"] += n
    d["s"] += s
    d["ops"][op] += n
    for c in stall_cols:
        v = int(r[ix[c]] or 0)
        # BAR.SYNC.DEFER_BLOCKING lets a warp run on past the barrier until its
        # first blocking (memory) instruction, and that is where a warp waiting
        # for the barrier is sampled: barrier-stall samples belong to the
        # region the barrier ENDS, i.e. the previous one
        if c == "stall_barrier" and seg > 0 and not op.startswith("BAR."):
            segs[seg - 1]["st"]["barrier"] += v
            segs[seg - 1]["s"] += v
            d["s"] -= v
            continue
        d["st"][c[6:]] += v
    if op.startswith("BAR.SYNC") or op.startswith("BAR.RED") or op.startswith("BAR.ARV"):
        seg += 1
N = sum(d["n"] for d in segs.values())
S = sum(d["s"] for d in segs.values())
for k, d in segs.items():
    if d["n"] == 0 and d["s"] == 0:
        continue
    print(f"region {k:3d} @{d['first']}: inst {d['n'] / div:10.1f} ({100 * d['n'] / N:5.1f}%)  stall samples "
          f"{100 * d['s'] / S:5.1f}%")
    print("    top ops: " + ", ".join(f"{o} {n / div:.0f}" for o, n in d["ops"].most_common(8)))
    print("    stalls:  " + ", ".join(f"{o} {100 * n / max(1, d['s']):.0f}%" for o, n in d["st"].most_common(6)))
