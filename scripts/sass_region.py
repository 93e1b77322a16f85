"""Print the SASS of one barrier-delimited region with per-instruction
execution counts (per unit) and stall samples (ncu source page CSV).
usage: python scripts/sass_region.py src.csv.gz REGION [units] [min_count]"""
import csv
import gzip
import io
import re
import sys

f = sys.argv[1]
want = int(sys.argv[2])
div = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
mn = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
txt = gzip.open(f, "rt").read() if f.endswith(".gz") else open(f).read()
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
seg = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    n = int(r[ix["Instructions Executed"]] or 0) / div
    smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    if seg == want and n >= mn:
        print(f"{n:8.2f} {smp:6d}  {src}")
    if re.search(r"\bBAR\.(SYNC|RED|ARV)", src):
        seg += 1
