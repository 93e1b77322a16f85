"""Dynamic SASS opcode histogram of one kernel from an ncu source-page CSV
(ncu -i rep --page source --csv --print-source sass): instructions executed
per opcode, pipe class, and the stall samples."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
tot = 0; h = collections.Counter(); st = collections.Counter(); seq = []
for r in rows[2:]:
    if len(r) < len(hdr): continue
    src = r[ix["Source"]].strip()
    m = re.match(r'(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?', src)
    if not m: continue
    op = m.group(2) + (m.group(3) or '')
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    h[op] += n; st[op] += s; tot += n
    seq.append((r[ix["Address"]], src, n, s))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
print(f"total warp instructions {tot} ({tot/div:.1f} per unit)")
for op, n in h.most_common(45):
    print(f"{n/div:9.1f} {100*n/tot:5.1f}%  stall {st[op]:6d}  {op}")
print("=== per instruction")
if len(sys.argv) > 3:
    for a, s, n, smp in seq:
        if n/div >= float(sys.argv[3]): print(f"{n/div:7.2f} {smp:5d} {s}")
