"""Per-source-line warp-instruction counts (per output pixel) of one kernel in
an ncu report (dev aid).  usage: python scripts/ncu_lines2.py rep kernel_regex n_px [min_per_px]"""
import collections
import csv
import subprocess
import sys

rep, kre, npx = sys.argv[1], sys.argv[2], float(sys.argv[3])
thr = float(sys.argv[4]) if len(sys.argv) > 4 else 2.0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
out, fname = [], ""
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("Line No", "#", "Address"):
        try:
            out.append((fname, int(r[0]), int(r[7] or 0), r[1][:110]))
        except ValueError:
            pass
tot = sum(o[2] for o in out)
print(f"total {tot} warp-inst = {tot * 32 / npx:.1f} thread-inst/px")
byf = collections.Counter()
for f, _, n, _ in out:
    byf[f] += n
print({k: round(v * 32 / npx, 1) for k, v in byf.items()})
for f, ln, n, s in sorted(out, key=lambda o: (o[0], o[1])):
    if n * 32 / npx > thr:
        print(f"{f}:{ln:4d} {n * 32 / npx:6.1f}/px  {s}")
