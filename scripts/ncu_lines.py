"""Per-source-line instruction / stall summary of an ncu report (dev aid).
usage: python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
data, fname = [], ""
for r in rows:
    if len(r) == 2 and r[0] in ("File Path",):
        fname = r[1].split("/")[-1]
    if len(r) > 8 and r[0] != "Line No":
        try:
            data.append((int(r[7] or 0), float(r[4] or 0), f"{fname}:{r[0]}", r[1][:90]))
        except ValueError:
            pass
ti = sum(d[0] for d in data) or 1
ts = sum(d[1] for d in data) or 1
print(f"total warp-instructions {ti}, stall samples {ts:.0f}")
for d in sorted(data, key=lambda x: -x[0])[:top]:
    print(f"{100*d[0]/ti:5.1f}% inst {100*d[1]/ts:5.1f}% stall {d[2]:>18s}  {d[3]}")
