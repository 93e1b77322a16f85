"""Attribute an ncu SASS source-page CSV (per-instruction executed counts and
stall samples) to CUDA source lines via nvdisasm -g of the kernel's cubin.
usage: sass_lines.py <ncu_sass.csv> <object.o> <mangled-kernel-substring> [div]"""
import csv, sys, re, subprocess, tempfile, os, collections, glob
csvp, obj, kname = sys.argv[1:4]
div = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
rows = list(csv.reader(open(csvp)))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
recs = [r for r in rows[2:] if len(r) >= len(hdr)]
base = int(recs[0][ix["Address"]], 16)
td = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
cub = glob.glob(td + "/*.cubin")[0]
dis = subprocess.run(["nvdisasm", "-gi", cub], capture_output=True, text=True).stdout.splitlines()
# locate the kernel's text section
start = None
for i, l in enumerate(dis):
    if l.startswith("//-----") and ".text." in l and kname in l:
        start = i; break
cur = None; off2line = {}; pending = False
for l in dis[start + 1:]:
    if l.startswith("//-----") and ".text." in l: break
    if l.strip().startswith("//## File"):
        locs = re.findall(r'"([^"]+)", line (\d+)', l)
        # depth: 0 = outermost (kernel body), -1 = innermost
        d = int(os.environ.get("DEPTH", "0"))
        f, n = locs[::-1][min(d, len(locs) - 1)] if d >= 0 else locs[0]
        if " inlined at " in l or cur is None or not pending:
            cur = f'{os.path.basename(f)}:{n}'
        pending = " inlined at " in l
        continue
    m = re.match(r'\s*/\*([0-9a-f]+)\*/\s+\S', l)
    if m:
        off2line[int(m.group(1), 16)] = cur; pending = False
agg = collections.Counter(); stl = collections.Counter(); tot = 0; stot = 0
for r in recs:
    off = int(r[ix["Address"]], 16) - base
    ln = off2line.get(off, "?")
    n = int(r[ix["Instructions Executed"]] or 0); s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    agg[ln] += n; stl[ln] += s; tot += n; stot += s
print(f"total {tot/div:.1f} instr/unit, {stot} stall samples")
for ln, s in stl.most_common(int(os.environ.get("TOP", "50"))):
    print(f"{ln:28s} instr {agg[ln]/div:8.1f}  stall {100*s/stot:5.1f}%")
