"""Iteration aid: rebuild ONE family unit with only the (strategy, p) kernels
named on the command line instantiated (the others return
cudaErrorNotSupported), then relink libdfg.so -- a 7x7 unit compiles in under a
minute instead of five.  Run `python -m paper_1009_0958_b200.build -f` before
committing or measuring anything but the named kernels.
usage: python scripts/dev_unit.py 7 ddf exact [minimax chroma]   (p = 2 only)"""
import subprocess
import sys
import tempfile

sys.path.insert(0, ".")
from paper_1009_0958_b200 import build as b  # noqa: E402

S, fam = sys.argv[1], sys.argv[2]
strategies = sys.argv[3:] or ["exact"]
FAM = {"bvdf": "FAM_BVDF", "ddf": "FAM_DDF", "acwddf": "FAM_ACWDDF", "vmf": "FAM_VMF", "cwvmf": "FAM_CWVMF",
       "cwddf": "FAM_CWDDF"}[fam]
ST = {"exact": "ST_EXACT", "minimax": "ST_MINIMAX", "chroma": "ST_CHROMA"}
body = "".join(
    f"    if (strategy == dfg::{ST[s]}) "
    f"return dfg::launch_fast<{S}, dfg::{FAM}, dfg::{ST[s]}, dfg::PC_2>(st, in, out, kp);\n" for s in strategies)
src = f"""#include "dfg_w3.cuh"
cudaError_t dfg_launch_s{S}_{fam}(int strategy, int pcode, cudaStream_t st, const uint8_t *in, uint8_t *out,
                                  const dfg::KParams &kp)
{{
{body}    return cudaErrorNotSupported;
}}
"""
nv = b._nvcc()
with tempfile.NamedTemporaryFile("w", suffix=".cu", dir=str(b.CSRC), delete=True) as f:
    f.write(src)
    f.flush()
    obj = b.OBJ / f"fast_s{S}_{fam}.o"
    r = subprocess.run([nv, *b.ARCH, *b.COMMON, "-Xptxas=-v", "-c", f.name, "-o", str(obj)], capture_output=True, text=True)
print("compile", r.returncode, r.stderr[-3000:] if r.returncode else "")
for line in r.stderr.splitlines():
    if "registers" in line or "spill" in line:
        print(line.strip()[:160])
objs = [b.OBJ / (s.stem + ".o") for s in sorted(b.CSRC.glob("*.cu"))]
r = subprocess.run([nv, *b.ARCH, "-shared", "-o", str(b.LIB), *map(str, objs), "-cudart", "static"],
                   capture_output=True, text=True)
print("link", r.returncode, r.stderr[-300:])
b.DEV_MARK.write_text("partial instantiation by scripts/dev_unit.py: run `python -m paper_1009_0958_b200.build -f`\n")
