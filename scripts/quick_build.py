"""Recompile only the given csrc units and relink libdfg.so (iteration aid:
the other objects stay as they are -- run `python -m paper_1009_0958_b200.build -f`
before committing).  usage: python scripts/quick_build.py fast_s7_ddf fast_s5_acwddf ..."""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, ".")
from paper_1009_0958_b200 import build as b  # noqa: E402

nv = b._nvcc()


def one(u):
    src = b.CSRC / (u + ".cu")
    r = subprocess.run([nv, *b.ARCH, *b.COMMON, "-c", str(src), "-o", str(b.OBJ / (u + ".o"))],
                       capture_output=True, text=True)
    return u, r.returncode, r.stderr[-800:] if r.returncode else ""


with ThreadPoolExecutor(8) as ex:
    for u, rc, err in ex.map(one, sys.argv[1:]):
        print(u, rc, err)
objs = [b.OBJ / (s.stem + ".o") for s in sorted(b.CSRC.glob("*.cu"))]
r = subprocess.run([nv, *b.ARCH, "-shared", "-o", str(b.LIB), *map(str, objs), "-cudart", "static"],
                   capture_output=True, text=True)
print("link", r.returncode, r.stderr[-300:])
