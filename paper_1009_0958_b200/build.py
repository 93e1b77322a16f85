"""Build the in-tree CUDA library ``libdfg.so`` for sm_100a.

Each translation unit under ``csrc/`` is compiled with nvcc
(``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3``) in parallel,
then linked into ``paper_1009_0958_b200/libdfg.so`` (static cudart, so the
library is self-contained and travels with the repo snapshot).  The float64
re-decision code is compiled with ``-fmad=false``: no contraction of
multiply-adds, so its arithmetic rounds like the reference's.  (Applied
to every unit: the float64 stage is inlined into the decision kernels; the
FP32 code spells its fused multiply-adds explicitly with fmaf.)
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "libdfg.so"
DEV_MARK = PKG / ".dev_build"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# (DFG_DEFS: extra -D flags for measurement builds, scripts/dev_unit.py; empty in product builds)
COMMON = [*os.environ.get("DFG_DEFS", "").split(), "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
          "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", f"-I{INCLUDE}", "--expt-relaxed-constexpr"]
PER_FILE: dict = {}


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libdfg.so")


def _headers_mtime() -> float:
    hs = list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return max(h.stat().st_mtime for h in hs)


def build(verbose: bool = False, force: bool = False, jobs: int | None = None) -> Path:
    sources = sorted(CSRC.glob("*.cu"))
    hdr = _headers_mtime()
    # scripts/dev_unit.py leaves this marker: the library then holds a partial
    # (measurement) instantiation of some unit and must not pass for a product
    # build -- unless the measurement scripts say so
    if DEV_MARK.exists() and os.environ.get("DFG_ALLOW_DEV_LIB") != "1":
        force = True
    if not force and LIB.exists() and LIB.stat().st_mtime >= max([hdr] + [s.stat().st_mtime for s in sources]):
        return LIB  # up to date (e.g. the prebuilt library shipped to a GPU box without its objects)
    nvcc = _nvcc()
    OBJ.mkdir(exist_ok=True)
    todo = []
    for src in sources:
        obj = OBJ / (src.stem + ".o")
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, hdr):
            todo.append((src, obj))

    def compile_one(item):
        src, obj = item
        cmd = [nvcc, *ARCH, *COMMON, *PER_FILE.get(src.name, []), "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(f"[build] {src.name}\n{r.stderr}")
        return src.name

    if todo:
        with ThreadPoolExecutor(max_workers=jobs or min(len(todo), os.cpu_count() or 4)) as ex:
            for name in ex.map(compile_one, todo):
                if verbose:
                    print(f"[build] compiled {name}", file=sys.stderr)
    objs = [OBJ / (s.stem + ".o") for s in sources]
    if todo or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    if force and DEV_MARK.exists():
        DEV_MARK.unlink()
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
