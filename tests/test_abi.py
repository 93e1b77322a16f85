"""CPU: the C-ABI library loads, exports every symbol include/dirfilt_gpu.h
declares, lays out dfg_params as the header does, validates like the
reference (no GPU needed for these paths), and its double-double arccos is
correctly rounded."""

import ctypes
import math
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_1009_0958_b200 import _lib, parse_filter_spec

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "dirfilt_gpu.h"


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = re.findall(r"DFG_API\s+[\w\s\*]+?\b(dfg_\w+)\s*\(", HEADER.read_text())
    assert declared and set(declared) == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.dfg_abi_version() == 1


def test_params_layout_matches_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "dirfilt_gpu.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(dfg_params), '
                   'offsetof(dfg_params,p), offsetof(dfg_params,asin_c), offsetof(dfg_params,lam), '
                   'offsetof(dfg_params,threshold), offsetof(dfg_params,intercept));return 0;}\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    P = _lib.DfgParams
    want = [ctypes.sizeof(P), P.p.offset, P.asin_c.offset, P.lam.offset, P.threshold.offset, P.intercept.offset]
    assert got == want


def test_noise_params_layout_matches_header(tmp_path):
    src = tmp_path / "nlayout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "dirfilt_gpu.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu\\n", sizeof(dfg_noise_params), '
                   'offsetof(dfg_noise_params,impulse), offsetof(dfg_noise_params,state_hi), '
                   'offsetof(dfg_noise_params,inc_lo));return 0;}\n')
    exe = tmp_path / "nlayout"
    subprocess.run(["gcc", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    P = _lib.DfgNoiseParams
    assert got == [ctypes.sizeof(P), P.impulse.offset, P.state_hi.offset, P.inc_lo.offset]


def test_noise_and_metrics_validate_before_any_cuda_call():
    """NoiseParams validation (reference noise.py:42-55) and dimension checks
    are reported as DFG_E_ARG without touching the device."""
    L = _lib.lib()
    good = dict(phi=0.1, phi1=0.25, phi2=0.25, phi3=0.25, impulse=0)
    for bad in (dict(phi=1.5), dict(phi=-0.1), dict(phi1=-0.01), dict(phi1=0.5, phi2=0.5, phi3=0.1),
                dict(impulse=2)):
        np_ = _lib.DfgNoiseParams(**{**good, **bad})
        assert L.dfg_corrupt_image(ctypes.c_void_p(1), 4, 4, 12, ctypes.c_void_p(1), 12, ctypes.byref(np_), None) == -1
    np_ = _lib.DfgNoiseParams(**good)
    assert L.dfg_corrupt_image(ctypes.c_void_p(1), 0, 4, 12, ctypes.c_void_p(1), 12, ctypes.byref(np_), None) == -1
    out = (ctypes.c_double * 3)()
    assert L.dfg_image_metrics(ctypes.c_void_p(1), ctypes.c_void_p(1), 4, 4, 11, 12, out, ctypes.c_void_p(1),
                               None) == -1


@pytest.mark.parametrize("text,code", [("vmf:window=33", _lib.DFG_E_UNSUP), ("bvdf:exact:window=101", _lib.DFG_E_UNSUP)])
def test_unsupported_window_reported_before_any_cuda_call(text, code):
    L = _lib.lib()
    prm = _lib.params_from_spec(parse_filter_spec(text), "replicate")
    rc = L.dfg_filter(ctypes.c_void_p(1), 4, 4, 12, ctypes.c_void_p(1), 12, ctypes.byref(prm), None, 0, None)
    assert rc == code
    assert b"window" in L.dfg_last_error()


def test_invalid_params_rejected():
    L = _lib.lib()
    prm = _lib.params_from_spec(parse_filter_spec("acwddf"), "replicate")
    prm.lam = 4  # lambda + 2 > (n+1)/2 for n = 9
    assert L.dfg_filter(ctypes.c_void_p(1), 4, 4, 12, ctypes.c_void_p(1), 12, ctypes.byref(prm), None, 0, None) == -1
    prm = _lib.params_from_spec(parse_filter_spec("ddf"), "replicate")
    prm.window = 4
    assert L.dfg_filter(ctypes.c_void_p(1), 4, 4, 12, ctypes.c_void_p(1), 12, ctypes.byref(prm), None, 0, None) == -1
    prm = _lib.params_from_spec(parse_filter_spec("ddf"), "replicate")
    assert L.dfg_filter(ctypes.c_void_p(1), 0, 4, 12, ctypes.c_void_p(1), 12, ctypes.byref(prm), None, 0, None) == -1
    # strips must carry their halo rows
    assert L.dfg_filter_rows(ctypes.c_void_p(1), 100, 4, 10, 20, 12, ctypes.c_void_p(1), 10, 20, 12,
                             ctypes.byref(prm), None, 0, None) == -1


def test_cr_acos_is_correctly_rounded():
    """The float64 re-decision's arccos (dfg_f64.cuh) returns the correctly
    rounded value from starting points several ulps off (the GPU's acos is
    within 2 ulps); checked against a 160-bit mpmath evaluation."""
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.prec = 160
    L = _lib.lib()
    rng = np.random.default_rng(7)
    a = rng.integers(0, 256, (3000, 3)).astype(float)
    b = rng.integers(0, 256, (3000, 3)).astype(float)
    a[(a == 0).all(1)] = 1
    b[(b == 0).all(1)] = 1
    zs = np.clip((a * b).sum(1) / np.sqrt((a * a).sum(1) * (b * b).sum(1)), 0, 1)
    zs = np.concatenate([zs, rng.random(2000), 1 - rng.random(2000) ** 6, [0.0, 0.5, 1.0, 1 - 2**-53]])
    glibc_off = 0
    for z in zs:
        z = float(z)
        cr = float(mpmath.acos(mpmath.mpf(z)))
        for pert in (-3, 0, 2):
            assert L.dfg_cr_acos_host(z, pert) == cr, (z, pert)
        glibc_off += math.acos(z) != cr
    # glibc's acos (the reference's) is correctly rounded on all but ~0.1-0.2 %
    assert glibc_off < 0.005 * len(zs)


def test_frame_stream_validates_before_any_cuda_call():
    """dfg_filter_host_frames rejects bad arguments (DFG_E_ARG) before it
    allocates or touches the device; an empty stream is a no-op."""
    L = _lib.lib()
    prm = _lib.params_from_spec(parse_filter_spec("ddf:exact"), "replicate")
    buf = (ctypes.c_uint8 * 48)()
    ptrs = (ctypes.c_void_p * 2)(ctypes.addressof(buf), None)
    assert L.dfg_filter_host_frames(ptrs, ptrs, 0, 4, 4, ctypes.byref(prm), None) == 0
    assert L.dfg_filter_host_frames(ptrs, ptrs, -1, 4, 4, ctypes.byref(prm), None) == -1
    assert L.dfg_filter_host_frames(ptrs, ptrs, 1, 0, 4, ctypes.byref(prm), None) == -1
    assert L.dfg_filter_host_frames(None, ptrs, 1, 4, 4, ctypes.byref(prm), None) == -1
    assert L.dfg_filter_host_frames(ptrs, ptrs, 2, 4, 4, ctypes.byref(prm), None) == -1  # null frame pointer
    assert b"frame" in L.dfg_last_error()
    bad = _lib.params_from_spec(parse_filter_spec("ddf:exact"), "replicate")
    bad.window = 4
    assert L.dfg_filter_host_frames(ptrs, ptrs, 1, 4, 4, ctypes.byref(bad), None) == -1


def test_frame_stream_python_validation():
    from paper_1009_0958_b200 import filter_host_frames
    s = parse_filter_spec("bvdf:exact")
    a = np.zeros((4, 5, 3), np.uint8)
    with pytest.raises(ValueError):
        filter_host_frames([a, np.zeros((4, 6, 3), np.uint8)], s)  # shapes differ
    with pytest.raises(ValueError):
        filter_host_frames([a.astype(np.float64)], s)
    with pytest.raises(ValueError):
        filter_host_frames([a], s, out=[a, a])  # one output per frame
    with pytest.raises(ValueError):
        filter_host_frames([np.zeros((4, 5), np.uint8)], s)


def test_host_conversions_dispatched_equal_scalar():
    """float64 <-> uint8 of the drop-in boundary (csrc/dfg_hostconv.cu): the
    AVX2 form equals the scalar one on every length / alignment, flags every
    value that is not an integer in 0..255 (NaN, infinities, huge, negative,
    fractional) and accepts -0.0."""
    L = _lib.lib()
    rng = np.random.default_rng(0)

    def run(src):
        n = src.size
        fast, ref, back = np.zeros(n, np.uint8), np.zeros(n, np.uint8), np.zeros(n)
        rc = L.dfg_hostconv_selftest(src.ctypes.data, n, fast.ctypes.data, ref.ctypes.data, back.ctypes.data)
        return rc, fast, ref, back

    for n in (1, 7, 16, 33, 1000, 100003):
        for off in (0, 1, 3):
            src = rng.integers(0, 256, n + off).astype(np.float64)[off:]
            rc, fast, ref, back = run(src)
            assert rc == 0 and (fast == ref).all() and (back == src).all(), (n, off, rc)
            for bad in (0.5, 256.0, -1.0, np.nan, np.inf, -np.inf, 255.0000001, 1e300, -0.25, 2.0 ** 31, 2.0 ** 32 + 5):
                for pos in (0, n // 2, n - 1):
                    s2 = src.copy()
                    s2[pos] = bad
                    assert run(s2)[0] == 3, (n, off, bad, pos)
            s2 = src.copy()
            s2[0] = -0.0
            assert run(s2)[0] == 0
