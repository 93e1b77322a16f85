"""ctypes binding of the in-tree CUDA library ``libdfg.so`` (C ABI in
``include/dirfilt_gpu.h``).  There is no fallback: if the library is missing
or cannot be loaded, every filter call raises."""

from __future__ import annotations

import ctypes
from pathlib import Path

from .spec import ACOS_COEFFICIENTS, ASIN_COEFFICIENTS

LIB_PATH = Path(__file__).resolve().parent / "libdfg.so"

DFG_OK, DFG_E_ARG, DFG_E_CUDA, DFG_E_UNSUP, DFG_E_WS = 0, -1, -2, -3, -4
FAMILY_CODE = {"identity": 0, "vmf": 1, "bvdf": 2, "ddf": 3, "acwddf": 4, "cwvmf": 5, "cwddf": 6}
STRATEGY_CODE = {"exact": 0, "minimax": 1, "chromaticity": 2}
BORDER_CODE = {"replicate": 0, "reflect": 1}

# every symbol include/dirfilt_gpu.h declares
EXPORTS = (
    "dfg_abi_version", "dfg_last_error", "dfg_workspace_bytes", "dfg_filter",
    "dfg_filter_rows", "dfg_filter_batch", "dfg_filter_host", "dfg_filter_host_f64", "dfg_filter_host_frames",
    "dfg_set_option", "dfg_get_option", "dfg_fixup_count",
    "dfg_reset_counts", "dfg_debug_values", "dfg_cr_acos_host", "dfg_corrupt_image",
    "dfg_image_metrics", "dfg_calib_scratch_bytes", "dfg_calib_reduce", "dfg_calib_samples", "dfg_moments_reduce",
    "dfg_hostconv_selftest",
)


class DfgParams(ctypes.Structure):
    _fields_ = [
        ("family", ctypes.c_int32),
        ("strategy", ctypes.c_int32),
        ("window", ctypes.c_int32),
        ("border", ctypes.c_int32),
        ("p", ctypes.c_double),
        ("asin_c", ctypes.c_double * 5),
        ("acos_c", ctypes.c_double * 5),
        ("lam", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("threshold", ctypes.c_double),
        ("slope", ctypes.c_double),
        ("intercept", ctypes.c_double),
    ]


class DfgNoiseParams(ctypes.Structure):
    _fields_ = [
        ("phi", ctypes.c_double),
        ("phi1", ctypes.c_double),
        ("phi2", ctypes.c_double),
        ("phi3", ctypes.c_double),
        ("impulse", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("state_hi", ctypes.c_uint64),
        ("state_lo", ctypes.c_uint64),
        ("inc_hi", ctypes.c_uint64),
        ("inc_lo", ctypes.c_uint64),
    ]


class DfgCalibParams(ctypes.Structure):
    _fields_ = [
        ("pairs", ctypes.c_int64),
        ("p", ctypes.c_double),
        ("state_hi", ctypes.c_uint64),
        ("state_lo", ctypes.c_uint64),
        ("inc_hi", ctypes.c_uint64),
        ("inc_lo", ctypes.c_uint64),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libdfg.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_1009_0958_b200.build` "
                           "(the GPU path has no CPU fallback)")
    L = ctypes.CDLL(str(LIB_PATH))
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    P = ctypes.POINTER(DfgParams)
    L.dfg_abi_version.restype = ctypes.c_int
    L.dfg_last_error.restype = ctypes.c_char_p
    L.dfg_workspace_bytes.argtypes = [i64]
    L.dfg_workspace_bytes.restype = sz
    L.dfg_filter.argtypes = [vp, i32, i32, i64, vp, i64, P, vp, sz, vp]
    L.dfg_filter_rows.argtypes = [vp, i32, i32, i32, i32, i64, vp, i32, i32, i64, P, vp, sz, vp]
    L.dfg_filter_batch.argtypes = [vp, i32, i32, i32, i64, i64, vp, i64, i64, P, vp, sz, vp]
    L.dfg_filter_host.argtypes = [vp, i32, i32, vp, P, vp]
    L.dfg_filter_host_f64.argtypes = [vp, i32, i32, vp, P, i32, vp]
    L.dfg_filter_host_frames.argtypes = [vp, vp, i32, i32, i32, P, vp]
    L.dfg_set_option.argtypes = [i32, ctypes.c_double]
    L.dfg_get_option.argtypes = [i32]
    L.dfg_get_option.restype = ctypes.c_double
    L.dfg_fixup_count.argtypes = [vp, vp, ctypes.POINTER(i64)]
    L.dfg_reset_counts.argtypes = [vp, vp]
    L.dfg_debug_values.argtypes = [vp, i32, i32, i64, vp, P, vp]
    L.dfg_cr_acos_host.argtypes = [ctypes.c_double, i32]
    L.dfg_cr_acos_host.restype = ctypes.c_double
    L.dfg_corrupt_image.argtypes = [vp, i32, i32, i64, vp, i64, ctypes.POINTER(DfgNoiseParams), vp]
    L.dfg_image_metrics.argtypes = [vp, vp, i32, i32, i64, i64, ctypes.POINTER(ctypes.c_double), vp, vp]
    L.dfg_calib_scratch_bytes.restype = sz
    L.dfg_calib_reduce.argtypes = [ctypes.POINTER(DfgCalibParams), i32, ctypes.c_double, ctypes.c_double,
                                   ctypes.POINTER(ctypes.c_double), vp, sz, vp]
    L.dfg_calib_samples.argtypes = [ctypes.POINTER(DfgCalibParams), vp, vp, vp]
    L.dfg_hostconv_selftest.argtypes = [vp, i64, vp, vp, vp]
    L.dfg_hostconv_selftest.restype = ctypes.c_int
    L.dfg_moments_reduce.argtypes = [vp, vp, i64, i32, ctypes.c_double, ctypes.c_double,
                                     ctypes.POINTER(ctypes.c_double), vp, sz, vp]
    for name in ("dfg_filter", "dfg_filter_rows", "dfg_filter_batch", "dfg_filter_host", "dfg_filter_host_f64",
                 "dfg_filter_host_frames", "dfg_set_option",
                 "dfg_fixup_count", "dfg_reset_counts", "dfg_debug_values", "dfg_corrupt_image",
                 "dfg_image_metrics", "dfg_calib_reduce", "dfg_calib_samples", "dfg_moments_reduce"):
        getattr(L, name).restype = ctypes.c_int
    if L.dfg_abi_version() != 1:
        raise RuntimeError("libdfg.so ABI version mismatch; rebuild")
    _lib = L
    return L


# schedule / diagnostic options (DFG_OPT_* in include/dirfilt_gpu.h)
OPTIONS = {"s3_schedule": 1, "no_fixup": 2, "host_bands": 3, "host_graph": 4, "host_w3_rpc": 5,
           "frame_slots": 6, "w3_wps": 7, "w3_rpc": 8, "w3_small_wps": 9, "cr_margin": 10, "tma": 11, "persist": 12}


def set_option(name: str, value) -> float:
    """Set a process-wide library option; returns the previous value."""
    key = OPTIONS[name]
    old = lib().dfg_get_option(key)
    check(lib().dfg_set_option(key, float(value)))
    return old


class option:
    """Context manager: ``with option("s3_schedule", 2): ...``"""

    def __init__(self, name: str, value):
        self.name, self.value = name, value

    def __enter__(self):
        self.old = set_option(self.name, self.value)
        return self

    def __exit__(self, *exc):
        set_option(self.name, self.old)
        return False


def check(rc: int) -> None:
    if rc == DFG_OK:
        return
    msg = lib().dfg_last_error().decode(errors="replace")
    if rc == DFG_E_ARG:
        raise ValueError(msg)
    if rc == DFG_E_UNSUP:
        raise NotImplementedError(msg)
    raise RuntimeError(f"libdfg error {rc}: {msg}")


def _pad5(t):
    t = tuple(float(x) for x in t)
    return t + (0.0,) * (5 - len(t))


def params_from_spec(spec, policy) -> DfgParams:
    """Pack a FilterSpec (this package's or the reference's) + BorderPolicy."""
    prm = DfgParams()
    fam = spec.family
    if fam not in FAMILY_CODE:
        raise ValueError(f"unknown engine family {fam!r}")
    prm.family = FAMILY_CODE[fam]
    kind = spec.strategy.kind
    prm.strategy = STRATEGY_CODE[kind] if fam not in ("vmf", "cwvmf") else 0
    prm.window = int(spec.window)
    mode = getattr(policy, "mode", policy)
    prm.border = BORDER_CODE[mode]
    if fam == "acwddf":
        prm.p = float(spec.acwddf.p)
        prm.lam = int(spec.acwddf.lam)
        prm.threshold = float(spec.acwddf.threshold)
    else:
        prm.p = float(spec.p)
        prm.lam = int(spec.k) if fam in ("cwvmf", "cwddf") else 2  # centre-weighted: smoothing level k
        prm.threshold = 10.8
    if kind == "minimax" and fam not in ("vmf", "cwvmf"):
        table = spec.strategy.table  # reference and this package both expose it
        if table is not None:
            cs, ca = table.asin_poly.coefficients, table.acos_poly.coefficients
        else:
            q = int(spec.strategy.q)
            cs, ca = ASIN_COEFFICIENTS[q][1], ACOS_COEFFICIENTS[q][1]
        prm.asin_c[:] = _pad5(cs)
        prm.acos_c[:] = _pad5(ca)
    prm.slope = float(spec.strategy.slope)
    prm.intercept = float(spec.strategy.intercept)
    return prm
