"""The angle-vs-chromaticity calibration line on the B200 -- drop-in for the
reference's ``LinearFit`` / ``fit_line`` / ``sample_angle_chromaticity_pairs``
/ ``fit_angular_chromaticity`` (reference ``pkg/src/dirfilt/calibration.py:
20-125``).

``fit_angular_chromaticity`` draws the reference's PCG64 sample stream on the
device (``csrc/dfg_calib.cu``) and reduces it there in three passes (means,
central second moments, residuals), regenerating the samples each pass
instead of storing them, so the paper's 10^8-pair "exact-replication mode"
(calibration.py:119-120) runs in milliseconds.  Only the final line formula
(a handful of float64 scalars) is evaluated on the host, in the reference's
expression order.  Results match the reference to ~1e-12 relative (reduction
order and the device arccos differ; the samples' B values are bit-exact).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .filters import _stream_ptr, _torch

_M64 = (1 << 64) - 1


@dataclass(frozen=True)
class LinearFit:
    """A fitted line A ~ slope*B + intercept with residual statistics
    (reference calibration.py:20-44)."""

    slope: float
    intercept: float
    fit_error: float
    sample_count: int
    mean_abs_residual: float
    rms_orthogonal: float
    method: str

    def __str__(self) -> str:
        return (
            f"A ~ {self.slope:.6f} * B + {self.intercept:.6f}  "
            f"[{self.method}, n={self.sample_count}, rms={self.fit_error:.6f}, "
            f"mean|r|={self.mean_abs_residual:.6f}, rms_orth={self.rms_orthogonal:.6f}]"
        )


def _slope(method: str, sxx: float, syy: float, sxy: float) -> float:
    if method == "ols":
        return sxy / sxx
    return (syy - sxx + float(np.hypot(syy - sxx, 2.0 * sxy))) / (2.0 * sxy)


def _params(pairs: int, seed: int, p: float) -> _lib.DfgCalibParams:
    st = np.random.PCG64(seed).state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    return _lib.DfgCalibParams(pairs=int(pairs), p=float(p), state_hi=s >> 64, state_lo=s & _M64,
                               inc_hi=inc >> 64, inc_lo=inc & _M64)


def _validate_p(p: float) -> float:
    p = float(p)
    if not p >= 1.0:  # distance.py _validate_p
        raise ValueError(f"Minkowski order must be >= 1, got {p}")
    return p


def fit_angular_chromaticity(pairs: int = 10**6, seed: int = 0, p: float = 2.0, method: str = "tls",
                             *, device=None) -> LinearFit:
    """Reproduce the angle-vs-chromaticity calibration line (reference
    calibration.py:116-125), deterministic given ``seed``."""
    if pairs < 1000:
        raise ValueError(f"need at least 1000 pairs, got {pairs}")
    if method not in ("tls", "ols"):
        raise ValueError(f"unknown regression method {method!r}")
    p = _validate_p(p)
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index)
    L = _lib.lib()
    nbytes = L.dfg_calib_scratch_bytes()
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    cp = _params(pairs, seed, p)
    out = (ctypes.c_double * 3)()
    stream = _stream_ptr(torch, None, dev)

    def reduce(mode, x0=0.0, x1=0.0):
        _lib.check(L.dfg_calib_reduce(ctypes.byref(cp), mode, x0, x1, out, ctypes.c_void_p(scratch.data_ptr()),
                                      nbytes, stream))
        return out[0], out[1], out[2]

    with torch.cuda.device(dev):
        sb, sa, _ = reduce(0)
        mb, ma = sb / pairs, sa / pairs
        cxx, cyy, cxy = reduce(1, mb, ma)
        sxx, syy, sxy = cxx / pairs, cyy / pairs, cxy / pairs
        if sxx < 1e-30:
            raise ValueError("degenerate samples: no variance in B (all pairs parallel?)")
        slope = _slope(method, sxx, syy, sxy)
        intercept = ma - slope * mb
        r2, rabs, _ = reduce(2, slope, intercept)
    rms = math.sqrt(r2 / pairs)
    return LinearFit(slope=float(slope), intercept=float(intercept), fit_error=rms, sample_count=int(pairs),
                     mean_abs_residual=rabs / pairs, rms_orthogonal=rms / math.sqrt(1.0 + slope * slope),
                     method=method)


def sample_angle_chromaticity_pairs(pairs: int, seed: int, p: float = 2.0, *, device=None):
    """(B, A) of ``pairs`` random vector pairs as CUDA float64 tensors
    (reference calibration.py:83-113 returns numpy arrays; ``.cpu().numpy()``
    gives those)."""
    p = _validate_p(p)
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index)
    b = torch.empty(int(pairs), dtype=torch.float64, device=dev)
    a = torch.empty_like(b)
    cp = _params(pairs, seed, p)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().dfg_calib_samples(ctypes.byref(cp), ctypes.c_void_p(b.data_ptr()),
                                                ctypes.c_void_p(a.data_ptr()), _stream_ptr(torch, None, dev)))
    return b, a


def fit_line(b, a, method: str = "tls") -> LinearFit:
    """Fit a line to (b, a) samples (reference calibration.py:47-80): the
    means, central second moments and residual sums are three passes of the
    device reduction kernel (``dfg_moments_reduce``, float64, fixed order);
    only the line formula's few scalars are evaluated on the host."""
    if method not in ("tls", "ols"):
        raise ValueError(f"unknown regression method {method!r}")
    torch = _torch()
    tb = torch.as_tensor(np.asarray(b, dtype=np.float64) if not torch.is_tensor(b) else b, dtype=torch.float64)
    ta = torch.as_tensor(np.asarray(a, dtype=np.float64) if not torch.is_tensor(a) else a, dtype=torch.float64)
    if tb.shape != ta.shape or tb.dim() != 1 or tb.numel() < 2:
        raise ValueError("need two equal-length 1-D sample arrays")
    dev = tb.device if tb.is_cuda else torch.device("cuda", torch.cuda.current_device())
    tb, ta = tb.to(dev).contiguous(), ta.to(dev).contiguous()
    n = int(tb.numel())
    L = _lib.lib()
    nbytes = L.dfg_calib_scratch_bytes()
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    out = (ctypes.c_double * 3)()
    stream = _stream_ptr(torch, None, dev)

    def reduce(mode, x0=0.0, x1=0.0):
        _lib.check(L.dfg_moments_reduce(ctypes.c_void_p(tb.data_ptr()), ctypes.c_void_p(ta.data_ptr()), n, mode,
                                        x0, x1, out, ctypes.c_void_p(scratch.data_ptr()), nbytes, stream))
        return out[0], out[1], out[2]

    with torch.cuda.device(dev):
        sb, sa, _ = reduce(0)
        mb, ma = sb / n, sa / n
        cxx, cyy, cxy = reduce(1, mb, ma)
        sxx, syy, sxy = cxx / n, cyy / n, cxy / n
        if sxx < 1e-30:
            raise ValueError("degenerate samples: no variance in B (all pairs parallel?)")
        slope = _slope(method, sxx, syy, sxy)
        intercept = ma - slope * mb
        r2, rabs, _ = reduce(2, slope, intercept)
    rms = math.sqrt(r2 / n)
    return LinearFit(slope=float(slope), intercept=float(intercept), fit_error=rms, sample_count=n,
                     mean_abs_residual=rabs / n, rms_orthogonal=rms / math.sqrt(1.0 + slope * slope),
                     method=method)
