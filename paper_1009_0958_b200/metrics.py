"""Effectiveness criteria (MAE, PSNR, NCD) on the B200 -- drop-in for the
reference's ``metrics.compare`` / ``mae`` / ``psnr`` / ``ncd`` and
``MetricsReport`` (reference ``pkg/src/dirfilt/metrics.py:33-118``).

One device reduction (``dfg_image_metrics``, ``csrc/dfg_metrics.cu``) yields
all three numbers with float64 sums; they match the reference's numpy values
to ~1e-12 relative (summation order differs), which the tests assert.
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .filters import _on_device, _stream_ptr, _torch
from .image import to_uint8

_scratch_lock = threading.Lock()
_scratch: dict = {}


@dataclass
class MetricsReport:
    """One row of filtering effectiveness numbers (reference metrics.py:33-52)."""

    mae: float
    psnr: float
    ncd_x1000: float
    time_seconds: float = 0.0

    def csv_row(self) -> str:
        return f"{self.mae:.6f},{_fmt(self.psnr)},{self.ncd_x1000:.6f},{self.time_seconds:.6f}"

    def table_row(self) -> str:
        return f"{self.mae:9.3f} {_fmt(self.psnr):>9s} {self.ncd_x1000:9.3f} {self.time_seconds:9.3f}"


def _fmt(x: float) -> str:
    return "inf" if math.isinf(x) else f"{x:.6f}"


def _scratch_for(torch, dev):
    with _scratch_lock:
        buf = _scratch.get(dev.index)
        if buf is None:
            buf = torch.zeros(4, dtype=torch.float64, device=dev)
            _scratch[dev.index] = buf
        return buf


def metrics_device(ref, test, stream=None):
    """(MAE, PSNR, NCD x 1000) of CUDA uint8 tensor ``test`` against ``ref``,
    both (H, W, 3) on the same device.  Synchronises the stream."""
    torch = _torch()
    for t in (ref, test):
        if t.dtype != torch.uint8 or t.dim() != 3 or t.shape[2] != 3 or not t.is_cuda:
            raise ValueError("expected CUDA uint8 tensors of shape (H, W, 3)")
    if tuple(ref.shape[:2]) != tuple(test.shape[:2]):
        raise ValueError(f"dimension mismatch: {ref.shape[0]}x{ref.shape[1]} vs {test.shape[0]}x{test.shape[1]}")
    if ref.stride(2) != 1 or ref.stride(1) != 3:
        ref = ref.contiguous()
    if test.stride(2) != 1 or test.stride(1) != 3:
        test = test.contiguous()
    H, W = int(ref.shape[0]), int(ref.shape[1])
    out = (ctypes.c_double * 3)()
    scratch = _scratch_for(torch, ref.device)
    with _on_device(torch, ref.device):
        rc = _lib.lib().dfg_image_metrics(ctypes.c_void_p(ref.data_ptr()), ctypes.c_void_p(test.data_ptr()), H, W,
                                          ref.stride(0), test.stride(0), out, ctypes.c_void_p(scratch.data_ptr()),
                                          _stream_ptr(torch, stream, ref.device))
    _lib.check(rc)
    return out[0], out[1], out[2]


def _pair(orig, test, device):
    a = orig.pixels if hasattr(orig, "pixels") else np.asarray(orig)
    b = test.pixels if hasattr(test, "pixels") else np.asarray(test)
    if a.shape[:2] != b.shape[:2]:
        raise ValueError(f"dimension mismatch: {a.shape[0]}x{a.shape[1]} vs {b.shape[0]}x{b.shape[1]}")
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index)
    return torch.from_numpy(to_uint8(a)).to(dev), torch.from_numpy(to_uint8(b)).to(dev)


def compare(orig, test, time_seconds: float = 0.0, *, device=None) -> MetricsReport:
    """All three criteria in one report (reference metrics.py:112-118)."""
    m, p, n = metrics_device(*_pair(orig, test, device))
    return MetricsReport(mae=m, psnr=p, ncd_x1000=n, time_seconds=time_seconds)


def mae(orig, test, *, device=None) -> float:
    return metrics_device(*_pair(orig, test, device))[0]


def psnr(orig, test, *, device=None) -> float:
    return metrics_device(*_pair(orig, test, device))[1]


def ncd(orig, test, *, device=None) -> float:
    return metrics_device(*_pair(orig, test, device))[2]
