"""Whole-image directional filtering on the B200 -- the drop-in for the
reference's ``apply_filter`` (reference ``pkg/src/dirfilt/filters.py:379-433``).

``apply_filter(img, spec, policy=REPLICATE, workers=1)`` keeps the
reference's signature, argument meaning and errors and returns a new
``RasterImage`` whose every pixel is the input pixel the reference selects.
Work happens in ``libdfg.so`` (hand-written sm_100a kernels) through the C
ABI; PyTorch only provides device buffers and the current stream.  There is
no CPU fallback: without a CUDA device or without the built library every
call raises ``RuntimeError``.

Device-resident entry points for pipelines (inputs already in HBM):
``filter_device`` (one (H, W, 3) uint8 tensor), ``filter_batch_device``
((B, H, W, 3)), ``filter_rows_device`` (a row strip of a taller image, used by
the multi-GPU strip sharding in ``parallel.py``), ``filter_host`` (the C
ABI's host-buffer path: H2D + filter + D2H in one call) and
``filter_host_frames`` (a stream of host frames with up to four in flight).
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _lib
from .image import REPLICATE, RasterImage

_ws_lock = threading.Lock()
_ws_cache: dict = {}


_torch_mod = None


def _torch():
    global _torch_mod
    if _torch_mod is None:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_1009_0958_b200 needs a CUDA device (sm_100a); no CPU fallback exists")
        _torch_mod = torch
    return _torch_mod


_prm_cache: dict = {}


def _params(spec, policy):
    """Packed C parameters, cached per (spec, border) -- specs are frozen
    dataclasses here and in the reference, so hashable."""
    mode = getattr(policy, "mode", policy)
    try:
        key = (spec, mode)
        prm = _prm_cache.get(key)
    except TypeError:  # unhashable duck-typed spec
        _validate_spec(spec)
        return _lib.params_from_spec(spec, policy)
    if prm is None:
        _validate_spec(spec)
        prm = _lib.params_from_spec(spec, policy)
        if len(_prm_cache) < 1024:
            _prm_cache[key] = prm
    return prm


class _on_device:
    """torch.cuda.device(d) only when d is not already current (cheap path)."""

    def __init__(self, torch, dev):
        self.ctx = None if dev.index == torch.cuda.current_device() else torch.cuda.device(dev)

    def __enter__(self):
        if self.ctx is not None:
            self.ctx.__enter__()

    def __exit__(self, *a):
        if self.ctx is not None:
            self.ctx.__exit__(*a)


def _validate_spec(spec) -> None:
    """Re-run the reference's construction-time checks on duck-typed specs."""
    fam = spec.family
    if fam not in _lib.FAMILY_CODE:
        raise ValueError(f"unknown filter family {fam!r}")
    if fam == "identity":
        return
    if not float(spec.p) >= 1.0:
        raise ValueError(f"Minkowski order must be >= 1, got {spec.p}")
    w = int(spec.window)
    if w < 3 or w % 2 == 0:
        raise ValueError(f"window side must be odd and >= 3, got {w}")
    if fam in ("cwvmf", "cwddf"):
        from .spec import center_weight

        center_weight(w * w, int(spec.k))
    if fam == "acwddf":
        if spec.acwddf is None:
            raise ValueError("acwddf parameters are required exactly when family is acwddf")
        n = w * w
        if spec.acwddf.lam + 2 > (n + 1) // 2:
            raise ValueError(f"lambda {spec.acwddf.lam} too large for a window of {n} vectors")


def workspace(nbytes: int, device=None, stream=None):
    """A cached, zeroed device workspace (the diagnostic counters) of at least
    ``nbytes`` for ``device``.  Calls only add to its counters, so every
    stream of a device shares one; it is allocated and zeroed synchronously,
    so it is ready before any stream's first launch."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index)
    with _ws_lock:
        buf = _ws_cache.get(dev.index)
        if buf is None or buf.numel() < nbytes:
            buf = torch.zeros(max(nbytes, 4096), dtype=torch.uint8, device=dev)
            torch.cuda.synchronize(dev)  # zero-fill done before launches on any stream
            _ws_cache[dev.index] = buf  # (a replaced buffer only ever held counters)
        return buf


def _stream_ptr(torch, stream, device):
    if stream is not None:
        return ctypes.c_void_p(stream.cuda_stream)
    idx = torch.cuda.current_device() if device is None else torch.device(device).index
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(idx))  # no Stream object per call


def _check_out(torch, out, shape, x):
    """Caller-supplied output buffers: uint8 rows of packed pixels on x's device."""
    if (not isinstance(out, torch.Tensor) or out.dtype != torch.uint8 or out.device != x.device or
            tuple(out.shape) != tuple(shape) or out.stride(-1) != 1 or out.stride(-2) != 3):
        raise ValueError(f"out must be a uint8 tensor of shape {tuple(shape)} on {x.device} with packed pixels "
                         "(stride 3 between pixels, 1 between channels)")
    if len(shape) == 4 and out.stride(1) * shape[1] > out.stride(0):
        raise ValueError("out frames overlap (frame stride smaller than its rows)")


def filter_device(x, spec, policy=REPLICATE, out=None, stream=None, ws=None):
    """Filter a CUDA uint8 tensor (H, W, 3) (row stride may be padded)."""
    torch = _torch()
    _validate_spec(spec)
    if x.dtype != torch.uint8 or x.dim() != 3 or x.shape[2] != 3 or not x.is_cuda:
        raise ValueError("expected a CUDA uint8 tensor of shape (H, W, 3)")
    if x.stride(2) != 1 or x.stride(1) != 3:
        x = x.contiguous()
    H, W = int(x.shape[0]), int(x.shape[1])
    if out is None:
        out = torch.empty((H, W, 3), dtype=torch.uint8, device=x.device)
    else:
        _check_out(torch, out, (H, W, 3), x)
    prm = _params(spec, policy)
    need = _lib.lib().dfg_workspace_bytes(H * W)
    if ws is None:
        ws = workspace(need, x.device, stream)
    with _on_device(torch, x.device):
        rc = _lib.lib().dfg_filter(ctypes.c_void_p(x.data_ptr()), H, W, x.stride(0),
                                   ctypes.c_void_p(out.data_ptr()), out.stride(0), ctypes.byref(prm),
                                   ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                   _stream_ptr(torch, stream, x.device))
    _lib.check(rc)
    return out


def filter_batch_device(x, spec, policy=REPLICATE, out=None, stream=None, ws=None):
    """Filter B frames at once: CUDA uint8 tensor (B, H, W, 3)."""
    torch = _torch()
    _validate_spec(spec)
    if x.dtype != torch.uint8 or x.dim() != 4 or x.shape[3] != 3 or not x.is_cuda:
        raise ValueError("expected a CUDA uint8 tensor of shape (B, H, W, 3)")
    x = x.contiguous()
    B, H, W = (int(s) for s in x.shape[:3])
    if out is None:
        out = torch.empty_like(x)
    else:
        _check_out(torch, out, (B, H, W, 3), x)
    prm = _params(spec, policy)
    need = _lib.lib().dfg_workspace_bytes(B * H * W)
    if ws is None:
        ws = workspace(need, x.device, stream)
    with _on_device(torch, x.device):
        rc = _lib.lib().dfg_filter_batch(ctypes.c_void_p(x.data_ptr()), B, H, W, x.stride(1), x.stride(0),
                                         ctypes.c_void_p(out.data_ptr()), out.stride(1), out.stride(0),
                                         ctypes.byref(prm), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                         _stream_ptr(torch, stream, x.device))
    _lib.check(rc)
    return out


def filter_rows_device(x, global_H, in_row0, out_row0, out_rows, spec, policy=REPLICATE,
                       out=None, stream=None, ws=None):
    """Filter output rows [out_row0, out_row0 + out_rows) of an image with
    ``global_H`` rows, from a CUDA strip ``x`` holding global rows
    [in_row0, in_row0 + x.shape[0]) (reference ``run_rows(r0, r1)``,
    ``_engine.py:560-583``)."""
    torch = _torch()
    _validate_spec(spec)
    if x.dtype != torch.uint8 or x.dim() != 3 or x.shape[2] != 3 or not x.is_cuda:
        raise ValueError("expected a CUDA uint8 tensor of shape (rows, W, 3)")
    if x.stride(2) != 1 or x.stride(1) != 3:
        x = x.contiguous()
    in_rows, W = int(x.shape[0]), int(x.shape[1])
    if out is None:
        out = torch.empty((out_rows, W, 3), dtype=torch.uint8, device=x.device)
    else:
        _check_out(torch, out, (out_rows, W, 3), x)
    prm = _params(spec, policy)
    need = _lib.lib().dfg_workspace_bytes(out_rows * W)
    if ws is None:
        ws = workspace(need, x.device, stream)
    with _on_device(torch, x.device):
        rc = _lib.lib().dfg_filter_rows(ctypes.c_void_p(x.data_ptr()), int(global_H), W, int(in_row0), in_rows,
                                        x.stride(0), ctypes.c_void_p(out.data_ptr()), int(out_row0),
                                        int(out_rows), out.stride(0), ctypes.byref(prm),
                                        ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                        _stream_ptr(torch, stream, x.device))
    _lib.check(rc)
    return out


def filter_host(pixels_u8: np.ndarray, spec, policy=REPLICATE, out: np.ndarray | None = None,
                stream=None) -> np.ndarray:
    """The C ABI's host-buffer path (``dfg_filter_host``): host uint8 in,
    host uint8 out, H2D + kernels + D2H inside one call."""
    torch = _torch()
    prm = _params(spec, policy)  # validates on first use of a spec
    a = pixels_u8 if (type(pixels_u8) is np.ndarray and pixels_u8.dtype == np.uint8 and
                      pixels_u8.flags.c_contiguous) else np.ascontiguousarray(pixels_u8, dtype=np.uint8)
    if a.ndim != 3 or a.shape[2] != 3:
        raise ValueError(f"pixel array must have shape (M, N, 3), got {a.shape}")
    H, W = a.shape[:2]
    if out is None:
        out = np.empty_like(a)
    elif out.shape != a.shape or out.dtype != np.uint8 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous uint8 array of the input's shape")
    rc = _lib.lib().dfg_filter_host(a.ctypes.data_as(ctypes.c_void_p), H, W,
                                    out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(prm),
                                    _stream_ptr(torch, stream, None))
    _lib.check(rc)
    return out


def filter_host_frames(frames, spec, policy=REPLICATE, out=None, stream=None):
    """A stream of independent host frames through ``dfg_filter_host_frames``:
    ``frames`` is a sequence of C-contiguous uint8 (H, W, 3) arrays of one
    shape (or an (F, H, W, 3) array); returns the list of filtered frames
    (written into ``out``'s arrays when given).  Up to four frames are in
    flight, so frame f's copy to the device overlaps the kernels and copies
    back of the frames before it; pin the buffers for the overlap.  Each output
    equals ``filter_host`` of its frame."""
    prm = _params(spec, policy)
    ins = [f for f in frames]
    if not ins:
        return []
    shape = ins[0].shape
    if len(shape) != 3 or shape[2] != 3:
        raise ValueError(f"pixel arrays must have shape (M, N, 3), got {shape}")
    for a in ins:
        if (type(a) is not np.ndarray or a.dtype != np.uint8 or not a.flags.c_contiguous or a.shape != shape):
            raise ValueError("frames must be C-contiguous uint8 arrays of one (M, N, 3) shape")
    if out is None:
        out = [np.empty_like(a) for a in ins]
    else:
        out = [o for o in out]
        if len(out) != len(ins) or any(type(o) is not np.ndarray or o.dtype != np.uint8 or o.shape != shape or
                                       not o.flags.c_contiguous or not o.flags.writeable for o in out):
            raise ValueError("out must hold one writable C-contiguous uint8 array per frame, of the frames' shape")
    torch = _torch()  # arguments are checked first (ValueError with or without a device)
    n = len(ins)
    pin = (ctypes.c_void_p * n)(*[a.ctypes.data for a in ins])
    pout = (ctypes.c_void_p * n)(*[o.ctypes.data for o in out])
    rc = _lib.lib().dfg_filter_host_frames(pin, pout, n, shape[0], shape[1], ctypes.byref(prm),
                                           _stream_ptr(torch, stream, None))
    _lib.check(rc)
    return out


def fixup_counts(device=None, stream=None, reset: bool = False):
    """(pixels re-decided in float64, of which needed the correctly rounded
    arccos pass) accumulated on ``device``'s cached workspace since the last
    reset (diagnostic; ``reset=True`` zeroes the counters after reading)."""
    torch = _torch()
    ws = workspace(1, device)
    counts = ws[:8].view(torch.int32).cpu().tolist()
    if reset:
        _lib.check(_lib.lib().dfg_reset_counts(ctypes.c_void_p(ws.data_ptr()),
                                               _stream_ptr(torch, stream, ws.device)))
        torch.cuda.synchronize(ws.device)
    return counts[0], counts[1]


def last_fixup_count(device=None, stream=None) -> int:
    """Float64 re-decisions since the previous call (resets the counter)."""
    return fixup_counts(device, stream, reset=True)[0]


def apply_filter(img, spec, policy=REPLICATE, workers: int = 1, *, device=None) -> RasterImage:
    """Filter the whole image; output pixel (r, c) is the filter of the window
    centred there, read from the original image (reference
    ``filters.apply_filter``, filters.py:379-433).

    Same signature, semantics and errors as the reference, plus one input
    restriction of the GPU path: pixel values must be integers in 0..255
    (``ValueError`` otherwise).  The float64 pixels go through the C ABI's
    ``dfg_filter_host_f64`` (validation and conversion on the host cores,
    pinned staging, banded H2D / kernels / D2H, float64 result); the
    result is a new ``RasterImage``.  ``workers`` keeps the reference's
    meaning (a row partition with bit-identical results): on the GPU the
    rows are banded inside the call, so the value only needs to be accepted.
    ``device`` (keyword-only addition) selects the CUDA device.
    """
    pixels = img.pixels if hasattr(img, "pixels") else np.asarray(img)
    if spec.family == "identity":  # filters.py:394-395
        return RasterImage._adopt(np.array(pixels, dtype=np.float64, copy=True))
    _validate_spec(spec)
    prm = _params(spec, policy)
    a = pixels if (type(pixels) is np.ndarray and pixels.dtype == np.float64 and pixels.flags.c_contiguous) \
        else np.ascontiguousarray(pixels, dtype=np.float64)
    if a.ndim != 3 or a.shape[2] != 3:
        raise ValueError(f"pixel array must have shape (M, N, 3), got {a.shape}")
    torch = _torch()
    M, N = a.shape[:2]
    out = np.empty((M, N, 3), dtype=np.float64)
    idx = torch.cuda.current_device() if device is None else torch.device(device).index
    with _on_device(torch, torch.device("cuda", idx)):
        rc = _lib.lib().dfg_filter_host_f64(a.ctypes.data_as(ctypes.c_void_p), M, N,
                                            out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(prm), 0,
                                            _stream_ptr(torch, None, torch.device("cuda", idx)))
    _lib.check(rc)
    return RasterImage._adopt(out)
