"""Correlated impulsive noise (paper Eq. 8) on the B200 -- drop-in for the
reference's ``NoiseParams`` / ``corrupt_image`` (reference
``pkg/src/dirfilt/noise.py:33-116``).

The corruption runs in ``dfg_corrupt_image`` (``csrc/dfg_noise.cu``): each
thread jumps numpy's PCG64 stream ahead to its first pixel and draws the same
five doubles per pixel, in row-major order, that the reference's
``rng.random((M*N, 5))`` draws, so a seed gives the reference's noisy image
bit for bit.  Only the SeedSequence seeding (``np.random.PCG64(seed)``) runs
on the host, once per call, exactly as the reference does it.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .filters import _on_device, _stream_ptr, _torch
from .image import RasterImage, to_uint8

IMPULSE_MODES = ("saltpepper", "uniform")


@dataclass(frozen=True)
class NoiseParams:
    """Corruption probabilities, impulse distribution and RNG seed (same
    fields, defaults and ValueErrors as reference noise.py:33-55)."""

    phi: float = 0.10
    phi1: float = 0.25
    phi2: float = 0.25
    phi3: float = 0.25
    impulse: str = "saltpepper"
    seed: int = 0

    def __post_init__(self) -> None:
        if not 0.0 <= self.phi <= 1.0:
            raise ValueError(f"phi must be in [0, 1], got {self.phi}")
        for name in ("phi1", "phi2", "phi3"):
            v = getattr(self, name)
            if v < 0.0:
                raise ValueError(f"{name} must be >= 0, got {v}")
        if self.phi1 + self.phi2 + self.phi3 > 1.0 + 1e-12:
            raise ValueError("phi1 + phi2 + phi3 must not exceed 1")
        if self.impulse not in IMPULSE_MODES:
            raise ValueError(f"impulse mode must be one of {IMPULSE_MODES}")


_M64 = (1 << 64) - 1


def noise_params_c(params) -> _lib.DfgNoiseParams:
    """Pack NoiseParams (this package's or the reference's) with the PCG64
    initial state numpy derives from ``params.seed``."""
    st = np.random.PCG64(params.seed).state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    return _lib.DfgNoiseParams(
        phi=float(params.phi), phi1=float(params.phi1), phi2=float(params.phi2), phi3=float(params.phi3),
        impulse=IMPULSE_MODES.index(params.impulse), reserved=0,
        state_hi=s >> 64, state_lo=s & _M64, inc_hi=inc >> 64, inc_lo=inc & _M64)


def corrupt_device(x, params, out=None, stream=None):
    """Corrupt a CUDA uint8 tensor (H, W, 3); returns ``out`` (new if None).
    ``x`` and ``out`` may alias (the kernel reads each pixel before writing
    it, pixel by pixel in the same thread)."""
    torch = _torch()
    if x.dtype != torch.uint8 or x.dim() != 3 or x.shape[2] != 3 or not x.is_cuda:
        raise ValueError("expected a CUDA uint8 tensor of shape (H, W, 3)")
    if x.stride(2) != 1 or x.stride(1) != 3:
        x = x.contiguous()
    H, W = int(x.shape[0]), int(x.shape[1])
    if out is None:
        out = torch.empty((H, W, 3), dtype=torch.uint8, device=x.device)
    np_c = noise_params_c(params)
    with _on_device(torch, x.device):
        rc = _lib.lib().dfg_corrupt_image(ctypes.c_void_p(x.data_ptr()), H, W, x.stride(0),
                                          ctypes.c_void_p(out.data_ptr()), out.stride(0), ctypes.byref(np_c),
                                          _stream_ptr(torch, stream, x.device))
    _lib.check(rc)
    return out


def corrupt_image(img, params, *, device=None) -> RasterImage:
    """Corrupt every pixel independently; deterministic given params.seed
    (reference noise.py:85-116).  8-bit pixel values only (the device path);
    returns a new float64 RasterImage like the reference."""
    pixels = img.pixels if hasattr(img, "pixels") else np.asarray(img)
    u8 = to_uint8(pixels)
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index)
    out = corrupt_device(torch.from_numpy(u8).to(dev), params)
    return RasterImage._adopt(out.cpu().numpy().astype(np.float64))
