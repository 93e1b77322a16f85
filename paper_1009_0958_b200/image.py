"""Image container and border policy, mirroring the reference's L1 types.

``RasterImage`` keeps the reference's contract (reference
``pkg/src/dirfilt/image.py:58-124``): an immutable (M, N, 3) float64 pixel
array, validated finite and nonnegative.  ``BorderPolicy`` is
replicate (numpy.pad 'edge') or reflect (numpy.pad 'symmetric';
``image.py:32-55,158-176``).

The GPU path works on uint8 RGB; ``to_uint8`` is the lossless boundary
conversion and rejects images whose components are not integers in
[0, 255] -- the reference accepts any finite nonnegative float64, so that is
the one documented input restriction of the drop-in.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

import numpy as np


class ColorVector(NamedTuple):
    x1: float
    x2: float
    x3: float


@dataclass(frozen=True)
class BorderPolicy:
    """Out-of-image window coordinates: ``replicate`` clamps, ``reflect``
    mirrors about the edge with the edge pixel included."""

    mode: str = "replicate"

    def __post_init__(self) -> None:
        if self.mode not in ("replicate", "reflect"):
            raise ValueError(f"unknown border mode {self.mode!r}")

    @property
    def pad_mode(self) -> str:
        return {"replicate": "edge", "reflect": "symmetric"}[self.mode]


REPLICATE = BorderPolicy("replicate")
REFLECT = BorderPolicy("reflect")


class RasterImage:
    """Immutable M x N RGB image, float64 (M, N, 3)."""

    __slots__ = ("_px",)

    def __init__(self, pixels) -> None:
        a = np.array(pixels, dtype=np.float64, copy=True)
        if a.ndim != 3 or a.shape[2] != 3:
            raise ValueError(f"pixel array must have shape (M, N, 3), got {a.shape}")
        if a.shape[0] < 1 or a.shape[1] < 1:
            raise ValueError("image must contain at least one pixel")
        if not np.isfinite(a).all() or (a < 0).any():
            raise ValueError("pixel components must be finite and nonnegative")
        a.flags.writeable = False
        self._px = a

    @classmethod
    def _adopt(cls, arr: np.ndarray) -> "RasterImage":
        """Wrap a freshly produced float64 array without copying."""
        obj = cls.__new__(cls)
        arr.flags.writeable = False
        obj._px = arr
        return obj

    _wrap = _adopt  # the reference's private spelling

    @classmethod
    def from_uint8(cls, arr: np.ndarray) -> "RasterImage":
        a = np.asarray(arr)
        if a.dtype != np.uint8 or a.ndim != 3 or a.shape[2] != 3:
            raise ValueError("expected a uint8 (M, N, 3) array")
        return cls._adopt(a.astype(np.float64))

    @property
    def rows(self) -> int:
        return self._px.shape[0]

    @property
    def cols(self) -> int:
        return self._px.shape[1]

    @property
    def pixels(self) -> np.ndarray:
        return self._px

    def pixel(self, r: int, c: int) -> ColorVector:
        """Pixel at 1-based (r, c)."""
        if not (1 <= r <= self.rows and 1 <= c <= self.cols):
            raise ValueError(f"coordinate ({r}, {c}) outside 1..{self.rows} x 1..{self.cols}")
        v = self._px[r - 1, c - 1]
        return ColorVector(float(v[0]), float(v[1]), float(v[2]))

    def __eq__(self, other: object) -> bool:
        px = getattr(other, "pixels", None)
        if not isinstance(px, np.ndarray):
            return NotImplemented
        return px.shape == self._px.shape and bool((px == self._px).all())

    __hash__ = None  # mutable-equality semantics, like the reference

    def __repr__(self) -> str:
        return f"RasterImage({self.rows}x{self.cols})"


def to_uint8(pixels: np.ndarray) -> np.ndarray:
    """float64 (M, N, 3) with integer values 0..255 -> uint8, else ValueError."""
    a = np.asarray(pixels)
    if a.dtype == np.uint8:
        return np.ascontiguousarray(a)
    if a.ndim != 3 or a.shape[2] != 3:
        raise ValueError(f"pixel array must have shape (M, N, 3), got {a.shape}")
    if not np.isfinite(a).all() or (a < 0).any() or (a > 255).any() or (a != np.floor(a)).any():
        raise ValueError("the GPU path requires integer pixel components in [0, 255] "
                         "(8-bit RGB); got non-integral or out-of-range values")
    return np.ascontiguousarray(a, dtype=np.uint8)
