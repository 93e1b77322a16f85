"""Seeded synthetic inputs standing in for the paper's photographs.

The paper measures on standard test photographs that are
not redistributable; BASELINE.json's configs define seeded synthetic images
instead: a linear colour gradient plus 20 uniformly coloured
axis-aligned rectangles, then impulsive noise -- uncorrelated (each channel
replaced independently with probability p) or correlated (the reference's
Eq. 8 simulator with phi1 = phi2 = phi3 = 0 and uniform impulses, i.e. all
three channels of a hit pixel replaced; reference noise.py:85-116, which
draws five uniform doubles per pixel from a PCG64 stream).

Large frames are generated in row bands; the band size is part of the
definition (streams are consumed band by band in a fixed order).
"""

from __future__ import annotations

import numpy as np

BAND = 256  # rows per generation band

# BASELINE.json configs (SURVEY.md 8(d) seeds: image seed; noise seed = seed + 10**6)
CONFIGS = {
    "c1": dict(spec="bvdf:exact", shape=(512, 512), noise=("uncorrelated", 0.10), seed=1),
    "c2": dict(spec="ddf:exact", shape=(1024, 1024), noise=("uncorrelated", 0.15), seed=2),
    "c3": dict(spec="acwddf:exact:window=5", shape=(2048, 2048), noise=("correlated", 0.20), seed=3),
    "c4_bvdf_minimax": dict(spec="bvdf:minimax:window=5", shape=(4096, 4096), noise=("uncorrelated", 0.10), seed=4),
    "c4_bvdf_rgb": dict(spec="bvdf:rgb:window=5", shape=(4096, 4096), noise=("uncorrelated", 0.10), seed=4),
    "c4_ddf_minimax": dict(spec="ddf:minimax:window=5", shape=(4096, 4096), noise=("uncorrelated", 0.10), seed=4),
    "c4_ddf_rgb": dict(spec="ddf:rgb:window=5", shape=(4096, 4096), noise=("uncorrelated", 0.10), seed=4),
    "c5a": dict(spec="ddf:exact:window=7", shape=(8192, 8192), noise=("correlated", 0.20), seed=5),
    "c5b": dict(spec="acwddf:exact", shape=(1080, 1920), noise=("uncorrelated", 0.10), seed=1000, frames=64),
}


def clean_image(H: int, W: int, seed: int, n_rects: int = 20) -> np.ndarray:
    """Gradient + rectangles, uint8 (H, W, 3)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    c00, c10, c01 = (rng.integers(0, 256, 3).astype(np.float64) for _ in range(3))
    xs = np.arange(W, dtype=np.float64) / max(W - 1, 1)
    out = np.empty((H, W, 3), dtype=np.uint8)
    for r0 in range(0, H, BAND):
        r1 = min(H, r0 + BAND)
        ys = (np.arange(r0, r1, dtype=np.float64) / max(H - 1, 1))[:, None, None]
        band = c00 + (c10 - c00) * xs[None, :, None] + (c01 - c00) * ys
        out[r0:r1] = np.clip(np.rint(band), 0, 255).astype(np.uint8)
    hlo, hhi = max(1, H // 32), max(2, H // 4)
    wlo, whi = max(1, W // 32), max(2, W // 4)
    for _ in range(n_rects):
        h = int(rng.integers(hlo, hhi))
        w = int(rng.integers(wlo, whi))
        y0 = int(rng.integers(0, max(1, H - h + 1)))
        x0 = int(rng.integers(0, max(1, W - w + 1)))
        col = rng.integers(0, 256, 3).astype(np.uint8)
        out[y0:y0 + h, x0:x0 + w] = col
    return out


def add_uncorrelated_noise(img: np.ndarray, p: float, seed: int) -> np.ndarray:
    """Each channel independently replaced with probability p by U{0..255}."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = img.copy()
    H = img.shape[0]
    for r0 in range(0, H, BAND):
        r1 = min(H, r0 + BAND)
        shape = out[r0:r1].shape
        hit = rng.random(shape) < p
        vals = rng.integers(0, 256, shape, dtype=np.uint8)
        band = out[r0:r1]
        band[hit] = vals[hit]
    return out


def add_correlated_noise(img: np.ndarray, p: float, seed: int) -> np.ndarray:
    """Eq. 8 with phi1 = phi2 = phi3 = 0, uniform impulses: a pixel is hit
    with probability p and then all three channels become floor(u * 256).
    Consumes the reference simulator's stream layout (5 doubles per pixel,
    row-major)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = img.copy()
    H, W = img.shape[:2]
    for r0 in range(0, H, BAND):
        r1 = min(H, r0 + BAND)
        d = rng.random(((r1 - r0) * W, 5))
        hit = (d[:, 0] < p).reshape(r1 - r0, W)
        imp = np.floor(d[:, 2:5] * 256.0).astype(np.uint8).reshape(r1 - r0, W, 3)
        band = out[r0:r1]
        band[hit] = imp[hit]
    return out


def noisy_image(H: int, W: int, seed: int, noise=("uncorrelated", 0.10)) -> np.ndarray:
    kind, p = noise
    img = clean_image(H, W, seed)
    if kind == "uncorrelated":
        return add_uncorrelated_noise(img, p, seed + 10**6)
    if kind == "correlated":
        return add_correlated_noise(img, p, seed + 10**6)
    raise ValueError(f"unknown noise kind {kind!r}")


def config_input(name: str, frames: int | None = None):
    """The seeded input of a BASELINE config: uint8 (H, W, 3), or (B, H, W, 3)
    for the frame batch (``frames`` limits the batch)."""
    cfg = CONFIGS[name]
    H, W = cfg["shape"]
    if "frames" in cfg:
        B = cfg["frames"] if frames is None else min(frames, cfg["frames"])
        return np.stack([noisy_image(H, W, cfg["seed"] + i, cfg["noise"]) for i in range(B)])
    return noisy_image(H, W, cfg["seed"], cfg["noise"])
