"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports the reference package ``dirfilt`` read-only from
/root/reference/pkg/src, runs its ``apply_filter`` (filters.py:379-433) on
seeded inputs, and stores inputs + outputs as uint8 arrays in
``filters.npz`` with a JSON manifest (spec text, border policy, case kind).
It also stores the reference's scalar distances (distance.py) for known-answer
pairs, and the reference's correlated-noise simulator output
(noise.py:85-116) used to pin ``synth.add_correlated_noise``.

The committed fixtures travel with the repo; nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import dirfilt  # noqa: E402  (the reference)
from dirfilt import (  # noqa: E402
    BorderPolicy, NoiseParams, RasterImage, apply_filter, compare, corrupt_image, parse_filter_spec,
)
from dirfilt.distance import (  # noqa: E402
    FastAcosTable, angular_distance_exact, chromaticity_distance, minkowski_distance,
)

from paper_1009_0958_b200 import synth  # noqa: E402  (input generator only)

ALL_SPECS = [
    "vmf", "vmf:p=1", "vmf:p=3",
    "bvdf:exact", "bvdf:minimax", "bvdf:minimax:q=2", "bvdf:minimax:q=3", "bvdf:rgb", "bvdf:rgb:p=1",
    "ddf:exact", "ddf:minimax", "ddf:rgb", "ddf:exact:p=1", "ddf:minimax:q=3",
    "acwddf:exact", "acwddf:minimax", "acwddf:rgb", "acwddf:exact:lambda=3:T=5",
]


def main() -> None:
    cases = []
    arrays = {}

    def add(kind, spec, border, img_u8):
        ref = RasterImage(img_u8.astype(np.float64))
        out = apply_filter(ref, parse_filter_spec(spec), BorderPolicy(border)).pixels
        assert (out == np.floor(out)).all() and out.max() <= 255
        i = len(cases)
        arrays[f"in{i}"] = img_u8
        arrays[f"out{i}"] = out.astype(np.uint8)
        cases.append({"kind": kind, "spec": spec, "border": border})

    rng = np.random.default_rng(41)
    # 1. random 8x8 images, every spec, both borders (T/test_filters.py:347-359 style)
    for spec in ALL_SPECS:
        for border in ("replicate", "reflect"):
            for _ in range(2):
                add("random8", spec, border, rng.integers(0, 256, (8, 8, 3), dtype=np.uint8))
    # 2. larger windows on random images
    for spec in ("bvdf:exact:window=5", "bvdf:minimax:window=5", "bvdf:rgb:window=5", "ddf:exact:window=5",
                 "ddf:minimax:window=5", "ddf:rgb:window=5", "acwddf:exact:window=5", "acwddf:rgb:window=5:lambda=3",
                 "acwddf:minimax:window=5", "vmf:window=5", "ddf:exact:window=7", "bvdf:minimax:window=7",
                 "bvdf:exact:window=7", "vmf:window=7", "acwddf:exact:window=7", "ddf:rgb:window=7"):
        for border in ("replicate", "reflect"):
            add("random_w", spec, border, rng.integers(0, 256, (11, 13, 3), dtype=np.uint8))
    # 3. tiny images: border resolution with sizes below the window (image.py:158-169)
    for shape in ((1, 1), (1, 5), (2, 2), (3, 7), (5, 1), (2, 9)):
        for spec in ("bvdf:exact", "ddf:minimax:window=5", "acwddf:exact", "vmf:window=7", "bvdf:rgb:window=7"):
            for border in ("replicate", "reflect"):
                add("tiny", spec, border, rng.integers(0, 256, shape + (3,), dtype=np.uint8))
    # 4. structured images: constant, parallel ramps, zero vectors, two colours
    const = np.full((6, 6, 3), 99, np.uint8)
    par = np.zeros((9, 9, 3), np.uint8)
    for i in range(9):
        for j in range(9):
            k = 1 + (i * 9 + j) % 40
            par[i, j] = (k, 2 * k, 3 * k)
    zeros = rng.integers(0, 3, (10, 10, 3), dtype=np.uint8)
    twoc = np.where(rng.random((12, 12, 1)) < 0.5, np.uint8(10), np.uint8(200)) * np.ones((1, 1, 3), np.uint8)
    for name, img in (("const", const), ("parallel", par), ("near_zero", zeros), ("two_colour", twoc)):
        for spec in ("vmf", "bvdf:exact", "bvdf:minimax", "bvdf:rgb", "ddf:exact", "ddf:minimax", "ddf:rgb",
                     "acwddf:exact", "acwddf:minimax", "acwddf:rgb", "bvdf:exact:window=5", "ddf:exact:window=7"):
            add(name, spec, "replicate", img)
    # 5. config-like crops (seeded generator of SURVEY 8(d), reduced shapes)
    cfg_like = [
        ("bvdf:exact", ("uncorrelated", 0.10), 1), ("ddf:exact", ("uncorrelated", 0.15), 2),
        ("acwddf:exact:window=5", ("correlated", 0.20), 3), ("bvdf:minimax:window=5", ("uncorrelated", 0.10), 4),
        ("bvdf:rgb:window=5", ("uncorrelated", 0.10), 4), ("ddf:minimax:window=5", ("uncorrelated", 0.10), 4),
        ("ddf:rgb:window=5", ("uncorrelated", 0.10), 4), ("ddf:exact:window=7", ("correlated", 0.20), 5),
        ("acwddf:exact", ("uncorrelated", 0.10), 1000),
    ]
    for spec, noise, seed in cfg_like:
        add("config_like", spec, "replicate", synth.noisy_image(40, 56, seed, noise))
    # 6. acceptance criterion 4 (T/test_acceptance.py:169-195): 100 random 8x8, 4 specs
    rng4 = np.random.default_rng(1234)
    acc = rng4.integers(0, 256, (100, 8, 8, 3)).astype(np.uint8)
    acc_out = {}
    for spec in ("vmf", "bvdf:exact", "ddf:exact", "acwddf:exact"):
        outs = [apply_filter(RasterImage(a.astype(np.float64)), parse_filter_spec(spec)).pixels for a in acc]
        acc_out[spec] = np.stack(outs).astype(np.uint8)
    arrays["acc_in"] = acc
    for k, v in acc_out.items():
        arrays["acc_out_" + k.replace(":", "_")] = v

    # scalar distances (engine form: distinct pairs only)
    prs = rng.integers(0, 256, (400, 2, 3)).astype(np.float64)
    prs[0] = [[0, 0, 0], [9, 9, 9]]
    prs[1] = [[1, 2, 3], [40, 80, 120]]
    prs[2] = [[255, 0, 0], [0, 255, 0]]
    prs[3] = [[0, 0, 0], [255, 0, 0]]
    V = dirfilt.ColorVector
    dist = {"pairs": prs, "exact": [], "chroma2": [], "chroma1": [], "l2": [], "minimax2": [], "minimax3": [],
            "minimax4": []}
    for a, b in prs:
        va, vb = V(*a), V(*b)
        dist["exact"].append(angular_distance_exact(va, vb))
        dist["chroma2"].append(chromaticity_distance(va, vb, 2.0))
        dist["chroma1"].append(chromaticity_distance(va, vb, 1.0))
        dist["l2"].append(minkowski_distance(va, vb, 2.0))
        for q in (2, 3, 4):
            dist[f"minimax{q}"].append(dirfilt.angular_distance_minimax(va, vb, FastAcosTable.for_degree(q)))
    for k, v in dist.items():
        arrays["dist_" + k] = np.asarray(v, dtype=np.float64)

    # correlated noise simulator (noise.py:85-116) on a seeded clean image
    clean = synth.clean_image(64, 80, 3)
    noisy = corrupt_image(RasterImage(clean.astype(np.float64)),
                          NoiseParams(phi=0.2, phi1=0.0, phi2=0.0, phi3=0.0, impulse="uniform", seed=3 + 10**6))
    arrays["noise_clean"] = clean
    arrays["noise_ref"] = noisy.pixels.astype(np.uint8)

    # the full simulator: both impulse modes, all four branches, a pixel
    # count that is not a multiple of the device's 16-pixel runs
    noise_cases = [
        ("sp_default", (37, 53), dict(seed=7)),
        ("uni_mixed", (41, 61), dict(phi=0.5, phi1=0.1, phi2=0.2, phi3=0.3, impulse="uniform", seed=123456789)),
        ("sp_all", (9, 7), dict(phi=1.0, phi1=0.0, phi2=0.0, phi3=0.0, seed=2**63 + 5)),
        ("sp_branch3", (16, 33), dict(phi=0.9, phi1=0.0, phi2=0.0, phi3=1.0, seed=0)),
    ]
    noise_manifest = []
    for name, (h, w), kw in noise_cases:
        img = synth.clean_image(h, w, len(noise_manifest) + 40)
        out = corrupt_image(RasterImage(img.astype(np.float64)), NoiseParams(**kw)).pixels
        arrays[f"noise_{name}_in"] = img
        arrays[f"noise_{name}_out"] = out.astype(np.uint8)
        noise_manifest.append({"name": name, **kw})

    # effectiveness criteria (metrics.py:64-118) on a few image pairs
    pairs = [("noise_clean", "noise_ref"), ("noise_sp_default_in", "noise_sp_default_out"),
             ("noise_uni_mixed_in", "noise_uni_mixed_out"), ("noise_clean", "noise_clean"),
             ("in0", "out0")]
    met = []
    for a, b in pairs:
        r = compare(RasterImage(arrays[a].astype(np.float64)), RasterImage(arrays[b].astype(np.float64)))
        met.append([r.mae, r.psnr, r.ncd_x1000])
    arrays["metrics_ref"] = np.asarray(met, dtype=np.float64)

    # calibration line (calibration.py:83-125): samples of a small draw and
    # fitted lines for a few (pairs, seed, p, method)
    from dirfilt.calibration import fit_angular_chromaticity, sample_angle_chromaticity_pairs
    cb, ca = sample_angle_chromaticity_pairs(2000, 7, 2.0)
    arrays["calib_b"], arrays["calib_a"] = cb, ca
    cb3, ca3 = sample_angle_chromaticity_pairs(1500, 8, 3.0)
    arrays["calib_b_p3"], arrays["calib_a_p3"] = cb3, ca3
    calib_cases = [(10**4, 0, 2.0, "tls"), (10**5, 1, 2.0, "ols"), (20000, 3, 1.0, "tls"), (10**6, 0, 2.0, "tls")]
    fits = []
    for n, sd, pp, meth in calib_cases:
        f = fit_angular_chromaticity(n, sd, pp, meth)
        fits.append([f.slope, f.intercept, f.fit_error, f.mean_abs_residual, f.rms_orthogonal])
    arrays["calib_fits"] = np.asarray(fits, dtype=np.float64)

    # centre-weighted filters (filters.py:296-337) applied to every window via
    # the reference's extract_window (image.py:179-200)
    from dirfilt.filters import cwddf, cwvmf
    from dirfilt.image import extract_window
    cw_cases = []
    cw_specs = [("cwvmf", 1, "ddf:exact", 2.0, 3), ("cwvmf", 3, "ddf:exact", 2.0, 3), ("cwvmf", 2, "ddf:exact", 1.0, 3),
                ("cwvmf", 5, "ddf:exact", 2.0, 3), ("cwvmf", 7, "ddf:exact", 2.0, 5), ("cwvmf", 4, "ddf:exact", 3.0, 5),
                ("cwddf", 1, "ddf:exact", 2.0, 3), ("cwddf", 2, "ddf:exact", 2.0, 3), ("cwddf", 4, "ddf:minimax", 2.0, 3),
                ("cwddf", 3, "ddf:minimax:q=2", 2.0, 3), ("cwddf", 2, "ddf:rgb", 2.0, 3), ("cwddf", 5, "ddf:exact", 2.0, 3),
                ("cwddf", 6, "ddf:exact", 2.0, 5), ("cwddf", 9, "ddf:minimax", 2.0, 5), ("cwddf", 3, "ddf:rgb", 1.0, 5),
                ("cwddf", 13, "ddf:exact", 2.0, 5), ("cwddf", 10, "ddf:exact", 2.0, 7)]
    for ci, (fam, k, stext, pp, win) in enumerate(cw_specs):
        for border in ("replicate", "reflect"):
            h, w = (11, 13) if win < 7 else (9, 10)
            img = synth.noisy_image(h, w, 500 + ci, ("correlated", 0.25))
            img[2:4, 3:6] = 0
            img[6:8, 1:3] = img[0, 0]  # duplicate colours (minimax a == b rule)
            ref = RasterImage(img.astype(np.float64))
            strat = parse_filter_spec(stext).strategy
            pol = BorderPolicy(border)
            out = np.zeros_like(img)
            for r in range(h):
                for c in range(w):
                    wv = extract_window(ref, r + 1, c + 1, win, pol)
                    v = cwvmf(wv, k, pp) if fam == "cwvmf" else cwddf(wv, k, pp, strat)
                    out[r, c] = (int(v.x1), int(v.x2), int(v.x3))
            i = len(cw_cases)
            arrays[f"cw_in{i}"] = img
            arrays[f"cw_out{i}"] = out
            cw_cases.append({"family": fam, "k": k, "strategy": stext.split(":", 1)[1], "p": pp, "window": win,
                             "border": border})

    np.savez_compressed(HERE / "filters.npz", **arrays)
    (HERE / "manifest.json").write_text(json.dumps({"reference": "dirfilt 0.1.0 (/root/reference/pkg)",
                                                    "numpy": np.__version__, "cases": cases,
                                                    "noise_cases": noise_manifest,
                                                    "metrics_pairs": pairs,
                                                    "calib_cases": calib_cases,
                                                    "cw_cases": cw_cases}, indent=1))
    print(f"{len(cases)} filter cases, {sum(a.nbytes for a in arrays.values())} bytes raw")


if __name__ == "__main__":
    main()
