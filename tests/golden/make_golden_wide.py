"""Golden fixtures for window sides above 7, from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_wide.py

The reference accepts any odd window side >= 3 (filters.py:141-151); its
``apply_filter`` (filters.py:379-433) is run on seeded inputs for sides 9, 11
and 13 and the inputs + outputs are stored as uint8 arrays in ``wide.npz``
with ``wide_manifest.json``.  Nothing at test time reads /root/reference.
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

from dirfilt import BorderPolicy, RasterImage, apply_filter, parse_filter_spec  # noqa: E402  (the reference)

from paper_1009_0958_b200 import synth  # noqa: E402  (input generator only)

SPECS = [
    "vmf:window=9", "vmf:window=9:p=1", "bvdf:exact:window=9", "bvdf:minimax:window=9", "bvdf:rgb:window=9",
    "ddf:exact:window=9", "ddf:minimax:window=9:q=3", "ddf:rgb:window=9", "ddf:exact:window=9:p=3",
    "acwddf:exact:window=9", "acwddf:minimax:window=9", "acwddf:rgb:window=9:lambda=5", "acwddf:exact:window=9:lambda=7:T=40",
    "bvdf:exact:window=11", "ddf:exact:window=11", "acwddf:exact:window=11", "ddf:rgb:window=11:p=1",
    "ddf:exact:window=13", "bvdf:minimax:window=13",
]


def main() -> None:
    cases, arrays = [], {}

    def add(kind, spec, border, img_u8):
        out = apply_filter(RasterImage(img_u8.astype(np.float64)), parse_filter_spec(spec), BorderPolicy(border)).pixels
        assert (out == np.floor(out)).all() and out.max() <= 255
        i = len(cases)
        arrays[f"in{i}"] = img_u8
        arrays[f"out{i}"] = out.astype(np.uint8)
        cases.append({"kind": kind, "spec": spec, "border": border})

    rng = np.random.default_rng(97)
    for spec in SPECS:
        for border in ("replicate", "reflect"):
            add("random", spec, border, rng.integers(0, 256, (14, 17, 3), dtype=np.uint8))
    # images smaller than the window (periodic reflection, image.py:158-169), zero vectors, duplicates
    for shape in ((1, 1), (3, 5), (8, 2)):
        for spec in ("ddf:exact:window=9", "acwddf:minimax:window=9", "bvdf:rgb:window=11"):
            for border in ("replicate", "reflect"):
                add("tiny", spec, border, rng.integers(0, 256, shape + (3,), dtype=np.uint8))
    zeros = rng.integers(0, 3, (12, 12, 3), dtype=np.uint8)
    twoc = np.where(rng.random((13, 13, 1)) < 0.5, np.uint8(10), np.uint8(200)) * np.ones((1, 1, 3), np.uint8)
    for name, img in (("near_zero", zeros), ("two_colour", twoc)):
        for spec in ("bvdf:exact:window=9", "ddf:exact:window=9", "ddf:minimax:window=9", "acwddf:exact:window=9",
                     "vmf:window=9"):
            add(name, spec, "replicate", img)
    # config-like content
    for spec, noise, seed in (("ddf:exact:window=9", ("correlated", 0.20), 5),
                              ("acwddf:exact:window=9", ("correlated", 0.20), 3),
                              ("bvdf:minimax:window=9", ("uncorrelated", 0.10), 4)):
        add("config_like", spec, "replicate", synth.noisy_image(24, 31, seed, noise))
    np.savez_compressed(HERE / "wide.npz", **arrays)
    (HERE / "wide_manifest.json").write_text(json.dumps({"reference": "dirfilt 0.1.0 (/root/reference/pkg)",
                                                         "numpy": np.__version__, "cases": cases}, indent=1))
    print(f"{len(cases)} wide-window cases, {sum(a.nbytes for a in arrays.values())} bytes raw")


if __name__ == "__main__":
    main()
