"""CPU: the product path has no CPU fallback and never touches the oracle."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_product_package_never_references_the_oracle():
    for f in (ROOT / "paper_1009_0958_b200").rglob("*"):
        if f.suffix in (".py", ".cu", ".cuh", ".h", ".c", ".cpp"):
            txt = f.read_text()
            assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
            assert "liboracle" not in txt and "orc_" not in txt, f


def test_apply_filter_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    from paper_1009_0958_b200 import RasterImage, apply_filter, parse_filter_spec

    with pytest.raises(RuntimeError, match="CUDA"):
        apply_filter(RasterImage(np.full((4, 4, 3), 7.0)), parse_filter_spec("bvdf:exact"))
