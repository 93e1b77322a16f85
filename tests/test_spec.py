"""CPU: the host-side mirror of the reference's spec/image interface keeps
its names, defaults, grammar and ValueError behaviour (reference
T/test_filters.py:269-302, T/test_distance.py:245-311, T/test_image.py)."""

import math

import numpy as np
import pytest

import oracle
from paper_1009_0958_b200 import (
    ACOS_COEFFICIENTS, ASIN_COEFFICIENTS, REFLECT, REPLICATE, AcwddfParams, BorderPolicy, DirectionalStrategy,
    FastAcosTable, FilterSpec, MinimaxPoly, RasterImage, center_weight, parse_filter_spec, to_uint8,
)


def test_parse_round_trip():
    for text in ["identity", "vmf", "bvdf:minimax:q=4", "bvdf:rgb", "ddf:exact:p=2", "acwddf:minimax:q=4:lambda=2:T=10.8",
                 "acwddf:rgb:lambda=3:T=5", "vmf:p=1:window=5", "ddf:minimax:q=3:window=7", "bvdf:rgb:p=1.5"]:
        spec = parse_filter_spec(text)
        assert parse_filter_spec(spec.name) == spec


def test_defaults():
    spec = parse_filter_spec("bvdf")
    assert spec.strategy.kind == "exact" and spec.p == 2.0 and spec.window == 3
    assert parse_filter_spec("acwddf:minimax").acwddf == AcwddfParams(2, 10.8, 2.0)
    rgb = parse_filter_spec("ddf:rgb").strategy
    assert (rgb.slope, rgb.intercept) == (1.436437, 0.027664)


@pytest.mark.parametrize("text", ["", "foo", "bvdf:fuzzy", "vmf:q=x", "bvdf:minimax:q=7", "vmf:window=4",
                                  "bvdf:bogus=1", "acwddf:lambda=9", "ddf:p=0.5", "acwddf:T=-1", "bvdf:rgb:slope=0"])
def test_invalid_specs_raise_value_error(text):
    with pytest.raises(ValueError):
        parse_filter_spec(text)


def test_acwddf_params_pairing_and_center_weight():
    with pytest.raises(ValueError):
        FilterSpec(family="vmf", acwddf=AcwddfParams())
    with pytest.raises(ValueError):
        FilterSpec(family="acwddf")
    assert [center_weight(9, k) for k in range(1, 6)] == [9, 7, 5, 3, 1]
    for bad in (0, 6):
        with pytest.raises(ValueError):
            center_weight(9, bad)


def test_coefficient_tables_match_oracle_copy():
    for q in (2, 3, 4):
        assert ASIN_COEFFICIENTS[q][1] == oracle.ASIN[q]
        assert ACOS_COEFFICIENTS[q][1] == oracle.ACOS[q]
        t = FastAcosTable.for_degree(q)
        assert abs(t.asin_poly.coefficients[1] - math.sqrt(2)) < 0.05
    with pytest.raises(ValueError):
        FastAcosTable.for_degree(5)
    with pytest.raises(ValueError):
        MinimaxPoly(2, (1.0, 2.0), (0.0, 1.0), 1e-3)
    poly = MinimaxPoly(2, (1.0, -2.0, 3.0), (0.0, 1.0), 1.0)
    assert poly(0.37) == 1.0 + 0.37 * (-2.0 + 0.37 * 3.0)


def test_reference_spec_objects_are_accepted():
    """Duck typing: the C-ABI packer takes the reference's FilterSpec too
    (here a stand-in with the same attribute names)."""
    from types import SimpleNamespace

    from paper_1009_0958_b200 import _lib

    ref_like = SimpleNamespace(family="acwddf", window=5, p=2.0,
                               strategy=SimpleNamespace(kind="minimax", q=3, slope=1.4, intercept=0.02,
                                                        table=FastAcosTable.for_degree(3)),
                               acwddf=SimpleNamespace(lam=2, threshold=7.5, p=1.0))
    prm = _lib.params_from_spec(ref_like, REFLECT)
    assert (prm.family, prm.strategy, prm.window, prm.border) == (4, 1, 5, 1)
    assert prm.p == 1.0 and prm.lam == 2 and prm.threshold == 7.5
    assert tuple(prm.asin_c) == ASIN_COEFFICIENTS[3][1] + (0.0,)


def test_raster_image_and_border_policy():
    with pytest.raises(ValueError):
        RasterImage(np.zeros((2, 2)))
    with pytest.raises(ValueError):
        RasterImage(np.full((2, 2, 3), -1.0))
    with pytest.raises(ValueError):
        RasterImage(np.full((2, 2, 3), np.nan))
    img = RasterImage(np.arange(12, dtype=float).reshape(2, 2, 3))
    assert not img.pixels.flags.writeable
    assert tuple(img.pixel(2, 2)) == (9.0, 10.0, 11.0)
    assert img == RasterImage(img.pixels)
    with pytest.raises(ValueError):
        BorderPolicy("wrap")
    assert (REPLICATE.pad_mode, REFLECT.pad_mode) == ("edge", "symmetric")


def test_uint8_boundary_conversion():
    a = np.array([[[0.0, 128.0, 255.0]]])
    assert to_uint8(a).tolist() == [[[0, 128, 255]]]
    for bad in (0.5, 256.0, -1.0, np.inf):
        with pytest.raises(ValueError):
            to_uint8(np.full((1, 1, 3), bad))


def test_centre_weighted_spec_validation():
    from paper_1009_0958_b200 import CenterWeightedSpec, DirectionalStrategy
    s = CenterWeightedSpec("cwddf", 3, DirectionalStrategy.minimax(2), window=5)
    assert s.name == "cwddf:k=3:minimax:q=2:window=5"
    assert CenterWeightedSpec("cwvmf", 1).name == "cwvmf:k=1"
    for bad in (dict(family="vmf", k=1), dict(family="cwvmf", k=0), dict(family="cwvmf", k=6),
                dict(family="cwddf", k=2, p=0.5), dict(family="cwddf", k=2, window=4)):
        with pytest.raises(ValueError):
            CenterWeightedSpec(**bad)
