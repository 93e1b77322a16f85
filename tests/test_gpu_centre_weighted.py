"""GPU: the centre-weighted filters -- the reference's
window-level cwvmf / cwddf (filters.py:296-337) applied to every window --
on the same kernels as the engine families, bit-exact with the reference's
fixtures and with the oracle on larger seeded images, both 3x3 schedules."""

import numpy as np
import pytest

import oracle
from paper_1009_0958_b200 import _lib
from paper_1009_0958_b200 import (
    REFLECT, REPLICATE, CenterWeightedSpec, RasterImage, apply_filter, filter_device, parse_filter_spec, synth,
)

pytestmark = pytest.mark.gpu


def _spec(c):
    strat = parse_filter_spec("ddf:" + c["strategy"]).strategy
    return CenterWeightedSpec(c["family"], c["k"], strat, c["p"], c["window"])


def _pol(b):
    return REPLICATE if b == "replicate" else REFLECT


def test_reference_fixtures(cuda, golden_full):
    data, man = golden_full
    for i, c in enumerate(man["cw_cases"]):
        img = RasterImage(data[f"cw_in{i}"].astype(np.float64))
        got = apply_filter(img, _spec(c), _pol(c["border"])).pixels.astype(np.uint8)
        assert (got == data[f"cw_out{i}"]).all(), (i, c)


CW = [("cwvmf", 2, "exact", 2.0, 3), ("cwvmf", 4, "exact", 1.0, 3), ("cwddf", 2, "exact", 2.0, 3),
      ("cwddf", 3, "minimax", 2.0, 3), ("cwddf", 1, "rgb", 2.0, 3), ("cwddf", 4, "exact", 3.0, 3),
      ("cwvmf", 8, "exact", 2.0, 5), ("cwddf", 6, "exact", 2.0, 5), ("cwddf", 11, "minimax:q=3", 2.0, 5),
      ("cwddf", 9, "rgb", 2.0, 5), ("cwddf", 20, "exact", 2.0, 7), ("cwvmf", 15, "exact", 2.0, 7)]


@pytest.mark.parametrize("kernel", ["w3", "cta"])
@pytest.mark.parametrize("fam,k,strat,p,win", CW)
def test_against_oracle(cuda, fam, k, strat, p, win, kernel):
    if win != 3 and kernel == "cta":
        pytest.skip("one schedule for 5x5/7x7")
    with _lib.option("s3_schedule", 1 if kernel == "w3" else 2):
        _check(cuda, fam, k, strat, p, win)


def _check(torch, fam, k, strat, p, win):
    s = _spec({"family": fam, "k": k, "strategy": strat, "p": p, "window": win})
    for H, W, seed, border in ((97, 61, 3, "replicate"), (40, 29, 4, "reflect")):
        img = synth.noisy_image(H, W, seed, ("correlated", 0.2))
        img[5:9, 7:12] = 0
        img[20:24, 3:9] = img[0, 0]
        want = oracle.filter_image(img, s, border)
        got = filter_device(torch.from_numpy(img).cuda(), s, _pol(border)).cpu().numpy()
        assert (got == want).all(), (s.name, kernel, H, W, int((got != want).any(-1).sum()))


def test_limits_reduce_to_centre_and_plain_filter(cuda):
    """k = 1 pins every output to the centre pixel; k = (n+1)/2 (weight 1)
    is the plain VMF / DDF (center_weight, filters.py:85-94)."""
    torch = cuda
    img = synth.noisy_image(64, 70, 9, ("uncorrelated", 0.15))
    x = torch.from_numpy(img).cuda()
    assert (filter_device(x, CenterWeightedSpec("cwvmf", 1)).cpu().numpy() == img).all()
    assert (filter_device(x, CenterWeightedSpec("cwddf", 1)).cpu().numpy() == img).all()
    assert torch.equal(filter_device(x, CenterWeightedSpec("cwvmf", 5)), filter_device(x, parse_filter_spec("vmf")))
    assert torch.equal(filter_device(x, CenterWeightedSpec("cwddf", 5)), filter_device(x, parse_filter_spec("ddf")))
