"""GPU parity for window sides above 7 (the float64 direct kernel,
csrc/dfg_wide.cu): reference-generated fixtures, the oracle on larger seeded
images, strips / batches / the host path, and the side limit."""

import numpy as np
import pytest

import oracle
from paper_1009_0958_b200 import (
    REFLECT, REPLICATE, RasterImage, apply_filter, filter_batch_device, filter_device, filter_host,
    filter_rows_device, parse_filter_spec, synth,
)

pytestmark = pytest.mark.gpu


def test_reference_fixtures_bit_exact(cuda, golden_wide):
    data, cases = golden_wide
    bad = []
    for i, c in enumerate(cases):
        img = RasterImage(data[f"in{i}"].astype(np.float64))
        out = apply_filter(img, parse_filter_spec(c["spec"]), REPLICATE if c["border"] == "replicate" else REFLECT)
        if not (out.pixels == data[f"out{i}"]).all():
            bad.append((i, c, int((out.pixels != data[f"out{i}"]).any(-1).sum())))
    assert not bad, bad[:10]


@pytest.mark.parametrize("spec", ["bvdf:exact:window=9", "ddf:exact:window=9", "acwddf:exact:window=9", "ddf:minimax:window=11",
                                  "acwddf:rgb:window=9", "vmf:window=9:p=3", "ddf:exact:window=15"])
@pytest.mark.parametrize("border", ["replicate", "reflect"])
def test_against_oracle(cuda, spec, border):
    torch = cuda
    sp = parse_filter_spec(spec)
    img = synth.noisy_image(45, 52, 11, ("correlated", 0.2))
    img[5:9, 7:12] = 0  # zero vectors
    got = filter_device(torch.from_numpy(img).cuda(), sp, border).cpu().numpy()
    want = oracle.filter_image(img, sp, border)
    assert (got == want).all(), int((got != want).any(-1).sum())


def test_strips_batch_and_host_path(cuda):
    torch = cuda
    sp = parse_filter_spec("ddf:exact:window=9")
    img = synth.noisy_image(40, 37, 12, ("uncorrelated", 0.15))
    x = torch.from_numpy(img).cuda()
    whole = filter_device(x, sp).cpu().numpy()
    assert (whole == oracle.filter_image(img, sp)).all()
    # a strip holding its 4-row halo reproduces the rows of the whole image
    strip = filter_rows_device(x[6:30], 40, 6, 10, 16, sp).cpu().numpy()
    assert (strip == whole[10:26]).all()
    frames = np.stack([img, img[::-1].copy()])
    got = filter_batch_device(torch.from_numpy(frames).cuda(), sp).cpu().numpy()
    assert (got[0] == whole).all() and (got[1] == oracle.filter_image(frames[1], sp)).all()
    assert (filter_host(img, sp) == whole).all()


def test_selection_property_and_limit(cuda):
    torch = cuda
    img = synth.noisy_image(33, 29, 13, ("correlated", 0.3))
    out = filter_device(torch.from_numpy(img).cuda(), parse_filter_spec("bvdf:rgb:window=31")).cpu().numpy()
    pad = np.pad(img, ((15, 15), (15, 15), (0, 0)), mode="edge")
    for (r, c) in ((0, 0), (16, 14), (32, 28)):
        win = pad[r:r + 31, c:c + 31].reshape(-1, 3)
        assert (win == out[r, c]).all(-1).any()
    with pytest.raises(NotImplementedError):
        filter_device(torch.from_numpy(img).cuda(), parse_filter_spec("bvdf:rgb:window=33"))
