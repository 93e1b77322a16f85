"""GPU: the on-device noise simulator (dfg_corrupt_image) is bit-exact with
the reference's corrupt_image (noise.py:85-116) and the device metrics
reduction (dfg_image_metrics) matches the reference's compare()
(metrics.py:64-118) within 1e-12 relative (float64 sums, different order)."""

import math

import numpy as np
import pytest

import oracle
from paper_1009_0958_b200 import noise, metrics, synth

pytestmark = pytest.mark.gpu

REL = 1e-12  # metrics tolerance: float64 sums in a different order


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_noise_matches_reference_fixtures(cuda, golden_full):
    torch = cuda
    data, man = golden_full
    for c in man["noise_cases"]:
        kw = {k: v for k, v in c.items() if k != "name"}
        got = noise.corrupt_device(_dev(torch, data[f"noise_{c['name']}_in"]), noise.NoiseParams(**kw))
        assert (got.cpu().numpy() == data[f"noise_{c['name']}_out"]).all(), c["name"]
    got = noise.corrupt_device(_dev(torch, data["noise_clean"]),
                               noise.NoiseParams(0.2, 0.0, 0.0, 0.0, "uniform", 3 + 10**6))
    assert (got.cpu().numpy() == data["noise_ref"]).all()


@pytest.mark.parametrize("H,W,kw", [
    (1, 1, dict(phi=1.0, seed=1)),
    (1, 17, dict(phi=0.7, impulse="uniform", seed=2)),
    (333, 517, dict(seed=99)),
    (1080, 1920, dict(phi=0.3, phi1=0.1, phi2=0.1, phi3=0.1, impulse="uniform", seed=2**40 + 3)),
    (2048, 3001, dict(phi=0.05, phi1=0.0, phi2=0.5, phi3=0.5, seed=11)),
])
def test_noise_matches_oracle_at_size(cuda, H, W, kw):
    """Jump-ahead across millions of draws stays on numpy's stream."""
    torch = cuda
    img = synth.clean_image(H, W, 5)
    got = noise.corrupt_device(_dev(torch, img), noise.NoiseParams(**kw)).cpu().numpy()
    assert (got == oracle.corrupt(img, **kw)).all()


def test_noise_in_place_padded_and_api(cuda):
    torch = cuda
    img = synth.clean_image(64, 50, 9)
    p = noise.NoiseParams(phi=0.4, seed=77)
    want = oracle.corrupt(img, phi=0.4, seed=77)
    buf = torch.zeros((64, 64, 3), dtype=torch.uint8, device="cuda")
    view = buf[:, :50]
    view.copy_(_dev(torch, img))
    noise.corrupt_device(view, p, out=view)  # in place on a padded-pitch view
    assert (view.cpu().numpy() == want).all()
    assert (buf[:, 50:] == 0).all()
    r = noise.corrupt_image(img.astype(np.float64), p)
    assert r.pixels.dtype == np.float64 and (r.pixels == want).all()
    with pytest.raises(ValueError):
        noise.NoiseParams(phi=2.0)
    with pytest.raises(ValueError):
        noise.NoiseParams(impulse="gaussian")


def _close(g, w):
    if math.isinf(w):
        return math.isinf(g)
    return abs(g - w) <= REL * max(1.0, abs(w))


def test_metrics_match_reference_fixtures(cuda, golden_full):
    torch = cuda
    data, man = golden_full
    for (a, b), want in zip(man["metrics_pairs"], data["metrics_ref"]):
        got = metrics.metrics_device(_dev(torch, data[a]), _dev(torch, data[b]))
        assert all(_close(g, w) for g, w in zip(got, want)), (a, b, got, want)
        rep = metrics.compare(data[a].astype(np.float64), data[b].astype(np.float64), 1.5)
        assert _close(rep.mae, want[0]) and _close(rep.psnr, want[1]) and _close(rep.ncd_x1000, want[2])
        assert rep.time_seconds == 1.5


@pytest.mark.parametrize("H,W", [(1, 1), (7, 3), (1080, 1920), (4096, 4096)])
def test_metrics_match_oracle_at_size(cuda, H, W):
    torch = cuda
    clean = synth.clean_image(H, W, 3)
    noisy = synth.add_uncorrelated_noise(clean, 0.2, 4)
    got = metrics.metrics_device(_dev(torch, clean), _dev(torch, noisy))
    want = oracle.metrics(clean, noisy)
    assert all(_close(g, w) for g, w in zip(got, want)), (got, want)


def test_metrics_edge_cases(cuda):
    torch = cuda
    black = np.zeros((5, 6, 3), np.uint8)
    white = np.full((5, 6, 3), 255, np.uint8)
    assert metrics.metrics_device(_dev(torch, black), _dev(torch, black)) == (0.0, math.inf, 0.0)
    m, p, n = metrics.metrics_device(_dev(torch, black), _dev(torch, white))
    assert m == 255.0 and p == 0.0 and math.isinf(n)  # reference luv == 0 -> inf NCD
    assert _close(n, math.inf)
    with pytest.raises(ValueError):
        metrics.metrics_device(_dev(torch, black), _dev(torch, np.zeros((5, 7, 3), np.uint8)))
