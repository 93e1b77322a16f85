"""GPU: the calibration sampler (dfg_calib_samples) reproduces the
reference's PCG64 draws -- B bit for bit, A within 4 ulp (device arccos) --
and fit_angular_chromaticity matches the reference's fitted lines
(calibration.py:116-125) within 1e-11 relative (device reduction order)."""

import numpy as np
import pytest

import oracle
from paper_1009_0958_b200 import calibration

pytestmark = pytest.mark.gpu


def test_samples_match_reference(cuda, golden_full):
    data, _ = golden_full
    for n, seed, p, kb, ka in ((2000, 7, 2.0, "calib_b", "calib_a"), (1500, 8, 3.0, "calib_b_p3", "calib_a_p3")):
        b, a = calibration.sample_angle_chromaticity_pairs(n, seed, p)
        b, a = b.cpu().numpy(), a.cpu().numpy()
        if p == 2.0:
            assert (b == data[kb]).all()
        else:
            assert np.allclose(b, data[kb], rtol=4e-16, atol=0)  # pow: <= 2 ulp
        assert np.allclose(a, data[ka], rtol=0, atol=4 * np.spacing(np.pi / 2))


def test_fits_match_reference(cuda, golden_full):
    data, man = golden_full
    for (n, seed, p, method), want in zip(man["calib_cases"], data["calib_fits"]):
        f = calibration.fit_angular_chromaticity(n, seed, p, method)
        got = [f.slope, f.intercept, f.fit_error, f.mean_abs_residual, f.rms_orthogonal]
        assert np.allclose(got, want, rtol=1e-11, atol=0), (n, seed, p, method, got, want)
        assert f.sample_count == n and f.method == method


def test_large_draw_against_oracle_and_fit_line(cuda):
    """10^7 pairs: the streamed three-pass device fit equals the oracle fit
    of the numpy samples and fit_line over the device samples."""
    n, seed = 10**7, 11
    f = calibration.fit_angular_chromaticity(n, seed)
    want = oracle.calib_fit(*oracle.calib_samples(n, seed))
    got = [f.slope, f.intercept, f.fit_error, f.mean_abs_residual, f.rms_orthogonal]
    assert np.allclose(got, want, rtol=1e-10, atol=0), (got, want)
    b, a = calibration.sample_angle_chromaticity_pairs(n, seed)
    g = calibration.fit_line(b, a)
    assert np.allclose([g.slope, g.intercept, g.fit_error], got[:3], rtol=1e-10, atol=0)


def test_validation(cuda):
    with pytest.raises(ValueError):
        calibration.fit_angular_chromaticity(999)
    with pytest.raises(ValueError):
        calibration.fit_angular_chromaticity(10**4, method="lad")
    with pytest.raises(ValueError):
        calibration.fit_angular_chromaticity(10**4, p=0.5)
    with pytest.raises(ValueError):
        calibration.fit_line(np.ones(10), np.arange(10.0))  # no variance in B
