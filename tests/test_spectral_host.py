"""Host-side spectral transforms (spectral.py:85-211 semantics): boundary Fourier transform with the
doubled one-sided convention, aliasing guard, decay of a triangle wave, and the truncation-error
estimate -- the behaviours the reference checks in pkg/tests/test_spectral.py:37-123, restated
against this package (no GPU needed)."""

import numpy as np
import pytest

from paper_2009_06725_b200 import BoundaryWaveform, fit_loglog_slope, fourier_transform_bcs, reconstruct_signal
from paper_2009_06725_b200 import truncation_error


def wave(samples=None, coefficients=None, kind="neumann", patch="inlet", period=1.0):
    return BoundaryWaveform(patch=patch, kind=kind, direction=np.array([1.0, 0.0]), period=period,
                            samples=None if samples is None else np.asarray(samples, float),
                            coefficients=None if coefficients is None else np.asarray(coefficients, complex))


def sampled(f, n=256):
    return wave(samples=f(np.arange(n) / n))


def test_constant_and_cosine_coefficients():
    c = fourier_transform_bcs([sampled(lambda t: np.full_like(t, 3.0))], 4).coefficients["inlet"]
    assert abs(c[0] - 3.0) < 1e-13 and np.max(np.abs(c[1:])) < 1e-13
    c = fourier_transform_bcs([sampled(lambda t: np.cos(2 * np.pi * t))], 4).coefficients["inlet"]
    assert abs(c[1] - 1.0) < 1e-12          # one-sided coefficients carry the factor 2
    assert abs(c[0]) < 1e-13 and np.max(np.abs(c[2:])) < 1e-12


def test_band_limited_signal_round_trips():
    rng = np.random.default_rng(11)
    coeffs = np.concatenate([[rng.normal()], rng.normal(size=5) + 1j * rng.normal(size=5)])
    t = np.arange(128) / 128.0
    sig = reconstruct_signal(coeffs, 1.0, t)
    back = fourier_transform_bcs([wave(samples=sig)], 5).coefficients["inlet"]
    assert np.linalg.norm(reconstruct_signal(back, 1.0, t) - sig) <= 1e-10 * np.linalg.norm(sig)


def test_too_few_samples_for_the_requested_modes():
    with pytest.raises(ValueError, match="samples"):
        wave(samples=np.cos(2 * np.pi * np.arange(8) / 8)).mode_coefficients(4)


def test_triangle_wave_decays_as_inverse_square():
    t = np.arange(512) / 512.0
    c = np.abs(fourier_transform_bcs([wave(samples=1.0 - 4.0 * np.abs(t - 0.5))], 15).coefficients["inlet"])
    odd = np.arange(1, 16, 2)
    assert fit_loglog_slope(odd, c[odd]) == pytest.approx(-2.0, abs=0.05)


def test_truncation_error_limits():
    bl = wave(coefficients=[0.5, 1.0, 0.25 + 0.1j])
    assert truncation_error([bl], fourier_transform_bcs([bl], 4)) == pytest.approx(0.0, abs=1e-12)
    cos = sampled(lambda t: np.cos(2 * np.pi * t))
    assert truncation_error([cos], fourier_transform_bcs([cos], 0)) == pytest.approx(1.0, abs=1e-10)


def test_truncation_error_of_a_square_wave_equals_the_time_domain_defect():
    n = 4096
    t = np.arange(n) / n
    sq = np.where(t < 0.5, 1.0, -1.0)
    w = wave(samples=sq)
    for m in (1, 3, 5):
        ms = fourier_transform_bcs([w], m)
        defect = sq - reconstruct_signal(ms.coefficients["inlet"], 1.0, t)
        direct = np.sqrt(np.mean(defect ** 2) / np.mean(sq ** 2))
        assert truncation_error([w], ms) == pytest.approx(direct, rel=1e-12)


def test_truncation_error_all_zero_data_warns():
    w = wave(coefficients=[0.0, 0.0])
    with pytest.warns(UserWarning, match="zero"):
        assert truncation_error([w], fourier_transform_bcs([w], 1)) == 0.0


def test_truncation_error_sums_per_kind_ratios():
    h = wave(coefficients=[0.0, 1.0, 0.5], kind="neumann", patch="inlet")
    g = wave(coefficients=[0.0, 2.0], kind="dirichlet", patch="lid")
    ms = fourier_transform_bcs([h, g], 1)
    # Neumann tail 0.25 of energy 1.25; the Dirichlet waveform is exactly represented
    assert truncation_error([h, g], ms) == pytest.approx(np.sqrt(0.25 / 1.25), rel=1e-12)
