"""Time-periodic boundary data and its one-sided Fourier modes (host side).

Behaviour of the reference's ``BoundaryWaveform`` (spectral.py:28-130), ``reconstruct_signal``
(133-138), ``ModeSet`` (141-191), ``fourier_transform_bcs`` (194-211) and ``truncation_error``
(214-240): same fields, validation messages, the one-sided factor-2 convention
(``ONE_SIDED_FACTOR``, spectral.py:25,98-100) and omega_n = 2 pi n / T.  These are O(modes x
samples) host computations that feed the device solve; when the reference package itself is
installed, :mod:`.dropin` uses its classes instead.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np

ONE_SIDED_FACTOR = 2.0
WAVEFORM_KINDS = ("dirichlet", "neumann")

__all__ = ["ONE_SIDED_FACTOR", "BoundaryWaveform", "ModeSet", "reconstruct_signal", "fourier_transform_bcs",
           "truncation_error"]


# -- spectra of a periodic scalar signal ----------------------------------------------------------

def _phase_matrix(t, n_coeffs, period):
    """exp(2 pi i t_j n / T) for every time t_j and mode n < n_coeffs."""
    return np.exp(1j * 2.0 * np.pi * np.outer(t, np.arange(n_coeffs)) / period)


def reconstruct_signal(coefficients, period, t):
    """u(t) = Re sum_n c_n exp(i omega_n t) for one-sided coefficients (spectral.py:133-138)."""
    t = np.asarray(t, dtype=float)
    c = np.asarray(coefficients, dtype=complex)
    return np.real(_phase_matrix(t, len(c), period) @ c).reshape(t.shape)


def _sampled_spectrum(samples, n_modes, patch):
    """One-sided DFT coefficients 0..n_modes of uniform samples over one period."""
    n = samples.size
    need = 2 * (n_modes + 1)
    if n < need:
        raise ValueError(f"waveform '{patch}' has {n} samples; at least {need} are needed to resolve "
                         f"{n_modes} modes")
    spec = (np.fft.rfft(samples) / n)[: n_modes + 1].astype(complex)
    spec[1:] *= ONE_SIDED_FACTOR
    return spec


def _truncated(coefficients, n_modes):
    out = np.zeros(n_modes + 1, dtype=complex)
    keep = min(n_modes + 1, coefficients.size)
    out[:keep] = coefficients[:keep]
    return out


def _coefficient_energy(c, period, n_modes):
    """Time integral of |signal|^2 (n_modes None) or of its tail beyond n_modes, by Parseval."""
    mag2 = np.abs(c) ** 2
    if n_modes is None:
        return float(period * (mag2[0] + 0.5 * mag2[1:].sum()))
    return float(0.5 * period * mag2[n_modes + 1:].sum())


@dataclass
class BoundaryWaveform:
    """A periodic scalar signal on one patch times a fixed direction (spectral.py:28-130).

    Give exactly one of ``samples`` (uniform over one period, endpoint excluded) or
    ``coefficients`` (one-sided, already carrying the factor-2 convention).
    """

    patch: str
    kind: str
    direction: np.ndarray
    period: float
    samples: np.ndarray | None = None
    coefficients: np.ndarray | None = None
    area: float = 1.0

    def __post_init__(self):
        if self.kind not in WAVEFORM_KINDS:
            raise ValueError(f"waveform kind must be dirichlet or neumann, got '{self.kind}'")
        if self.period <= 0:
            raise ValueError("period must be positive")
        self.direction = np.asarray(self.direction, dtype=float)
        has_samples, has_coeffs = self.samples is not None, self.coefficients is not None
        if has_samples == has_coeffs:
            raise ValueError("provide exactly one of samples or coefficients")
        if has_coeffs:
            self.coefficients = np.asarray(self.coefficients, dtype=complex)
            return
        self.samples = np.asarray(self.samples, dtype=float)
        if self.samples.size < 2:
            raise ValueError("sampled waveform needs at least 2 samples")

    @classmethod
    def from_samples(cls, patch, kind, direction, times, values, area=1.0):
        """From (t, value) pairs; a closed sampling (last value = first) drops the repeated endpoint."""
        times = np.asarray(times, dtype=float)
        values = np.asarray(values, dtype=float)
        if times.ndim != 1 or times.shape != values.shape or times.size < 2:
            raise ValueError("need matching 1D time and value arrays")
        steps = np.diff(times)
        if np.any(np.abs(steps - steps[0]) > 1e-9 * abs(steps[0])):
            raise ValueError("waveform samples must be uniformly spaced")
        closed = values[-1] == values[0]
        period = times[-1] - times[0] if closed else times[-1] + steps[0] - times[0]
        return cls(patch=patch, kind=kind, direction=direction, period=period,
                   samples=values[:-1] if closed else values, area=area)

    def max_modes(self) -> int:
        """Largest resolvable mode index (aliasing guard for sampled signals)."""
        return self.samples.size // 2 - 1 if self.samples is not None else self.coefficients.size - 1

    def mode_coefficients(self, n_modes: int) -> np.ndarray:
        """One-sided coefficients of modes 0..n_modes (spectral.py:85-101)."""
        if self.samples is None:
            return _truncated(self.coefficients, n_modes)
        return _sampled_spectrum(self.samples, n_modes, self.patch)

    def evaluate(self, t):
        """Signal value at time(s) ``t``: the mode sum, or periodic linear interpolation of the samples."""
        t = np.asarray(t, dtype=float)
        if self.samples is None:
            return reconstruct_signal(self.coefficients, self.period, t)
        n = self.samples.size
        knots = np.linspace(0.0, self.period, n + 1)
        return np.interp(np.mod(t, self.period), knots, np.concatenate([self.samples, self.samples[:1]]))

    def signal_norm_sq(self, n_modes: int | None = None) -> float:
        """Integral over one period of |signal|^2 (n_modes None) or of |signal - truncation|^2."""
        if self.samples is None:
            return _coefficient_energy(self.coefficients, self.period, n_modes)
        if n_modes is None:
            return float(np.mean(self.samples ** 2) * self.period)
        t = np.arange(self.samples.size) * self.period / self.samples.size
        residual = self.samples - reconstruct_signal(self.mode_coefficients(n_modes), self.period, t)
        return float(np.mean(residual ** 2) * self.period)


@dataclass
class ModeSet:
    """Modes 0..N_m: frequencies and per-patch complex coefficients (spectral.py:141-191)."""

    indices: np.ndarray
    frequencies: np.ndarray
    period: float
    coefficients: dict
    waveforms: list = field(default_factory=list)

    @property
    def n_modes(self) -> int:
        return int(np.max(self.indices))

    def patch_kind(self, patch: str) -> str:
        kinds = {wf.patch: wf.kind for wf in reversed(self.waveforms)}
        if patch not in kinds:
            raise KeyError(patch)
        return kinds[patch]

    def _with_coefficients(self, coefficients):
        return ModeSet(indices=self.indices, frequencies=self.frequencies, period=self.period,
                       coefficients=coefficients, waveforms=self.waveforms)

    def scaled(self, alpha: complex) -> "ModeSet":
        return self._with_coefficients({p: alpha * c for p, c in self.coefficients.items()})

    def thresholded(self, relative_amplitude: float) -> "ModeSet":
        """Zero every mode whose amplitude is below ``relative_amplitude`` x the largest on all patches
        (a mode survives if it reaches the threshold on any patch)."""
        keep = np.zeros(len(self.indices), dtype=bool)
        for c in self.coefficients.values():
            mag = np.abs(c)
            if mag.max() > 0:
                keep |= mag >= relative_amplitude * mag.max()
        return self._with_coefficients({p: np.where(keep, c, 0.0) for p, c in self.coefficients.items()})


def fourier_transform_bcs(waveforms, n_modes: int) -> ModeSet:
    """Coefficients of every boundary signal for modes 0..n_modes, omega_n = 2 pi n / T (spectral.py:194-211)."""
    waveforms = list(waveforms)
    if not waveforms:
        raise ValueError("no boundary waveforms given")
    period = waveforms[0].period
    if any(abs(wf.period - period) > 1e-12 * period for wf in waveforms):
        raise ValueError("all waveforms must share one period")
    idx = np.arange(n_modes + 1)
    return ModeSet(indices=idx, frequencies=2.0 * np.pi * idx / period, period=period,
                   coefficients={wf.patch: wf.mode_coefficients(n_modes) for wf in waveforms}, waveforms=waveforms)


def truncation_error(waveforms, mode_set: ModeSet) -> float:
    """A-priori truncation estimate sqrt(sum over kinds of tail energy / total energy), patches
    weighted by area x |direction|^2; kinds without data are skipped (spectral.py:214-240)."""
    n_modes = mode_set.n_modes
    ratio_sum, seen = 0.0, False
    for kind in ("neumann", "dirichlet"):
        group = [wf for wf in waveforms if wf.kind == kind]
        weights = [wf.area * float(np.dot(wf.direction, wf.direction)) for wf in group]
        total = sum(w * wf.signal_norm_sq() for w, wf in zip(weights, group))
        tail = sum(w * wf.signal_norm_sq(n_modes) for w, wf in zip(weights, group))
        if total > 0.0:
            seen = True
            ratio_sum += tail / total
    if not seen:
        warnings.warn("truncation_error: all boundary signals are zero; e_M defined as 0")
        return 0.0
    return float(np.sqrt(ratio_sum))
