"""Seeded synthetic spectral states for the BASELINE configs.

Host-side input generation only (numpy); nothing here is on the GPU hot
path.  The recipe is a variant of the reference test fixture
`random_coeffs` (/root/reference/pkg/tests/conftest.py:20-30) with the
amplitude envelope (s+1)^-1.5 and an area-weighted grid-rms rescale that
follows from Parseval (reference test_spharm.py:176-184) and
GaussianGrid.quad_mean (spharm.py:116-118).
"""

from __future__ import annotations

import numpy as np

# rms targets per prognostic variable (phi_prime m^2/s^2, zeta 1/s, delta 1/s)
RMS_TARGETS = (1.0e3, 1.0e-5, 1.0e-6)

# Physical constants of every BASELINE config (BASELINE.json configs[0]);
# nu is the reference default (testcases.py:49, cli.py:116).
EARTH = dict(radius=6.37122e6, omega=7.292e-5, gravity=9.80616, nu=1.0e5, h_bar=1.0e4)


def spectral_noise(rng: np.random.Generator, R: int, target_rms: float,
                   zero_mean: bool) -> np.ndarray:
    """One (R+1, R+1) complex128 field: Gaussian coefficients times
    (s+1)^-1.5, r=0 row real, optional zero mean, rescaled to the target
    area-weighted grid rms sqrt(sum mult_r |c_rs|^2 / 2)."""
    c = np.zeros((R + 1, R + 1), dtype=complex)
    s = np.arange(R + 1, dtype=float)
    for r in range(R + 1):
        n = R + 1 - r
        re = rng.normal(size=n)
        im = rng.normal(size=n)
        c[r, r:] = (re + 1j * im) * (s[r:] + 1.0) ** -1.5
    c[0] = c[0].real
    if zero_mean:
        c[0, 0] = 0.0
    mult = np.full((R + 1, 1), 2.0)
    mult[0] = 1.0
    rms = np.sqrt(np.sum(mult * np.abs(c) ** 2) / 2.0)
    if rms > 0:
        c *= target_rms / rms
    return c


def seeded_state(R: int, seed: int) -> np.ndarray:
    """(3, R+1, R+1) state (phi_prime, zeta, delta) from one seed, drawn in
    that field order; zeta and delta have a zero n=0 mode."""
    rng = np.random.default_rng(seed)
    return np.stack([
        spectral_noise(rng, R, RMS_TARGETS[0], False),
        spectral_noise(rng, R, RMS_TARGETS[1], True),
        spectral_noise(rng, R, RMS_TARGETS[2], True),
    ])


def transform_batch(R: int, n_fields: int = 15) -> np.ndarray:
    """Config-1 batch: field i is variable i % 3 of node i // 3, drawn from
    its own seed i with that variable's rms target."""
    out = np.empty((n_fields, R + 1, R + 1), dtype=complex)
    for i in range(n_fields):
        v = i % 3
        out[i] = spectral_noise(np.random.default_rng(i), R, RMS_TARGETS[v], v != 0)
    return out


def ensemble_states(R: int, members: int) -> np.ndarray:
    """Config-4 ensemble: member k uses seed k."""
    return np.stack([seeded_state(R, k) for k in range(members)])
