"""CPU restatement of the reference forward channel -- TEST/MEASUREMENT INFRASTRUCTURE ONLY.

Follows pkg/src/fiberdbp/channel.py: the split-step span (:74-94), the ASE
amplifier (:97-128), the Haar unitary (:131-138) and the link loop with its
seeded child streams (:174-207), on (2, n) complex128 arrays.  Pinned by
tests/test_oracle_golden.py to tests/golden/golden_fwd_v1.npz (made by the
reference itself, tests/golden/make_golden_forward.py); used as the checker
of the GPU simulator at sizes above the fixtures and as its CPU baseline.
"""

from __future__ import annotations

import math

import numpy as np

from .dbp_port import LN10_OVER_10, bin_frequencies, effective_len

PLANCK = 6.62607015e-34
LIGHT = 299792458.0


def _gen(rng):
    return rng if isinstance(rng, np.random.Generator) else np.random.default_rng(rng)


def span(x, rate_hz, beta2, gamma, alpha_db_per_km, length_km, steps, nonlinear=True):
    """channel.py:74-94 (dispersion, rotation weighted by the step effective length, loss)."""
    n = x.shape[1]
    f = bin_frequencies(n, rate_hz)
    alpha = LN10_OVER_10 * alpha_db_per_km
    dz = length_km / steps
    dz_eff = effective_len(alpha, dz) if alpha > 0.0 else dz
    lin = np.exp(1j * (-2.0 * np.pi ** 2 * (beta2 * 1e-24) * f ** 2 * dz))
    loss = np.exp(-alpha * dz / 2.0)
    cur = np.asarray(x, dtype=np.complex128)
    for _ in range(steps):
        cur = np.fft.ifft(np.fft.fft(cur, axis=1) * lin, axis=1)
        if nonlinear:
            cur = cur * np.exp(-1j * gamma * dz_eff * (np.abs(cur[0]) ** 2 + np.abs(cur[1]) ** 2))
        cur = cur * loss
    return cur


def ase_noise(n, rate_hz, gain_db, nf_db, wavelength_nm, rng):
    """The (2, n) complex ASE draw of channel.py:112-125."""
    g_lin = 10.0 ** (gain_db / 10.0)
    f_lin = 10.0 ** (nf_db / 10.0)
    var = (g_lin - 1.0) * f_lin * PLANCK * (LIGHT / (wavelength_nm * 1e-9)) / 2.0 * rate_hz
    z = _gen(rng).normal(scale=np.sqrt(var / 2.0), size=(2, 2, n))
    return z[:, 0] + 1j * z[:, 1]


def amplify(x, rate_hz, gain_db, nf_db, wavelength_nm=1550.0, rng=None):
    """channel.py:97-128."""
    if gain_db < 0.0:
        raise ValueError("gain_db must be non-negative")
    out = np.asarray(x, dtype=np.complex128) * 10.0 ** (gain_db / 20.0)
    if nf_db is not None:
        out = out + ase_noise(x.shape[1], rate_hz, gain_db, nf_db, wavelength_nm, rng)
    return out


def haar(rng=None):
    """channel.py:131-138."""
    g = _gen(rng)
    z = g.normal(size=(2, 2)) + 1j * g.normal(size=(2, 2))
    q, r = np.linalg.qr(z)
    d = np.diagonal(r)
    return q * (d / np.abs(d))


def link(x, rate_hz, beta2, gamma, alpha_db_per_km, length_km, num_spans, steps, amp_gain_db=None,
         nf_db=5.0, pol_rotation=True, wavelength_nm=1550.0, rng=None, nonlinear=True):
    """channel.py:174-207: span, amplifier, optional rotation; children[2s], [2s+1]."""
    if isinstance(rng, np.random.Generator):
        raise ValueError("pass an integer seed or SeedSequence, not a Generator")
    ss = rng if isinstance(rng, np.random.SeedSequence) else np.random.SeedSequence(rng)
    children = ss.spawn(2 * num_spans)
    gain_db = alpha_db_per_km * length_km if amp_gain_db is None else amp_gain_db
    cur = np.asarray(x, dtype=np.complex128)
    for s in range(num_spans):
        cur = span(cur, rate_hz, beta2, gamma, alpha_db_per_km, length_km, steps, nonlinear)
        cur = amplify(cur, rate_hz, gain_db, nf_db, wavelength_nm, children[2 * s])
        if pol_rotation:
            cur = haar(children[2 * s + 1]) @ cur
    return cur
