"""Synthetic test-signal generators -- TEST INFRASTRUCTURE ONLY.

Seeded stand-ins for the inputs BASELINE.json's configs describe (PM-QPSK,
28 GBd, 2 samples/symbol, i.i.d. uniform symbols, root-raised-cosine pulses,
forward propagation over an amplified link, AWGN at a given OSNR) plus a
minimal coherent receiver used to compare hard decisions between the GPU
product and this oracle.  The reference package has no RRC or OSNR
generator (its modem is PRBS + NRZ/RC, pkg/src/fiberdbp/modem.py:146-180),
so these follow the textbook formulas.  The forward link restates the
reference split-step solver (pkg/src/fiberdbp/channel.py:47-94, 174-207)
for noiseless, rotation-free links.
"""

from __future__ import annotations

import math

import numpy as np

from .dbp_port import LN10_OVER_10, bin_frequencies, effective_len

PLANCK = 6.62607015e-34
LIGHT = 299792458.0


def d_to_beta2(d_ps_nm_km: float, wavelength_nm: float = 1550.0) -> float:
    """Dispersion parameter D (ps/nm/km) -> beta2 (ps^2/km)."""
    lam = wavelength_nm * 1e-9
    beta2_s2_per_m = -d_ps_nm_km * 1e-6 * lam ** 2 / (2.0 * math.pi * LIGHT)
    return beta2_s2_per_m * 1e3 * 1e24


def rrc_response(n: int, sps: int, rolloff: float) -> np.ndarray:
    """Frequency response of a unit-energy root-raised-cosine pulse on an n-bin grid."""
    f = np.abs(bin_frequencies(n, float(sps)))          # in units of the symbol rate
    lo, hi = (1.0 - rolloff) / 2.0, (1.0 + rolloff) / 2.0
    h = np.zeros(n)
    h[f <= lo] = 1.0
    mid = (f > lo) & (f <= hi)
    h[mid] = np.sqrt(0.5 * (1.0 + np.cos(np.pi / rolloff * (f[mid] - lo))))
    return h


def qpsk_rrc(num_symbols: int, sps: int = 2, rolloff: float = 0.1, seed: int = 0,
             power_dbm: float = 0.0):
    """Dual-pol i.i.d. uniform QPSK with RRC pulses, circular, scaled to the launch power.

    Returns ``(samples (2, n) complex128, symbols (2, num_symbols) complex128)``.
    """
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2, size=(2, 2, num_symbols))
    symbols = ((1.0 - 2.0 * bits[:, 0]) + 1j * (1.0 - 2.0 * bits[:, 1])) / math.sqrt(2.0)
    n = num_symbols * sps
    up = np.zeros((2, n), dtype=np.complex128)
    up[:, ::sps] = symbols
    wave = np.fft.ifft(np.fft.fft(up, axis=1) * rrc_response(n, sps, rolloff), axis=1)
    p = np.mean(np.abs(wave[0]) ** 2 + np.abs(wave[1]) ** 2)
    wave *= math.sqrt(10.0 ** ((power_dbm - 30.0) / 10.0) / p)
    return wave, symbols


def forward_link(samples: np.ndarray, rate_hz: float, beta2: float, gamma: float,
                 alpha_db_per_km: float, span_km: float, num_spans: int,
                 steps_per_span: int) -> np.ndarray:
    """Noiseless forward SSFM over transparent amplified spans (channel.py:74-94, 174-207)."""
    n = samples.shape[1]
    f = bin_frequencies(n, rate_hz)
    alpha = LN10_OVER_10 * alpha_db_per_km
    dz = span_km / steps_per_span
    dz_eff = effective_len(alpha, dz) if alpha > 0.0 else dz
    lin = np.exp(1j * (-2.0 * np.pi ** 2 * (beta2 * 1e-24) * f ** 2 * dz))
    loss = math.exp(-alpha * dz / 2.0)
    gain = math.sqrt(10.0 ** (alpha_db_per_km * span_km / 10.0))
    cur = np.asarray(samples, dtype=np.complex128)
    for _ in range(num_spans):
        for _ in range(steps_per_span):
            cur = np.fft.ifft(np.fft.fft(cur, axis=1) * lin, axis=1)
            power = np.abs(cur[0]) ** 2 + np.abs(cur[1]) ** 2
            cur = cur * np.exp(-1j * gamma * dz_eff * power) * loss
        cur = cur * gain
    return cur


def add_awgn_osnr(samples: np.ndarray, rate_hz: float, osnr_db: float, seed: int,
                  ref_bw_hz: float = 12.5e9) -> np.ndarray:
    """Complex AWGN over the full sampled band for a given OSNR in ``ref_bw_hz``."""
    p_sig = np.mean(np.abs(samples[0]) ** 2 + np.abs(samples[1]) ** 2)
    n_ref = p_sig / 10.0 ** (osnr_db / 10.0)             # noise power (both pols) in ref_bw
    sigma2 = n_ref * rate_hz / ref_bw_hz / 2.0            # per polarisation, full band
    rng = np.random.default_rng(seed)
    noise = (rng.standard_normal(samples.shape) + 1j * rng.standard_normal(samples.shape))
    return samples + noise * math.sqrt(sigma2 / 2.0)


def receive_symbols(samples: np.ndarray, sps: int = 2, rolloff: float = 0.1) -> np.ndarray:
    """Matched RRC filter, symbol-centre sampling and a blind 4th-power phase fix."""
    n = samples.shape[1]
    mf = np.fft.ifft(np.fft.fft(samples, axis=1) * rrc_response(n, sps, rolloff), axis=1)
    sym = mf[:, ::sps]
    phase = np.angle(np.sum(sym ** 4, axis=1)) / 4.0 - np.pi / 4.0
    sym = sym * np.exp(-1j * phase)[:, None]
    return sym / np.sqrt(np.mean(np.abs(sym) ** 2, axis=1, keepdims=True))


def hard_decisions(sym: np.ndarray) -> np.ndarray:
    """Gray QPSK decisions, I and Q bits interleaved (modem.py:118-125 convention)."""
    bits = np.empty(sym.shape[:-1] + (2 * sym.shape[-1],), dtype=np.uint8)
    bits[..., 0::2] = sym.real < 0.0
    bits[..., 1::2] = sym.imag < 0.0
    return bits


def q_factor_db(bits: np.ndarray, ref_bits: np.ndarray) -> float:
    """Q = 20 log10(sqrt(2) erfcinv(2 BER)) (modem.py:409-412), inf when error-free."""
    from scipy.special import erfcinv
    ber = float(np.mean(bits != ref_bits))
    if ber == 0.0:
        return math.inf
    return 20.0 * math.log10(math.sqrt(2.0) * float(erfcinv(2.0 * ber)))


def gaussian_coeffs(n_coeffs: int, width: float = 5.0) -> np.ndarray:
    """A fixed, seeded-free ESSFM coefficient set: Gaussian taps with c0 + 2 sum c_i = 1."""
    i = np.arange(n_coeffs + 1, dtype=np.float64)
    c = np.exp(-0.5 * (i / width) ** 2)
    return c / (c[0] + 2.0 * np.sum(c[1:]))
