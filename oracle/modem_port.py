"""CPU restatement of the reference transmitter -- TEST INFRASTRUCTURE ONLY.

Follows pkg/src/fiberdbp/modem.py: ``generate_prbs`` (:90-107), ``qpsk_map``
(:110-113), ``_raised_cosine_taps`` (:136-143), ``modulate_pm_qpsk``
(:146-180), plus ``scale_to_power`` / ``signal_power`` (sigkit.py:215-226)
and ``apply_laser_phase_noise`` (channel.py:156-171).  Pinned by
tests/test_oracle_golden.py to tests/golden/golden_rx_v1.npz; the GPU
tests use it to build the reference's own test waveforms (PRBS NRZ / RC
PM-QPSK) and the ber-sweep scenario of cli.py:599-615.
"""

from __future__ import annotations

import math

import numpy as np

PRBS_TAPS = {7: 6, 9: 5, 11: 9, 15: 14, 23: 18}
SQRT1_2 = 1.0 / math.sqrt(2.0)


def generate_prbs(order: int, seed_state: int) -> np.ndarray:
    """Fibonacci LFSR, x^order + x^tap + 1, period 2^order - 1 (modem.py:90-107)."""
    tap = PRBS_TAPS[order]
    state = int(seed_state) & ((1 << order) - 1)
    if state == 0:
        raise ValueError("seed_state must be nonzero modulo 2^order")
    n = (1 << order) - 1
    bits = np.empty(n, dtype=np.uint8)
    for k in range(n):
        new = (state ^ (state >> (order - tap))) & 1
        bits[k] = new
        state = (state >> 1) | (new << (order - 1))
    return bits


def qpsk_map(bits_i, bits_q):
    return ((1.0 - 2.0 * np.asarray(bits_i)) + 1j * (1.0 - 2.0 * np.asarray(bits_q))) * SQRT1_2


def raised_cosine_taps(sps: int, rolloff: float, half_span_symbols: int = 8) -> np.ndarray:
    t = np.arange(-half_span_symbols * sps, half_span_symbols * sps + 1) / sps
    h = np.sinc(t) * np.cos(np.pi * rolloff * t)
    den = 1.0 - (2.0 * rolloff * t) ** 2
    sing = np.isclose(den, 0.0)
    h[~sing] /= den[~sing]
    h[sing] = np.pi / 4.0 * np.sinc(1.0 / (2.0 * rolloff))
    return h


def modulate_pm_qpsk(num_symbols: int, rng_seed: int, sps: int = 2, pulse: str = "nrz", rolloff: float = 0.2,
                     prbs_order: int = 11):
    """(2, num_symbols * sps) waveform and (2, num_symbols) reference symbols (modem.py:146-180)."""
    period = (1 << prbs_order) - 1
    seed_state = int(np.random.default_rng(rng_seed).integers(1, period + 1))
    base = generate_prbs(prbs_order, seed_state)
    offsets = (0, period // 4, period // 2, (3 * period) // 4)
    rails = [np.resize(np.roll(base, -off), num_symbols) for off in offsets]
    ref = np.stack([qpsk_map(rails[0].astype(np.float64), rails[1].astype(np.float64)),
                    qpsk_map(rails[2].astype(np.float64), rails[3].astype(np.float64))])
    if pulse == "nrz":
        wave = np.repeat(ref, sps, axis=1)
    else:
        up = np.zeros((2, num_symbols * sps), dtype=np.complex128)
        up[:, ::sps] = ref
        taps = raised_cosine_taps(sps, rolloff)
        n = up.shape[1]
        kernel = np.zeros(n)
        half = taps.size // 2
        np.add.at(kernel, (np.arange(taps.size) - half) % n, taps)
        wave = np.fft.ifft(np.fft.fft(up, axis=1) * np.fft.fft(kernel), axis=1)
    return wave, ref


def signal_power(x) -> float:
    return float(np.mean(np.abs(x[0]) ** 2 + np.abs(x[1]) ** 2))


def scale_to_power(x, target_dbm: float):
    p = signal_power(x)
    return x * math.sqrt(10.0 ** ((target_dbm - 30.0) / 10.0) / p)


def laser_phase_noise(x, linewidth_hz: float, sample_rate: float, rng=None):
    """Common Wiener phase noise, increment variance 2 pi linewidth / fs (channel.py:156-171)."""
    if linewidth_hz == 0.0:
        return x
    gen = rng if isinstance(rng, np.random.Generator) else np.random.default_rng(rng)
    sigma = np.sqrt(2.0 * np.pi * linewidth_hz / sample_rate)
    phi = np.cumsum(gen.normal(scale=sigma, size=x.shape[1]))
    return x * np.exp(1j * phi)[None]
