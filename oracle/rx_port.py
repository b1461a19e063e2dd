"""CPU restatement of the reference receiver DSP -- TEST/MEASUREMENT INFRASTRUCTURE ONLY.

Follows pkg/src/fiberdbp/modem.py: the CMA butterfly (``_cma_pass`` :183-204,
``butterfly_equalize`` :207-271), carrier recovery (``_vv_phase`` :274-280,
``carrier_recover`` :283-351), decisions (:116-125) and ``measure_ber``
(:358-413), on float64 numpy arrays.  The CMA loop is jitted with numba when
it is importable (as the reference does), else runs as plain Python.
Pinned by tests/test_oracle_golden.py to tests/golden/golden_rx_v1.npz;
used as the checker of the GPU receiver and as its CPU baseline.
"""

from __future__ import annotations

import math

import numpy as np

SQRT1_2 = 1.0 / math.sqrt(2.0)


def _cma_sweep(ext_x, ext_y, taps, mu, n_sym, hxx, hxy, hyx, hyy, out_x, out_y):
    for n in range(n_sym):
        b = 2 * n
        ox = 0.0 + 0.0j
        oy = 0.0 + 0.0j
        for i in range(taps):
            ox += hxx[i] * ext_x[b + i] + hxy[i] * ext_y[b + i]
            oy += hyx[i] * ext_x[b + i] + hyy[i] * ext_y[b + i]
        ex = mu * (1.0 - (ox.real * ox.real + ox.imag * ox.imag)) * ox
        ey = mu * (1.0 - (oy.real * oy.real + oy.imag * oy.imag)) * oy
        for i in range(taps):
            cx = np.conj(ext_x[b + i])
            cy = np.conj(ext_y[b + i])
            hxx[i] += ex * cx
            hxy[i] += ex * cy
            hyx[i] += ey * cx
            hyy[i] += ey * cy
        out_x[n] = ox
        out_y[n] = oy


try:  # the reference jits the same loop with numba (modem.py:183)
    from numba import njit
    _cma_sweep = njit(cache=False)(_cma_sweep)
    JITTED = True
except Exception:  # pragma: no cover
    JITTED = False


def equalize(x, taps=15, mu=1e-3, passes=2):
    """(2, 2m) -> ((2, m) symbols, reinits, (hxx, hxy, hyx, hyy)) -- modem.py:230-271."""
    x = np.asarray(x, dtype=np.complex128)
    n = x.shape[1]
    m = n // 2
    p = np.mean(np.abs(x[0]) ** 2 + np.abs(x[1]) ** 2) / 2.0
    g = 1.0 / math.sqrt(p)
    half = taps // 2
    idx = np.arange(-half, n + half) % n
    ex = np.ascontiguousarray(x[0][idx] * g)
    ey = np.ascontiguousarray(x[1][idx] * g)
    h = [np.zeros(taps, dtype=np.complex128) for _ in range(4)]
    h[0][half] = 1.0
    h[3][half] = 1.0
    ox = np.empty(m, dtype=np.complex128)
    oy = np.empty(m, dtype=np.complex128)
    reinits = 0
    for _ in range(passes):
        _cma_sweep(ex, ey, taps, mu, m, h[0], h[1], h[2], h[3], ox, oy)
        num = np.abs(np.vdot(ox, oy))
        den = math.sqrt(float(np.vdot(ox, ox).real * np.vdot(oy, oy).real))
        if den > 0.0 and num / den > 0.95:
            h[3][:] = np.conj(h[0][::-1])
            h[2][:] = -np.conj(h[1][::-1])
            reinits += 1
            _cma_sweep(ex, ey, taps, mu, m, h[0], h[1], h[2], h[3], ox, oy)
    return np.stack([ox, oy]), reinits, tuple(h)


def carrier(symbols, symbol_rate, reference=None, window=32):
    """modem.py:305-351; returns (recovered, f_off, edge) with edge True where the reference raises."""
    s = np.asarray(symbols, dtype=np.complex128)
    n = s.shape[1]
    spec = np.abs(np.fft.fft(s[0] ** 4)) ** 2 + np.abs(np.fft.fft(s[1] ** 4)) ** 2
    peak = int(np.argmax(spec))
    s0 = math.log(max(spec[(peak - 1) % n], 1e-300))
    s1 = math.log(max(spec[peak], 1e-300))
    s2 = math.log(max(spec[(peak + 1) % n], 1e-300))
    den = s0 - 2.0 * s1 + s2
    frac = 0.5 * (s0 - s2) / den if den != 0.0 else 0.0
    bin_step = symbol_rate / n
    f4 = np.fft.fftfreq(n, d=1.0 / symbol_rate)[peak] + frac * bin_step
    edge = abs(f4) >= symbol_rate / 2.0 - 2.0 * bin_step
    f_off = f4 / 4.0
    d = s * np.exp(-2j * np.pi * f_off * np.arange(n) / symbol_rate)
    out = np.empty_like(d)
    pad = window // 2
    for p in range(2):
        q = d[p] ** 4
        ext = np.concatenate([q[n - pad:], q, q[: window - pad - 1]])
        sm = np.convolve(ext, np.ones(window) / window, mode="valid")
        phi = (np.unwrap(np.angle(sm)) - np.pi) / 4.0
        out[p] = d[p] * np.exp(-1j * phi)
    if reference is not None:
        rf = np.fft.fft(np.asarray(reference, dtype=np.complex128), axis=1)
        for p in range(2):
            sp = np.fft.fft(out[p])
            best = None
            for r in range(2):
                c = np.fft.ifft(sp * np.conj(rf[r]))
                i = int(np.argmax(np.abs(c)))
                if best is None or abs(c[i]) > abs(best):
                    best = c[i]
            out[p] *= np.exp(-1j * round(np.angle(best) / (np.pi / 2.0)) * np.pi / 2.0)
    return out, f_off, edge


def decide(symbols):
    s = np.asarray(symbols)
    bits = np.empty(s.shape[:-1] + (2 * s.shape[-1],), dtype=np.uint8)
    bits[..., 0::2] = s.real < 0.0
    bits[..., 1::2] = s.imag < 0.0
    return bits


def count_errors(dec, ref, skip=0):
    """(best-pairing errors, counted) of modem.py:376-405 (BER = errors / (2 counted))."""
    def sym(b):
        return ((1.0 - 2.0 * b[..., 0::2].astype(np.float64)) + 1j * (1.0 - 2.0 * b[..., 1::2].astype(np.float64))) * SQRT1_2
    ds, rs = sym(np.asarray(dec)), sym(np.asarray(ref))
    dfft, rfft = np.fft.fft(ds, axis=1), np.conj(np.fft.fft(rs, axis=1))
    skip_sym = (skip + 1) // 2
    n_sym = ds.shape[1]
    best = None
    for perm in ((0, 1), (1, 0)):
        e = 0
        for p, r in enumerate(perm):
            shift = int(np.argmax(np.fft.ifft(dfft[p] * rfft[r]).real))
            rr = np.roll(rs[r], shift)
            e += int(np.sum((ds[p, skip_sym:].real < 0) != (rr[skip_sym:].real < 0)))
            e += int(np.sum((ds[p, skip_sym:].imag < 0) != (rr[skip_sym:].imag < 0)))
        if best is None or e < best:
            best = e
    return best, 2 * (n_sym - skip_sym)
