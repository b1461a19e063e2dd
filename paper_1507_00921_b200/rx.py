"""Post-DBP receiver DSP on the GPU.

Mirrors ``fiberdbp.modem`` (pkg/src/fiberdbp/modem.py): ``butterfly_equalize``
(:207-271, the CMA loop ``_cma_pass`` :183-204), ``carrier_recover``
(:283-351), ``qpsk_decide`` (:116-125), ``measure_ber`` (:358-413) with the
same arguments, validation and exceptions, plus ``receive_batch`` -- the
whole receiver of cli.py:677-685 device-resident for a batch of waveforms.
Equalisation, carrier recovery, decisions and error counting run in the
``dbp_rx_*`` kernels (csrc/rx_capi.cu, float64 like the reference);
``qpsk_map`` and ``evm_percent`` are the reference's closed-form helpers.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass

import numpy as np

from . import _native
from .params import DualPolSignal

_SQRT1_2 = 1.0 / math.sqrt(2.0)


class AlignmentError(RuntimeError):
    """No bit alignment with an error rate below the plausibility bound (modem.py:34)."""


class FrequencyOffsetError(RuntimeError):
    """Frequency offset at or beyond the estimable range, symbol rate / 8 (modem.py:38)."""


@dataclass(frozen=True)
class RxMetrics:
    """modem.py:79-90."""

    ber: float
    q_factor_db: float
    evm_percent: float
    bits_counted: int

    def __post_init__(self):
        if not (0.0 <= self.ber <= 1.0):
            raise ValueError("ber out of range")
        if self.bits_counted <= 0:
            raise ValueError("bits_counted must be positive")


class _RxCache:
    """One receiver per (device, length), grown to the largest batch seen; a
    replaced one is dropped (freed with its last reference), not closed under
    a caller that may still be using it.  Calls on one receiver serialise on
    its lock (``_native.NativeRx``)."""

    rx: dict = {}
    lock = threading.Lock()

    @classmethod
    def get(cls, device: int, n_symbols: int, batch: int) -> _native.NativeRx:
        key = (device, n_symbols)
        with cls.lock:
            r = cls.rx.get(key)
            if r is None or r.max_batch < batch:
                r = _native.NativeRx(device, n_symbols, max(batch, 1))
                cls.rx[key] = r
            return r


def qpsk_map(bits_i, bits_q) -> np.ndarray:
    """Gray mapping, unit symbol power (modem.py:110-113)."""
    return ((1.0 - 2.0 * np.asarray(bits_i)) + 1j * (1.0 - 2.0 * np.asarray(bits_q))) * _SQRT1_2


def evm_percent(rx_symbols, ref_symbols) -> float:
    """RMS error vector magnitude in percent of the reference RMS (modem.py:128-133)."""
    rx, ref = np.asarray(rx_symbols), np.asarray(ref_symbols)
    if rx.shape != ref.shape:
        raise ValueError("shape mismatch")
    return float(100.0 * np.sqrt(np.mean(np.abs(rx - ref) ** 2) / np.mean(np.abs(ref) ** 2)))


def _q_db(ber: float) -> float:
    if ber == 0.0:
        return math.inf
    from scipy.special import erfcinv
    return 20.0 * math.log10(math.sqrt(2.0) * float(erfcinv(2.0 * ber)))


def butterfly_equalize_batch(samples: np.ndarray, taps: int = 15, step_size: float = 1e-3, passes: int = 2,
                             *, device: int = 0, return_taps: bool = False):
    """(B, 2, 2 m) waveforms at 2 samples/symbol -> ((B, 2, m) complex128 symbols, reinits[B] [, taps])."""
    x = np.asarray(samples)
    if x.ndim == 2:
        x = x[None]
    if taps < 1 or taps % 2 == 0:
        raise ValueError("taps must be odd and positive")
    if step_size <= 0.0:
        raise ValueError("step_size must be positive")
    if passes < 1:
        raise ValueError("passes must be >= 1")
    n_samp = x.shape[-1]
    if n_samp % 2:
        raise ValueError("input length must be even (2 samples per symbol)")
    r = _RxCache.get(device, n_samp // 2, x.shape[0])
    out, reinits, tp = r.equalize(x, taps, step_size, passes, want_taps=return_taps)
    return (out, reinits, tp) if return_taps else (out, reinits)


def butterfly_equalize(sig: DualPolSignal, taps: int = 15, step_size: float = 1e-3, passes: int = 2,
                       return_info: bool = False, *, device: int = 0):
    """Adaptive 2x2 CMA equaliser, T/2 spaced, decimating to symbol rate (modem.py:207-271)."""
    x = np.stack([np.asarray(sig.x), np.asarray(sig.y)])
    if len(sig) % 2:
        raise ValueError("input length must be even (2 samples per symbol)")
    out, reinits, tp = butterfly_equalize_batch(x, taps, step_size, passes, device=device, return_taps=True)
    res = DualPolSignal(out[0, 0], out[0, 1], sig.sample_rate / 2.0)
    if return_info:
        return res, {"reinits": int(reinits[0]), "taps": tuple(tp[0, i].copy() for i in range(4))}
    return res


def carrier_recover_batch(symbols: np.ndarray, symbol_rate: float, reference=None, window: int = 32, *,
                          device: int = 0):
    """(B, 2, m) -> ((B, 2, m) recovered, f_off[B], status[B]); status 1 = offset at the aliasing edge."""
    s = np.asarray(symbols, dtype=np.complex128)
    if s.ndim == 2:
        s = s[None]
    if s.ndim != 3 or s.shape[1] != 2:
        raise ValueError("expected a (2, n) symbol array")
    m = s.shape[-1]
    if window < 1 or window > m:
        raise ValueError("window must be in [1, n]")
    if symbol_rate <= 0.0:
        raise ValueError("symbol_rate must be positive")
    if reference is not None:
        reference = np.asarray(reference, dtype=np.complex128)
        if reference.shape != s.shape[1:]:
            raise ValueError("reference shape must match the symbol array")
    r = _RxCache.get(device, m, s.shape[0])
    return r.carrier_recover(s, symbol_rate, reference, window)


def carrier_recover(symbols, symbol_rate: float, reference=None, window: int = 32, *, device: int = 0):
    """4th-power frequency/phase recovery with the 90-degree search (modem.py:283-351)."""
    s = np.asarray(symbols, dtype=np.complex128)
    if s.ndim != 2 or s.shape[0] != 2:
        raise ValueError("expected a (2, n) symbol array")
    out, f_off, status = carrier_recover_batch(s, symbol_rate, reference, window, device=device)
    if status[0]:
        n = s.shape[1]
        f4 = 4.0 * f_off[0]
        raise FrequencyOffsetError(
            f"4th-power peak at {f4:.3e} Hz sits at the aliasing edge; "
            f"offsets beyond {symbol_rate / 8.0:.3e} Hz are not estimable (n = {n})")
    return out[0]


def qpsk_decide(symbols, *, device: int = 0) -> np.ndarray:
    """Hard decisions, I and Q bits interleaved along the last axis (modem.py:116-125)."""
    s = np.asarray(symbols)
    shape = s.shape
    flat = s.reshape(-1).astype(np.complex128)
    n = flat.size
    if n == 0:
        return np.empty(shape[:-1] + (0,), dtype=np.uint8)
    m = (n + 1) // 2
    if 2 * m != n:
        flat = np.concatenate([flat, np.zeros(1, dtype=np.complex128)])
    r = _RxCache.get(device, m, 1)
    bits = r.decide(flat.reshape(1, 2, m)).reshape(-1)[: 2 * n]
    return bits.reshape(shape[:-1] + (2 * shape[-1],))


def _check_bits(dec, ref, skip):
    if dec.shape != ref.shape or dec.ndim != 2 or dec.shape[0] != 2:
        raise ValueError("expected matching (2, 2*n_sym) bit arrays")
    n_bits = dec.shape[1]
    if n_bits % 2:
        raise ValueError("bit streams must hold whole symbols (even length)")
    if skip < 0 or skip >= n_bits:
        raise ValueError("skip must be in [0, n_bits)")


def measure_ber(decided_bits, reference_bits, skip: int = 0, evm: float = math.nan, *,
                device: int = 0) -> RxMetrics:
    """Bit errors at the best circular alignment and polarisation pairing (modem.py:358-413)."""
    dec = np.asarray(decided_bits)
    ref = np.asarray(reference_bits)
    _check_bits(dec, ref, skip)
    r = _RxCache.get(device, dec.shape[1] // 2, 1)
    errors, counted = r.count_errors(dec[None], ref, skip)
    ber = int(errors[0]) / (2 * counted)
    if ber >= 0.4:
        raise AlignmentError(f"no alignment below BER 0.4 (best {ber:.3f})")
    return RxMetrics(ber=ber, q_factor_db=_q_db(ber), evm_percent=evm, bits_counted=2 * counted)


def receive_batch(samples: np.ndarray, symbol_rate: float, reference_symbols: np.ndarray, taps: int = 15,
                  step_size: float = 1e-3, passes: int = 2, window: int = 32, skip_bits: int = 0, *,
                  device: int = 0, devices=None):
    """cli.py:677-685 for B waveforms on the GPU: equalise, recover the carrier
    against ``reference_symbols`` (2, m), decide, count.  Returns a list with one
    ``RxMetrics`` per waveform (EVM against the scaled nearest constellation
    point, cli.py:691-695), or the exception the reference would raise."""
    x = np.asarray(samples)
    if x.ndim == 2:
        x = x[None]
    if x.dtype not in (np.complex64, np.complex128):
        x = x.astype(np.complex128)
    if devices is not None:
        devs = list(dict.fromkeys(int(d) for d in devices))
        if not devs:
            raise ValueError("devices must not be empty")
        b = x.shape[0]
        if len(devs) > 1 and b > 1:   # independent waveforms: contiguous groups, one per GPU
            from concurrent.futures import ThreadPoolExecutor
            bounds = [round(i * b / len(devs)) for i in range(len(devs) + 1)]
            parts = [(d, bounds[i], bounds[i + 1]) for i, d in enumerate(devs) if bounds[i + 1] > bounds[i]]
            with ThreadPoolExecutor(max_workers=len(parts)) as pool:
                futs = [pool.submit(receive_batch, x[lo:hi], symbol_rate, reference_symbols, taps, step_size,
                                    passes, window, skip_bits, device=d) for d, lo, hi in parts]
                return [m for f in futs for m in f.result()]
        device = devs[0]
    if taps < 1 or taps % 2 == 0:
        raise ValueError("taps must be odd and positive")
    n_samp = x.shape[-1]
    if n_samp % 2:
        raise ValueError("input length must be even (2 samples per symbol)")
    m = n_samp // 2
    ref = np.asarray(reference_symbols, dtype=np.complex128)
    if ref.shape != (2, m):
        raise ValueError("reference shape must match the symbol array")
    r = _RxCache.get(device, m, x.shape[0])
    metrics, status = r.chain(x, taps, step_size, passes, symbol_rate, ref, window, skip_bits)
    out = []
    for row, st in zip(metrics, status):
        if st == 1:
            out.append(FrequencyOffsetError(f"frequency offset {row[4]:.3e} Hz at the aliasing edge"))
        elif st == 2:
            out.append(AlignmentError(f"no alignment below BER 0.4 (best {row[0]:.3f})"))
        else:
            out.append(RxMetrics(ber=float(row[0]), q_factor_db=_q_db(float(row[0])), evm_percent=float(row[3]),
                                 bits_counted=int(row[2])))
    return out
