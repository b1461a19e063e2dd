"""Golden fixtures for the receiver DSP, made by the REFERENCE.

Run in the build container (the reference is not present on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_rx.py

Records ``fiberdbp.modem`` (pkg/src/fiberdbp/modem.py) outputs --
``butterfly_equalize`` (:207-271, symbols, final taps, re-initialisations),
``carrier_recover`` (:283-351), ``qpsk_decide`` (:116-125), ``measure_ber``
(:358-413) -- for the scenarios of pkg/tests/test_modem.py (back to back,
polarisation swap, unitary mix, laser linewidth, fixed frequency offset,
collapsed outputs) and for the golden_v1 40 x 80 km link after the
reference's own ESSFM DBP (errors at OSNR 14 dB).  Inputs are rounded to
complex64 first.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, os.environ.get("FIBERDBP_REF", "/root/reference/pkg/src"))

import fiberdbp  # noqa: E402
from fiberdbp import DualPolSignal, TxConfig, modulate_pm_qpsk  # noqa: E402
from fiberdbp import modem as ref_modem  # noqa: E402
from fiberdbp.channel import apply_jones_matrix, apply_laser_phase_noise  # noqa: E402

OUT = HERE / "golden_rx_v1.npz"
MANIFEST = HERE / "golden_rx_v1.json"


def c64(a):
    return np.asarray(a).astype(np.complex64)


def chain(arrays, cases, name, sig, ref, symbol_rate=28e9, skip_bits=128, window=32, shift=None):
    x = c64(np.stack([sig.x, sig.y]))
    sig = DualPolSignal(x[0], x[1], sig.sample_rate)
    eq, info = ref_modem.butterfly_equalize(sig, return_info=True)
    eqs = eq.stack()
    cr_in = eqs if shift is None else eqs * shift
    rec = ref_modem.carrier_recover(cr_in, symbol_rate, reference=ref, window=window)
    dec = ref_modem.qpsk_decide(rec)
    ref_bits = ref_modem.qpsk_decide(ref)
    met = ref_modem.measure_ber(dec, ref_bits, skip=skip_bits)
    arrays[f"{name}_in"] = x
    arrays[f"{name}_ref"] = ref
    arrays[f"{name}_eq"] = eqs
    arrays[f"{name}_taps"] = np.stack(info["taps"])
    arrays[f"{name}_cr_in"] = cr_in
    arrays[f"{name}_rec"] = rec
    arrays[f"{name}_dec"] = dec
    cases.append(dict(name=name, symbol_rate=symbol_rate, skip_bits=skip_bits, window=window,
                      reinits=info["reinits"], ber=met.ber, q_db=met.q_factor_db, bits_counted=met.bits_counted,
                      shifted=shift is not None))
    print(f"{name}: reinits {info['reinits']} ber {met.ber:.3e} bits {met.bits_counted}")


def main():
    t0 = time.time()
    arrays, cases = {}, []
    sig, ref = modulate_pm_qpsk(TxConfig(num_symbols=2 ** 12, rng_seed=1))
    chain(arrays, cases, "b2b", sig, ref)
    sig, ref = modulate_pm_qpsk(TxConfig(num_symbols=2 ** 12, rng_seed=2))
    chain(arrays, cases, "swap", apply_jones_matrix(sig, np.array([[0.0, 1.0], [1.0, 0.0]])), ref)
    sig, ref = modulate_pm_qpsk(TxConfig(num_symbols=2 ** 12, rng_seed=3))
    th = 0.3
    jones = np.array([[math.cos(th), math.sin(th)], [-math.sin(th), math.cos(th)]], dtype=complex)
    chain(arrays, cases, "mix", apply_jones_matrix(sig, jones), ref)
    sig, ref = modulate_pm_qpsk(TxConfig(num_symbols=2 ** 12, rng_seed=4))
    chain(arrays, cases, "linewidth", apply_laser_phase_noise(sig, 100e3, rng=11), ref)
    sig, ref = modulate_pm_qpsk(TxConfig(num_symbols=2 ** 12, rng_seed=6))
    n = 2 ** 12
    rot = np.exp(2j * np.pi * 1e9 * np.arange(n) / 28e9 + 0.7j)
    chain(arrays, cases, "freq", sig, ref, shift=rot)
    # identical polarisations: the two outputs collapse and the second filter pair is re-initialised
    sig, ref = modulate_pm_qpsk(TxConfig(num_symbols=2 ** 12, rng_seed=5))
    jones = np.array([[1.0, 0.0], [1.0, 0.0]], dtype=complex) / math.sqrt(2.0)
    x = c64(np.stack([sig.x, sig.y]))
    mixed = apply_jones_matrix(DualPolSignal(x[0], x[1], sig.sample_rate), jones)
    eq, info = ref_modem.butterfly_equalize(mixed, return_info=True)
    arrays["collapse_in"] = c64(mixed.stack())
    arrays["collapse_eq"] = eq.stack()
    arrays["collapse_taps"] = np.stack(info["taps"])
    cases.append(dict(name="collapse", reinits=info["reinits"], equalize_only=True))
    print(f"collapse: reinits {info['reinits']}")
    # the golden_v1 link after the reference's ESSFM DBP (errors at OSNR 14 dB)
    g = np.load(HERE / "golden_v1.npz")
    dbp_out = g["link_c0_sym_out"]
    chain(arrays, cases, "link", DualPolSignal(dbp_out[0], dbp_out[1], 56e9), g["link_tx_symbols"], skip_bits=0)
    # measure_ber known answers (test_modem.py:201-235): reference bit streams
    _, ref = modulate_pm_qpsk(TxConfig(num_symbols=2 ** 10, rng_seed=8))
    arrays["bits8"] = ref_modem.qpsk_decide(ref)
    _, ref = modulate_pm_qpsk(TxConfig(num_symbols=2 ** 10, rng_seed=9))
    arrays["bits9"] = ref_modem.qpsk_decide(ref)
    # transmitter and laser phase noise (modem.py:90-180, channel.py:156-171)
    sig, ref = modulate_pm_qpsk(TxConfig(num_symbols=2 ** 8, rng_seed=8))
    arrays["tx_nrz"], arrays["tx_nrz_ref"] = sig.stack(), ref
    sig, ref = modulate_pm_qpsk(TxConfig(num_symbols=2 ** 8, rng_seed=9, pulse="rc", rolloff=0.2))
    arrays["tx_rc"], arrays["tx_rc_ref"] = sig.stack(), ref
    arrays["laser_out"] = apply_laser_phase_noise(sig, 100e3, rng=11).stack()
    np.savez_compressed(OUT, **arrays)
    MANIFEST.write_text(json.dumps(dict(generator="tests/golden/make_golden_rx.py",
                                        reference="fiberdbp " + fiberdbp.__version__,
                                        numpy=np.__version__, cases=cases), indent=1))
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB) in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
