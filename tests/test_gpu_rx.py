"""GPU parity of the receiver DSP against the reference.

Fixtures: tests/golden/golden_rx_v1.npz, the reference's own
``butterfly_equalize`` / ``carrier_recover`` / ``qpsk_decide`` /
``measure_ber`` outputs (modem.py:116-413) for the pkg/tests/test_modem.py
scenarios and for the 40 x 80 km link after the reference DBP.  The GPU
computes in float64 like the reference; only the summation order differs,
so equalised symbols and taps agree to 1e-10 (absolute, unit-power
symbols) and decisions, re-initialisations, error counts, BER and Q are
identical.  Carrier recovery is held to CARRIER_ATOL = 1e-4: its parabolic
peak refinement takes the log of the 4th-power spectrum next to the peak,
which for a clean (back-to-back) signal is FFT rounding noise in both
implementations, so the refined offset -- and, after the phase tracker,
the symbols -- differ at the 1e-5 level; decisions stay identical.
Known answers follow test_modem.py:201-256.
"""

import math

import numpy as np
import pytest

import paper_1507_00921_b200 as pb
from paper_1507_00921_b200 import _native
from oracle import rx_port

pytestmark = pytest.mark.gpu
ATOL = 1e-10
CARRIER_ATOL = 1e-4


def _sig(x, rate=56e9):
    return pb.DualPolSignal(x[0], x[1], rate)


def test_equalizer_matches_reference(golden_rx, manifest_rx):
    before = _native.launch_count()
    for case in manifest_rx["cases"]:
        name = case["name"]
        eq, info = pb.butterfly_equalize(_sig(golden_rx[f"{name}_in"]), return_info=True)
        assert info["reinits"] == case["reinits"], name
        np.testing.assert_allclose(eq.stack(), golden_rx[f"{name}_eq"], rtol=0, atol=ATOL, err_msg=name)
        np.testing.assert_allclose(np.stack(info["taps"]), golden_rx[f"{name}_taps"], rtol=0, atol=ATOL,
                                   err_msg=name)
        assert eq.sample_rate == 28e9
    assert _native.launch_count() > before


def test_carrier_decide_count_match_reference(golden_rx, manifest_rx):
    for case in manifest_rx["cases"]:
        if case.get("equalize_only"):
            continue
        name = case["name"]
        rec = pb.carrier_recover(golden_rx[f"{name}_cr_in"], case["symbol_rate"], reference=golden_rx[f"{name}_ref"],
                                 window=case["window"])
        err = float(np.max(np.abs(rec - golden_rx[f"{name}_rec"])))
        print(f"{name}: carrier max |diff| {err:.2e}")
        assert err <= CARRIER_ATOL, (name, err)
        dec = pb.qpsk_decide(rec)
        np.testing.assert_array_equal(dec, golden_rx[f"{name}_dec"])
        met = pb.measure_ber(dec, pb.qpsk_decide(golden_rx[f"{name}_ref"]), skip=case["skip_bits"])
        assert met.ber == case["ber"] and met.bits_counted == case["bits_counted"], name
        assert met.q_factor_db == case["q_db"], name


def test_receive_chain_matches_reference(golden_rx, manifest_rx):
    for case in manifest_rx["cases"]:
        if case.get("equalize_only") or case["shifted"]:
            continue
        name = case["name"]
        x = golden_rx[f"{name}_in"]
        for dtype in (np.complex128, np.complex64):
            (met,) = pb.receive_batch(x.astype(dtype), case["symbol_rate"], golden_rx[f"{name}_ref"],
                                      window=case["window"], skip_bits=case["skip_bits"])
            assert met.ber == case["ber"] and met.bits_counted == case["bits_counted"], (name, dtype)
            assert met.q_factor_db == case["q_db"]
            if dtype is np.complex128:
                # EVM against the scaled nearest point (cli.py:691-695) of the reference's symbols
                rec = golden_rx[f"{name}_rec"]
                scale = np.sqrt(np.mean(np.abs(rec) ** 2))
                nearest = scale * pb.qpsk_map((rec.real < 0).astype(float), (rec.imag < 0).astype(float))
                assert met.evm_percent == pytest.approx(pb.evm_percent(rec, nearest), rel=1e-3, abs=1e-2)


def test_receive_batch_equals_single(golden_rx, manifest_rx):
    x = golden_rx["link_in"]
    ref = golden_rx["link_ref"]
    batch = np.stack([x, x * np.exp(0.3j), x[::-1].copy()])
    many = pb.receive_batch(batch, 28e9, ref)
    for i in range(3):
        (one,) = pb.receive_batch(batch[i], 28e9, ref)
        if isinstance(one, Exception):
            assert type(many[i]) is type(one)
        else:
            assert many[i] == one


def test_measure_ber_known_answers(golden_rx):
    bits = golden_rx["bits8"]
    clean = pb.measure_ber(bits, bits)
    assert clean.ber == 0.0 and clean.bits_counted == 2 * bits.shape[1]
    flipped = bits.copy()
    flipped[0, 100] ^= 1
    flipped[1, 200] ^= 1
    assert pb.measure_ber(flipped, bits).ber == pytest.approx(2.0 / clean.bits_counted)
    bits = golden_rx["bits9"]
    flipped = bits.copy()
    for k in (11, 303, 707, 1501):
        flipped[0, k] ^= 1
    met = pb.measure_ber(flipped[:, :2000], bits[:, :2000])
    assert met.ber == pytest.approx(1e-3, rel=1e-12)
    assert met.q_factor_db == pytest.approx(9.79982256904398, rel=1e-9)
    flipped = bits[:, :512].copy()
    flipped[0, 3] ^= 1
    assert pb.measure_ber(flipped, bits[:, :512], skip=16).ber == 0.0
    with pytest.raises(ValueError):
        pb.measure_ber(bits[:, :10], bits[:, :12])
    with pytest.raises(ValueError):
        pb.measure_ber(bits, bits, skip=-1)
    rng = np.random.default_rng(0)
    a = rng.integers(0, 2, size=(2, 4096)).astype(np.uint8)
    b = rng.integers(0, 2, size=(2, 4096)).astype(np.uint8)
    with pytest.raises(pb.AlignmentError):
        pb.measure_ber(a, b)


def test_awgn_error_counts_equal_oracle():
    rng = np.random.default_rng(7)
    n_sym = 2 ** 18
    bi = rng.integers(0, 2, size=(2, n_sym)).astype(np.float64)
    bq = rng.integers(0, 2, size=(2, n_sym)).astype(np.float64)
    sym = pb.qpsk_map(bi, bq)
    noise = math.sqrt(0.1 / 2.0) * (rng.normal(size=sym.shape) + 1j * rng.normal(size=sym.shape))
    ref = np.empty((2, 2 * n_sym), dtype=np.uint8)
    ref[:, 0::2] = bi
    ref[:, 1::2] = bq
    dec = pb.qpsk_decide(sym + noise)
    np.testing.assert_array_equal(dec, rx_port.decide(sym + noise))
    met = pb.measure_ber(dec, ref, skip=64)
    errors, counted = rx_port.count_errors(dec, ref, 64)
    assert met.ber == errors / (2 * counted) and met.bits_counted == 2 * counted
    ber_theory = 0.5 * math.erfc(math.sqrt(10.0 / 2.0))
    assert met.ber == pytest.approx(ber_theory, rel=0.15)


def test_validation_and_edge_offset(golden_rx):
    x = golden_rx["b2b_in"]
    with pytest.raises(ValueError):
        pb.butterfly_equalize(_sig(x), taps=14)
    with pytest.raises(ValueError):
        pb.butterfly_equalize(_sig(x), step_size=0.0)
    with pytest.raises(ValueError):
        pb.butterfly_equalize(_sig(x), passes=0)
    with pytest.raises(ValueError):
        pb.butterfly_equalize(_sig(np.ones((2, 15), dtype=complex)))
    with pytest.raises(ValueError):
        pb.carrier_recover(np.ones(16, dtype=complex), 28e9)
    with pytest.raises(ValueError):
        pb.carrier_recover(np.ones((2, 16), dtype=complex), 28e9, window=0)
    with pytest.raises(ValueError):
        pb.carrier_recover(np.ones((2, 16), dtype=complex), 0.0)
    eq = golden_rx["b2b_eq"]
    n = eq.shape[1]
    rot = np.exp(2j * np.pi * (28e9 / 8.0) * np.arange(n) / 28e9)
    with pytest.raises(pb.FrequencyOffsetError):
        pb.carrier_recover(eq * rot, 28e9, reference=golden_rx["b2b_ref"])
    _, _, edge = rx_port.carrier(eq * rot, 28e9, golden_rx["b2b_ref"])
    assert edge


def test_config_size_batch_matches_oracle():
    # 2^16 symbols per polarisation (BASELINE configs), 4 waveforms with different channels
    from oracle.waveforms import qpsk_rrc
    tx, sym = qpsk_rrc(2 ** 16, seed=3)
    rng = np.random.default_rng(1)
    xs = []
    for i in range(4):
        th = 0.2 * i
        j = np.array([[math.cos(th), math.sin(th)], [-math.sin(th), math.cos(th)]])
        y = j @ tx
        y = y + 0.05 * (rng.normal(size=y.shape) + 1j * rng.normal(size=y.shape)) * np.sqrt(np.mean(np.abs(y) ** 2))
        xs.append(y)
    xs = np.stack(xs)
    eq, reinits = pb.butterfly_equalize_batch(xs)
    for i in (0, 3):
        want, nre, _ = rx_port.equalize(xs[i])
        assert reinits[i] == nre
        np.testing.assert_allclose(eq[i], want, rtol=0, atol=1e-9)
    mets = pb.receive_batch(xs, 28e9, sym)
    for i in (0, 3):
        rec, _, _ = rx_port.carrier(eq[i], 28e9, sym)
        errors, counted = rx_port.count_errors(rx_port.decide(rec), rx_port.decide(sym))
        assert mets[i].ber == errors / (2 * counted)
