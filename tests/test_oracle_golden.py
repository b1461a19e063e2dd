"""Pin the CPU oracle (oracle/dbp_port.py) to the reference's own outputs.

The fixtures were produced by tests/golden/make_golden.py running the
reference ``fiberdbp`` package; the known answers come from the reference
tests (pkg/tests/test_dbp.py, test_spectral.py, test_sigkit.py, oracles.py).
"""

import cmath

import numpy as np
import pytest

from oracle import dbp_port

from .helpers import case_config, port_config


def test_channel_memory_matches_reference(golden):
    for args, want in zip(golden["memory_args"], golden["memory_vals"]):
        assert dbp_port.memory_in_samples(*args) == want
    # test_dbp.py:31-37 known answers
    assert dbp_port.memory_in_samples(21.0, 3000.0, 50e9) == pytest.approx(989.6016858807848)
    assert dbp_port.pow2_ceil(dbp_port.memory_in_samples(21.0, 3200.0, 56e9)) == 2048
    assert dbp_port.pow2_ceil(dbp_port.memory_in_samples(21.0, 2000.0, 50e9)) == 1024
    assert dbp_port.pow2_ceil(989.6016858807848) == 1024 and dbp_port.pow2_ceil(0.3) == 1


def test_schedule_matches_reference(golden, manifest):
    for i in range(manifest["sched_cases"]):
        beta2, gamma, adb, span, ns, steps = golden[f"sched{i}_args"]
        got = np.array(dbp_port.step_table(adb, span, int(ns), int(steps)))
        np.testing.assert_array_equal(got, golden[f"sched{i}"])


def test_schedule_known_answers():
    le = dbp_port.effective_len(dbp_port.LN10_OVER_10 * 0.2, 40.0)
    (dz, w, g), = dbp_port.step_table(0.2, 40.0, 4, 1)      # test_dbp.py:157-164
    assert dz == pytest.approx(160.0) and w == pytest.approx(4 * le, rel=1e-12) and g == pytest.approx(1.0)
    for num_steps in (1, 2, 3, 5, 8, 160):                    # test_dbp.py:177-192
        rows = dbp_port.step_table(0.2, 40.0, 8, num_steps)
        assert sum(r[1] for r in rows) >= 8 * le - 1e-9
        assert np.prod([r[2] for r in rows]) == pytest.approx(1.0, rel=1e-12)
        assert sum(r[0] for r in rows) == pytest.approx(320.0)
    for dz, w, g in dbp_port.step_table(0.0, 50.0, 2, 5):     # test_dbp.py:195-200
        assert w == pytest.approx(dz) and g == pytest.approx(1.0)
    assert dbp_port.effective_len(0.0461, 80.0) == pytest.approx(21.149197483217407)


def _nested_loop(block, gamma, dz_eff, c):
    """Sample-by-sample filtered rotation (the reference's oracles.py:28-43 geometry)."""
    n = block.shape[1]
    power = [abs(block[0, j]) ** 2 + abs(block[1, j]) ** 2 for j in range(n)]
    out = np.empty_like(block)
    for k in range(n):
        acc = c[0] * power[k]
        for i in range(1, len(c)):
            acc += c[i] * (power[(k - i) % n] + power[(k + i) % n])
        out[:, k] = block[:, k] * cmath.exp(-1j * gamma * dz_eff * acc)
    return out


@pytest.mark.parametrize("nc", [0, 1, 2, 4])
def test_rotation_matches_reference_and_nested_loop(golden, nc):
    blk, c = golden[f"sub{nc}_in"], golden[f"sub{nc}_c"]
    got = dbp_port.rotate_essfm(blk, 1.7, 0.25, c)
    np.testing.assert_array_equal(got, golden[f"sub{nc}_out"])
    np.testing.assert_allclose(got, _nested_loop(blk, 1.7, 0.25, c), rtol=0, atol=1e-14)


def test_identity_rotation_is_plain_rotation(rng):
    blk = rng.normal(size=(2, 64)) + 1j * rng.normal(size=(2, 64))
    c = np.zeros(7)
    c[0] = 1.0
    np.testing.assert_array_equal(dbp_port.rotate_essfm(blk, 1.3, 18.2, c),
                                  dbp_port.rotate_ssfm(blk, 1.3, 18.2))


def test_backpropagate_cases_match_reference(golden, manifest):
    for case in manifest["cases"]:
        name = case["name"]
        key = f"bp_{name}" if case["signal"] == "white" else f"link_{name}"
        x = golden[f"bp_{name}_in"] if case["signal"] == "white" else golden["link_rx"]
        coeffs = None
        if case["algorithm"] == "essfm":
            coeffs = golden[f"bp_{name}_c"] if case["signal"] == "white" else golden["link_c17"]
        cfg = case_config(case, coeffs)
        got = dbp_port.backpropagate_arrays(x.astype(np.complex128), case["sample_rate"], port_config(cfg))
        want = golden[f"{key}_out"]
        scale = np.max(np.abs(want))
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-12 * scale, err_msg=name)


def test_block_operator_matches_captured_closure(golden, manifest):
    for case in manifest["cases"]:
        if case["signal"] != "link":
            continue
        name = case["name"]
        coeffs = golden["link_c17"] if case["algorithm"] == "essfm" else None
        cfg = case_config(case, coeffs)
        blocks = golden[f"link_{name}_blk_in"].astype(np.complex128)
        got = dbp_port.process_blocks(blocks, case["sample_rate"], port_config(cfg))
        np.testing.assert_allclose(got, golden[f"link_{name}_blk_out"], rtol=0,
                                   atol=1e-12 * np.max(np.abs(got)), err_msg=name)


@pytest.mark.parametrize("n_total", [1, 5, 1536, 1537, 4096, 5000])
def test_framing_identity(rng, n_total):                       # test_spectral.py:72-77
    x = rng.normal(size=(2, n_total)) + 1j * rng.normal(size=(2, n_total))
    blocks = dbp_port.cut_blocks(x, 2048, 512)
    np.testing.assert_array_equal(dbp_port.join_blocks(blocks, n_total, 512), x)


def test_frequency_grid():                                     # test_spectral.py:47-53
    np.testing.assert_allclose(dbp_port.bin_frequencies(8, 8e9),
                               np.array([0, 1, 2, 3, -4, -3, -2, -1]) * 1e9)


def test_training_port_matches_reference(golden):
    # train.py:86-188 restated on the oracle port, pinned to the reference's own fit
    from oracle import train_port
    from oracle.waveforms import d_to_beta2
    cfg = dbp_port.PortConfig("essfm", 2048, 700, d_to_beta2(17.0), 1.3, 0.2, 80.0, 40, 1,
                              np.array([1.0, 0, 0, 0, 0]), "symmetric")
    c, err, initial, _, iters = train_port.fit(golden["link_rx"].astype(np.complex128), 56e9, cfg,
                                               n_coeffs=4, target_steps_per_span=2, train_samples=8192,
                                               max_iterations=6)
    ref_initial, ref_final, ref_iters, _ = golden["train_mse"]
    assert iters == ref_iters
    np.testing.assert_allclose([initial, err], [ref_initial, ref_final], rtol=1e-9)
    np.testing.assert_allclose(c, golden["train_c"], rtol=0, atol=1e-9)


def test_channel_port_matches_reference_forward_fixtures(golden_fwd, manifest_fwd):
    # channel.py:74-207 restated in oracle/channel_port.py, pinned to the reference's own outputs
    from oracle import channel_port as cp
    for case in manifest_fwd["cases"]:
        name, x = case["name"], golden_fwd[f"{case['name']}_in"].astype(np.complex128)
        if case["kind"] == "span":
            got = cp.span(x, case["sample_rate"], case["beta2"], case["gamma"], case["alpha_db_per_km"],
                          case["length"], case["steps_per_span"], case["nonlinear"])
        else:
            got = cp.link(x, case["sample_rate"], case["beta2"], case["gamma"], case["alpha_db_per_km"],
                          case["length"], case["num_spans"], case["steps_per_span"], case["amp_gain_db"],
                          case["amp_noise_figure_db"], case["pol_rotation"], case["center_wavelength_nm"],
                          case["rng"], case["nonlinear"])
        want = golden_fwd[f"{name}_out"]
        tol = 1e-6 if want.dtype == np.complex64 else 1e-12
        np.testing.assert_allclose(got, want, rtol=0, atol=tol * np.max(np.abs(want)), err_msg=name)
    x = golden_fwd["amp_in"].astype(np.complex128)
    np.testing.assert_allclose(cp.amplify(x, 56e9, 16.0, 5.0, 1550.0, 3), golden_fwd["amp_out"], rtol=1e-13, atol=0)
    np.testing.assert_allclose(cp.amplify(x, 56e9, 16.0, None), golden_fwd["amp_quiet_out"], rtol=1e-13, atol=0)
    np.testing.assert_allclose(cp.haar(11), golden_fwd["haar11"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(cp.haar(5) @ x, golden_fwd["rot_out"], rtol=0, atol=1e-13)


def test_rx_port_matches_reference_receiver_fixtures(golden_rx, manifest_rx):
    # modem.py:183-413 restated in oracle/rx_port.py, pinned to the reference's own outputs
    from oracle import rx_port
    for case in manifest_rx["cases"]:
        name = case["name"]
        eq, reinits, taps = rx_port.equalize(golden_rx[f"{name}_in"])
        assert reinits == case["reinits"], name
        np.testing.assert_allclose(eq, golden_rx[f"{name}_eq"], rtol=0, atol=1e-12, err_msg=name)
        np.testing.assert_allclose(np.stack(taps), golden_rx[f"{name}_taps"], rtol=0, atol=1e-12, err_msg=name)
        if case.get("equalize_only"):
            continue
        rec, _, edge = rx_port.carrier(golden_rx[f"{name}_cr_in"], case["symbol_rate"], golden_rx[f"{name}_ref"],
                                       case["window"])
        assert not edge
        np.testing.assert_allclose(rec, golden_rx[f"{name}_rec"], rtol=0, atol=1e-12, err_msg=name)
        dec = rx_port.decide(rec)
        np.testing.assert_array_equal(dec, golden_rx[f"{name}_dec"])
        errors, counted = rx_port.count_errors(dec, rx_port.decide(golden_rx[f"{name}_ref"]), case["skip_bits"])
        assert errors / (2 * counted) == case["ber"] and 2 * counted == case["bits_counted"], name


def test_modem_port_matches_reference_transmitter(golden_rx):
    # modem.py:90-180 and channel.py:156-171 restated in oracle/modem_port.py
    from oracle import modem_port as mp
    wave, ref = mp.modulate_pm_qpsk(2 ** 8, 8)
    np.testing.assert_array_equal(ref, golden_rx["tx_nrz_ref"])
    np.testing.assert_array_equal(wave, golden_rx["tx_nrz"])
    wave, ref = mp.modulate_pm_qpsk(2 ** 8, 9, pulse="rc", rolloff=0.2)
    np.testing.assert_array_equal(ref, golden_rx["tx_rc_ref"])
    np.testing.assert_allclose(wave, golden_rx["tx_rc"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(mp.laser_phase_noise(wave, 100e3, 56e9, rng=11), golden_rx["laser_out"],
                               rtol=0, atol=1e-13)
    assert mp.generate_prbs(7, 1).size == 127 and abs(int(mp.generate_prbs(7, 1).sum()) - 64) == 0
