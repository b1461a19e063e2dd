"""Host-side mirror of the reference API: validation, warnings, schedule, tables (no GPU)."""

import math
import warnings

import numpy as np
import pytest

import paper_1507_00921_b200 as pb
from paper_1507_00921_b200 import backprop
from oracle import dbp_port

STD = pb.FiberParams(beta2=-21.0, gamma=1.3, alpha_db_per_km=0.2, length=40.0)


def quiet(n, span=STD):
    return pb.LinkConfig(span=span, num_spans=n, amp_noise_figure_db=None, pol_rotation=False)


def test_dbp_config_validation():                       # test_dbp.py:75-87
    plan = pb.OverlapPlan(256, 64)
    link = quiet(2)
    for kw in (dict(algorithm="trellis"), dict(algorithm="ssfm", num_steps=0),
               dict(algorithm="ssfm", arrangement="diagonal"), dict(algorithm="essfm"),
               dict(algorithm="essfm", coeffs=pb.EssfmCoefficients.identity(128))):
        alg = kw.pop("algorithm")
        with pytest.raises(ValueError):
            pb.DbpConfig(alg, plan, link, **kw)


def test_value_type_validation():                       # test_sigkit.py / test_spectral.py
    with pytest.raises(ValueError):
        pb.DualPolSignal(np.zeros(3), np.zeros(4), 1e9)
    with pytest.raises(ValueError):
        pb.DualPolSignal(np.zeros(0), np.zeros(0), 1e9)
    with pytest.raises(ValueError):
        pb.DualPolSignal(np.zeros(3), np.zeros(3), 0.0)
    with pytest.raises(ValueError):
        pb.FiberParams(-21.0, 1.3, -0.1, 40.0)
    with pytest.raises(ValueError):
        pb.LinkConfig(STD, 0)
    with pytest.raises(ValueError):
        pb.EssfmCoefficients([])
    with pytest.raises(ValueError):
        pb.EssfmCoefficients([1.0, np.nan])
    with pytest.raises(ValueError):
        pb.OverlapPlan(1000, 100)
    with pytest.raises(ValueError):
        pb.OverlapPlan(1024, 1024)
    assert pb.OverlapPlan(2048, 512).usable == 1536
    s = pb.DualPolSignal([1, 2], [3, 4], 1e9)
    assert s.x.dtype == np.complex128 and len(s) == 2


def test_channel_memory_and_fft_grid():
    assert pb.channel_memory_samples(21.0, 3000.0, 50e9) == pytest.approx(989.6016858807848)
    assert pb.estimate_channel_memory(21.0, 3200.0, 56e9) == 2048
    np.testing.assert_allclose(pb.fft_frequencies(8, 8e9), np.array([0, 1, 2, 3, -4, -3, -2, -1]) * 1e9)
    with pytest.raises(ValueError):
        pb.fft_frequencies(12, 8e9)


def test_schedule_matches_reference_fixture(golden, manifest):
    for i in range(manifest["sched_cases"]):
        beta2, gamma, adb, span, ns, steps = golden[f"sched{i}_args"]
        link = quiet(int(ns), pb.FiberParams(beta2, gamma, adb, span))
        np.testing.assert_array_equal(np.array(backprop._reverse_step_schedule(link, int(steps))),
                                      golden[f"sched{i}"])


def test_short_overlap_warning_text():                  # dbp.py:175-181
    cfg = pb.DbpConfig("ffe", pb.OverlapPlan(1024, 256), quiet(80))
    with pytest.warns(UserWarning, match="channel memory"):
        backprop._warn_short_overlap(cfg, 56e9, stacklevel=1)
    cfg = pb.DbpConfig("ffe", pb.OverlapPlan(2048, 512), quiet(1))
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        backprop._warn_short_overlap(cfg, 56e9, stacklevel=1)


def test_dispersion_tables_match_oracle():
    f = pb.fft_frequencies(2048, 56e9)
    np.testing.assert_array_equal(backprop._dispersion(f, -21.68, 3200.0),
                                  dbp_port.dispersion_response(2048, 56e9, -21.68, 3200.0))


def test_jobs_validated_before_gpu():
    sig = pb.DualPolSignal(np.ones(8), np.ones(8), 56e9)
    cfg = pb.DbpConfig("ffe", pb.OverlapPlan(16, 4), quiet(1))
    with pytest.raises(ValueError):
        pb.backpropagate(sig, cfg, jobs=0)


def test_effective_length():
    assert pb.effective_length(0.0461, 80.0) == pytest.approx(21.149197483217407)
    assert pb.effective_length(0.0, 5.0) == 5.0
    assert pb.effective_length(1e-12, 1.0) == pytest.approx(1.0)
    assert pb.scale_to_power(pb.DualPolSignal([1, 1], [1, 1], 1.0), 0.0).x[0] == pytest.approx(math.sqrt(1e-3 / 2))


def test_train_config_validation_and_coefficient_files(tmp_path):   # test_train.py
    with pytest.raises(ValueError):
        pb.TrainConfig(n_coeffs=-1)
    with pytest.raises(ValueError):
        pb.TrainConfig(n_coeffs=32, train_samples=100)
    c = pb.EssfmCoefficients(np.array([0.9, 0.05, -0.01]))
    pb.save_coefficients(tmp_path / "c.txt", c)
    np.testing.assert_array_equal(pb.load_coefficients(tmp_path / "c.txt").c, c.c)
    (tmp_path / "bad.txt").write_text("3\n1.0\n")
    with pytest.raises(ValueError):
        pb.load_coefficients(tmp_path / "bad.txt")
    assert pb.mse(np.ones((2, 4)), np.ones((2, 4))) == 0.0


def test_receiver_and_simulator_validation_before_any_gpu_work():
    # argument checks mirror modem.py / channel.py and raise before a device is touched
    x = np.ones((2, 64), dtype=np.complex128)
    s = pb.DualPolSignal(x[0], x[1], 56e9)
    with pytest.raises(ValueError):
        pb.butterfly_equalize(s, taps=14)
    with pytest.raises(ValueError):
        pb.butterfly_equalize(s, step_size=0.0)
    with pytest.raises(ValueError):
        pb.butterfly_equalize(s, passes=0)
    with pytest.raises(ValueError):
        pb.butterfly_equalize(pb.DualPolSignal(np.ones(15, complex), np.ones(15, complex), 2e9))
    with pytest.raises(ValueError):
        pb.carrier_recover(np.ones(16, dtype=complex), 28e9)
    with pytest.raises(ValueError):
        pb.carrier_recover(np.ones((2, 16), dtype=complex), 28e9, window=0)
    with pytest.raises(ValueError):
        pb.carrier_recover(np.ones((2, 16), dtype=complex), 0.0)
    bits = np.zeros((2, 8), dtype=np.uint8)
    with pytest.raises(ValueError):
        pb.measure_ber(bits[:, :6], bits)
    with pytest.raises(ValueError):
        pb.measure_ber(bits, bits, skip=-1)
    with pytest.raises(ValueError):
        pb.SsfmStepConfig(0)
    span = pb.FiberParams(-21.0, 1.3, 0.2, 40.0)
    with pytest.raises(ValueError):
        pb.propagate_span(pb.DualPolSignal(np.ones(1000, complex), np.ones(1000, complex), 56e9), span,
                          pb.SsfmStepConfig(2))
    with pytest.raises(ValueError):
        pb.propagate_link(s, pb.LinkConfig(span=span, num_spans=1), pb.SsfmStepConfig(1),
                          rng=np.random.default_rng(0))
    with pytest.raises(ValueError):
        pb.amplify_with_ase(s, -1.0, None)
    u = pb.haar_random_unitary(3)
    np.testing.assert_allclose(u @ u.conj().T, np.eye(2), atol=1e-12)


def test_gpu_entry_points_fail_loudly_without_a_device():
    # no CPU fallback: on a machine without a CUDA device the simulator / receiver refuse to run
    from paper_1507_00921_b200 import _native
    if _native.device_count() > 0:
        pytest.skip("a CUDA device is visible")
    x = np.ones((2, 1024), dtype=np.complex64)
    with pytest.raises(RuntimeError):
        pb.propagate_span(pb.DualPolSignal(x[0], x[1], 56e9), pb.FiberParams(-21.0, 1.3, 0.2, 40.0),
                          pb.SsfmStepConfig(1))
    with pytest.raises(RuntimeError):
        pb.butterfly_equalize(pb.DualPolSignal(x[0], x[1], 56e9))


def test_output_row_arena_never_aliases_live_results():
    # backprop._RowArena: the complex128 output rows of backpropagate() are recycled only
    # once nothing refers to them (sigkit.py:56-68 promises the caller its own arrays)
    arena = backprop._RowArena(16 << 20)
    n = 1 << 16                                            # 1 MiB rows
    a, b = arena.take(n), arena.take(n)
    assert a.dtype == np.complex128 and a.shape == (n,) and not np.shares_memory(a, b)
    addr = a.__array_interface__["data"][0]
    part = a[7:99]                                         # a slice keeps the row busy
    sig = pb.DualPolSignal(b, b, 1.0)                      # so does a signal built on it
    baddr = b.__array_interface__["data"][0]
    del a, b
    c = arena.take(n)
    assert c.__array_interface__["data"][0] not in (addr, baddr)
    del part
    d = arena.take(n)
    assert d.__array_interface__["data"][0] == addr        # recycled once free
    assert arena.take(n // 2).size == n // 2               # other lengths get their own rows
    del sig
    # the cap bounds what is tracked; rows that do not fit are plain allocations
    held = [arena.take(n) for _ in range(40)]
    assert arena.tracked_bytes() <= 16 << 20
    assert len({h.__array_interface__["data"][0] for h in held}) == 40
    small = arena.take(16)                                 # heap-sized rows bypass the arena
    assert small.base is None
    assert backprop._RowArena(0).take(n).base is None      # DBP_HOST_ARENA_MB=0: disabled
