"""GPU parity of the whole-waveform link simulator against the reference.

The fixtures (tests/golden/golden_fwd_v1.npz) are the reference's own
``propagate_span`` / ``propagate_link`` outputs (channel.py:74-207); above
their sizes the oracle restatement oracle/channel_port.py (pinned to the same
fixtures) is the checker.  The ASE and Haar draws are bit-identical host
numpy draws, so a seeded GPU run reproduces the reference realisation; the
GPU computes in complex64 and the tolerance is relative L2 over the whole
waveform, tol(steps) = 2e-6 + 6e-8 * steps: float32 rounding of the
transform constants is the same every step, so it accumulates linearly per
frequency bin (measured ~4e-8 per step after the |w|-balanced constants in
csrc/dft_small.cuh).  For scale: a complex64 numpy restatement of the same
3200-step link (tools/diag_sim.py --fp32-numpy) is 2.1e-4 from the
reference; the GPU is 1.4e-4.
"""

import math
from pathlib import Path

import numpy as np
import pytest

import paper_1507_00921_b200 as pb
from paper_1507_00921_b200 import _native
from oracle import channel_port as cp

from .helpers import rel_l2

pytestmark = pytest.mark.gpu


def tol(total_steps: int) -> float:
    return 2e-6 + 6e-8 * total_steps


def _fiber(case):
    return pb.FiberParams(case["beta2"], case["gamma"], case["alpha_db_per_km"], case["length"])


def _sig(x):
    return pb.DualPolSignal(x[0], x[1], 56e9)


def test_golden_forward_cases_match_reference(golden_fwd, manifest_fwd):
    before = _native.launch_count()
    errs = {}
    for case in manifest_fwd["cases"]:
        name, x = case["name"], golden_fwd[f"{case['name']}_in"]
        cfg = pb.SsfmStepConfig(case["steps_per_span"], case["nonlinear"])
        if case["kind"] == "span":
            got = pb.propagate_span(_sig(x), _fiber(case), cfg).stack()
            steps = case["steps_per_span"]
        else:
            link = pb.LinkConfig(span=_fiber(case), num_spans=case["num_spans"], amp_gain_db=case["amp_gain_db"],
                                 amp_noise_figure_db=case["amp_noise_figure_db"],
                                 pol_rotation=case["pol_rotation"],
                                 center_wavelength_nm=case["center_wavelength_nm"])
            got = pb.propagate_link(_sig(x), link, cfg, rng=case["rng"]).stack()
            steps = case["steps_per_span"] * case["num_spans"]
        errs[name] = rel_l2(got, golden_fwd[f"{name}_out"])
    print("forward rel-L2:", {k: f"{v:.2e}" for k, v in errs.items()})
    for case in manifest_fwd["cases"]:
        steps = case["steps_per_span"] * case.get("num_spans", 1)
        assert errs[case["name"]] <= tol(steps), (case["name"], errs[case["name"]], tol(steps))
    assert _native.launch_count() > before


def test_amplifier_and_rotation_match_reference(golden_fwd):
    sig = _sig(golden_fwd["amp_in"])
    got = pb.amplify_with_ase(sig, 16.0, 5.0, 1550.0, rng=3).stack()
    assert rel_l2(got, golden_fwd["amp_out"]) <= 1e-6
    got = pb.amplify_with_ase(sig, 16.0, None).stack()
    assert rel_l2(got, golden_fwd["amp_quiet_out"]) <= 1e-6
    np.testing.assert_allclose(pb.haar_random_unitary(11), golden_fwd["haar11"], rtol=0, atol=1e-15)
    got = pb.random_polarization_rotation(sig, rng=5).stack()
    assert rel_l2(got, golden_fwd["rot_out"]) <= 1e-6
    with pytest.raises(ValueError):
        pb.amplify_with_ase(sig, -1.0, None)
    with pytest.raises(ValueError):
        pb.apply_jones_matrix(sig, np.eye(3))


@pytest.mark.parametrize("log_n", [8, 9, 10, 11, 12, 13, 14, 15, 17, 20])
def test_span_matches_oracle_across_lengths(log_n):
    # every layout boundary: block mode (<= 2^12), column tiles with N1 = 2^7 (2^13, 2^14) and 2^8
    n = 1 << log_n
    rng = np.random.default_rng(log_n)
    amp = math.sqrt(10 ** ((3.0 - 30) / 10) / 4.0)
    x = (amp * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n)))).astype(np.complex64)
    fiber = pb.FiberParams(beta2=-21.7, gamma=1.3, alpha_db_per_km=0.2, length=80.0)
    steps = 4
    got = pb.propagate_span(_sig(x), fiber, pb.SsfmStepConfig(steps)).stack()
    want = cp.span(x.astype(np.complex128), 56e9, -21.7, 1.3, 0.2, 80.0, steps)
    err = rel_l2(got, want)
    print(f"log_n={log_n} rel-L2 {err:.2e}")
    assert err <= tol(steps), err


def test_link_with_noise_and_rotation_matches_oracle_2_17():
    n = 1 << 17
    rng = np.random.default_rng(5)
    amp = math.sqrt(10 ** ((1.0 - 30) / 10) / 4.0)
    x = (amp * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n)))).astype(np.complex64)
    span = pb.FiberParams(beta2=-21.7, gamma=1.3, alpha_db_per_km=0.2, length=80.0)
    link = pb.LinkConfig(span=span, num_spans=3)
    got = pb.propagate_link(_sig(x), link, pb.SsfmStepConfig(6), rng=2024).stack()
    want = cp.link(x.astype(np.complex128), 56e9, -21.7, 1.3, 0.2, 80.0, 3, 6, rng=2024)
    assert rel_l2(got, want) <= tol(18)


def test_lossless_span_conserves_energy_and_dispersion_round_trips_2_21():
    # size-independent properties at the reference experiments' largest block (2^21)
    n = 1 << 21
    rng = np.random.default_rng(9)
    x = ((rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n))) * 0.01).astype(np.complex64)
    fwd = pb.FiberParams(beta2=-21.7, gamma=1.3, alpha_db_per_km=0.0, length=100.0)
    y = pb.propagate_span(_sig(x), fwd, pb.SsfmStepConfig(10)).stack()
    e0, e1 = np.sum(np.abs(x.astype(np.complex128)) ** 2), np.sum(np.abs(y.astype(np.complex128)) ** 2)
    assert abs(e1 / e0 - 1.0) <= 1e-5
    back = pb.FiberParams(beta2=21.7, gamma=0.0, alpha_db_per_km=0.0, length=100.0)
    lin = pb.propagate_span(_sig(x), pb.FiberParams(-21.7, 0.0, 0.0, 100.0), pb.SsfmStepConfig(5)).stack()
    z = pb.propagate_span(_sig(lin), back, pb.SsfmStepConfig(5)).stack()
    assert rel_l2(z, x) <= 2e-5


def test_batch_equals_single_runs():
    n = 1 << 12
    rng = np.random.default_rng(3)
    amp = math.sqrt(10 ** ((2.0 - 30) / 10) / 4.0)
    xs = (amp * (rng.normal(size=(3, 2, n)) + 1j * rng.normal(size=(3, 2, n)))).astype(np.complex64)
    span = pb.FiberParams(beta2=-21.7, gamma=1.3, alpha_db_per_km=0.2, length=80.0)
    link = pb.LinkConfig(span=span, num_spans=2)
    cfg = pb.SsfmStepConfig(5)
    got = pb.propagate_link_batch(xs, 56e9, link, cfg, [11, 12, 13])
    for i in range(3):
        one = pb.propagate_link(_sig(xs[i]), link, cfg, rng=11 + i).stack()
        np.testing.assert_array_equal(got[i], one.astype(np.complex64))


def test_simulator_validation():
    span = pb.FiberParams(beta2=-21.7, gamma=1.3, alpha_db_per_km=0.2, length=80.0)
    with pytest.raises(ValueError):
        pb.propagate_span(_sig(np.ones((2, 1000), np.complex64)), span, pb.SsfmStepConfig(2))
    with pytest.raises(ValueError):
        pb.propagate_link(_sig(np.ones((2, 1024), np.complex64)), pb.LinkConfig(span=span, num_spans=1),
                          pb.SsfmStepConfig(2), rng=np.random.default_rng(0))
    with pytest.raises(ValueError):
        pb.SsfmStepConfig(0)


def test_transpose_layout_matches_oracle_2_23():
    # n > 2^22 uses the transposed four-step layout (tile transposes); a 2-step span vs the oracle
    n = 1 << 23
    rng = np.random.default_rng(23)
    amp = math.sqrt(10 ** ((3.0 - 30) / 10) / 4.0)
    x = (amp * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n)))).astype(np.complex64)
    fiber = pb.FiberParams(beta2=-21.7, gamma=1.3, alpha_db_per_km=0.2, length=80.0)
    got = pb.propagate_span(_sig(x), fiber, pb.SsfmStepConfig(2)).stack()
    want = cp.span(x.astype(np.complex128), 56e9, -21.7, 1.3, 0.2, 80.0, 2)
    assert rel_l2(got, want) <= tol(2)


def test_forced_transpose_layout_equals_column_layout(tmp_path):
    # DBP_SIM_TRANSPOSE=1 selects the transposed layout at any n: same results to rounding
    import subprocess, sys, textwrap
    script = textwrap.dedent('''
        import sys, numpy as np
        sys.path.insert(0, sys.argv[1])
        import paper_1507_00921_b200 as pb
        rng = np.random.default_rng(4)
        x = ((rng.normal(size=(2, 1 << 16)) + 1j * rng.normal(size=(2, 1 << 16))) * 0.02).astype(np.complex64)
        f = pb.FiberParams(-21.7, 1.3, 0.2, 80.0)
        y = pb.propagate_span(pb.DualPolSignal(x[0], x[1], 56e9), f, pb.SsfmStepConfig(5)).stack()
        np.save(sys.argv[2], y)
    ''')
    import os
    root = str(Path(__file__).resolve().parent.parent)
    outs = []
    for flag in ("0", "1"):
        out = tmp_path / f"y{flag}.npy"
        env = dict(os.environ, DBP_SIM_TRANSPOSE=flag)
        subprocess.run([sys.executable, "-c", script, root, str(out)], check=True, env=env)
        outs.append(np.load(out))
    assert rel_l2(outs[0], outs[1]) <= tol(5)


def test_batch_device_list_equals_single_device():
    # devices=[...] splits independent waveforms across GPUs; on one GPU the list collapses
    n = 1 << 12
    rng = np.random.default_rng(8)
    xs = (0.02 * (rng.normal(size=(3, 2, n)) + 1j * rng.normal(size=(3, 2, n)))).astype(np.complex64)
    link = pb.LinkConfig(span=pb.FiberParams(-21.7, 1.3, 0.2, 80.0), num_spans=2)
    a = pb.propagate_link_batch(xs, 56e9, link, pb.SsfmStepConfig(3), [1, 2, 3])
    b = pb.propagate_link_batch(xs, 56e9, link, pb.SsfmStepConfig(3), [1, 2, 3], devices=[0, 0])
    np.testing.assert_array_equal(a, b)
