"""GPU parity: the fused CUDA path (through the C ABI) against the reference.

Tolerance (BASELINE north_star): relative L2 error <= 1e-5 per kept
overlap-save block against the float64 reference / oracle; identical QPSK
decisions; |dQ| <= 0.02 dB.  Bit-exact where the reference's own tests
demand exactness (identity coefficients == plain SSFM, jobs invariance) and
where the GPU design guarantees it (batching, block-range sharding).
"""

import warnings

import numpy as np
import pytest

import paper_1507_00921_b200 as pb
from paper_1507_00921_b200 import _native
from oracle import dbp_port, waveforms

from .helpers import case_config, port_config, quiet_link, rel_l2

pytestmark = pytest.mark.gpu

TOL_BLOCK = 1e-5   # per-block relative L2, north_star
STD = pb.FiberParams(beta2=-21.0, gamma=1.3, alpha_db_per_km=0.2, length=40.0)


def _run(x, case_or_cfg, rate=56e9, **kw):
    cfg = case_or_cfg
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return pb.backpropagate_batch(x, rate, cfg, **kw)


def _case_inputs(golden, case):
    name = case["name"]
    if case["signal"] == "white":
        x = golden[f"bp_{name}_in"]
        c = golden.get(f"bp_{name}_c")
        want = golden[f"bp_{name}_out"]
    else:
        x = golden["link_rx"]
        c = golden["link_c17"] if case["algorithm"] == "essfm" else None
        want = golden[f"link_{name}_out"]
    return x, c, want


def test_library_sees_a_device():
    assert _native.device_count() >= 1


def test_golden_cases_match_reference_per_block(golden, manifest):
    before = _native.launch_count()
    worst = {}
    for case in manifest["cases"]:
        x, c, want = _case_inputs(golden, case)
        cfg = case_config(case, c)
        got = _run(x, cfg)[0]
        errs = dbp_port.per_block_rel_l2(got, want, case["block_len"], case["overlap"])
        worst[case["name"]] = float(errs.max())
        assert errs.max() <= TOL_BLOCK, (case["name"], errs.max())
        # and against the oracle port on the same inputs
        port = dbp_port.backpropagate_arrays(x.astype(np.complex128), 56e9, port_config(cfg))
        assert dbp_port.per_block_rel_l2(got, port, case["block_len"], case["overlap"]).max() <= TOL_BLOCK
    assert _native.launch_count() > before  # the CUDA kernel ran
    print("worst per-block rel-L2:", worst)


@pytest.mark.parametrize("arrangement", pb.ARRANGEMENTS)
@pytest.mark.parametrize("steps,spans,side", [(1, 1, 16), (3, 2, 5), (5, 3, 32), (2, 1, 0)])
def test_identity_coefficients_bit_equal_plain(rng, arrangement, steps, spans, side):
    # test_dbp.py:90-114 / test_acceptance.py:207-234: worst == 0.0
    x = (rng.normal(size=(2, 1024)) + 1j * rng.normal(size=(2, 1024))).astype(np.complex64)
    plan = pb.OverlapPlan(512, 128)
    link = quiet_link(spans, STD)
    plain = _run(x, pb.DbpConfig("ssfm", plan, link, num_steps=steps, arrangement=arrangement))
    ident = _run(x, pb.DbpConfig("essfm", plan, link, num_steps=steps,
                                 coeffs=pb.EssfmCoefficients.identity(side), arrangement=arrangement))
    np.testing.assert_array_equal(plain, ident)


def test_ffe_is_linear(rng):
    # test_dbp.py:117-128
    plan = pb.OverlapPlan(1024, 256)
    cfg = pb.DbpConfig("ffe", plan, quiet_link(4, STD))
    a = (rng.normal(size=(2, 4096)) + 1j * rng.normal(size=(2, 4096))).astype(np.complex64)
    b = (rng.normal(size=(2, 4096)) + 1j * rng.normal(size=(2, 4096))).astype(np.complex64)
    mix = (2.0 * a - 0.5j * b).astype(np.complex64)
    oa, ob, om = _run(a, cfg)[0], _run(b, cfg)[0], _run(mix, cfg)[0]
    err = np.max(np.abs(om - (2.0 * oa - 0.5j * ob)))
    assert err < 1e-5 * np.max(np.abs(om))  # float32 arithmetic (reference: 1e-10 in float64)


@pytest.mark.parametrize("nc", [0, 1, 2, 4])
def test_substep_matches_reference(golden, nc):
    # test_dbp.py:47-57 geometry (N = 16): the sub-step operator runs in float64
    # (dbp_nonlinear_substep_c128), like the reference
    blk, c = golden[f"sub{nc}_in"], golden[f"sub{nc}_c"]
    got = pb.nonlinear_substep_essfm(blk, 1.7, 0.25, pb.EssfmCoefficients(c))
    want = golden[f"sub{nc}_out"]
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-13 * np.max(np.abs(want)))


@pytest.mark.parametrize("n", [3, 37, 100, 1000, 6000])
@pytest.mark.parametrize("nc", [0, 1, 17])
def test_substep_any_length_matches_oracle(rng, n, nc):
    # dbp.py:63-70 accepts any n > 2 N_c (not only powers of two)
    if n <= 2 * nc:
        with pytest.raises(ValueError, match="too short"):
            pb.nonlinear_substep_essfm(np.ones((2, n), complex), 1.3, 1.0, pb.EssfmCoefficients.identity(nc))
        return
    blk = 0.05 * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n)))
    c = rng.normal(size=nc + 1) * 0.1
    c[0] = 1.0
    got = pb.nonlinear_substep_essfm(blk, -1.3, 800.0, pb.EssfmCoefficients(c))
    want = dbp_port.rotate_essfm(blk, -1.3, 800.0, c)
    assert rel_l2(got, want) < 1e-13


def test_substep_ssfm_equals_identity_essfm(rng):
    blk = rng.normal(size=(2, 64)) + 1j * rng.normal(size=(2, 64))
    a = pb.nonlinear_substep_essfm(blk, 1.3, 18.2, pb.EssfmCoefficients.identity(6))
    b = pb.nonlinear_substep_ssfm(blk, 1.3, 18.2)
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("n_blk", [256, 1024, 2048, 8192])
@pytest.mark.parametrize("nc", [1, 3, 9, 13, 17, 24, 32, 33, 64])
def test_fir_paths_match_oracle(rng, n_blk, nc):
    # every intensity-FIR path of the block kernel inside the DBP program: the
    # folded form (N <= 512), the streamed direct form (N >= 1024) for the
    # compiled N_c in {1, 9, 17, 32, 33}, and fir8_generic (kProgGenericFir) for
    # the others; random taps, strong nonlinearity (ESSFM N_s = 1 symmetric)
    m = n_blk // 4
    n = 3 * (n_blk - m) + 55
    x = (0.03 * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n)))).astype(np.complex64)
    c = rng.normal(size=nc + 1) * 0.1
    c[0] = 1.0
    span = pb.FiberParams(-21.0, 1.3, 0.2, 80.0)
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(n_blk, m), quiet_link(40, span), num_steps=1,
                       coeffs=pb.EssfmCoefficients(c))
    got = _run(x[None], cfg)[0]
    want = dbp_port.backpropagate_arrays(x.astype(np.complex128), 56e9, port_config(cfg))
    assert dbp_port.per_block_rel_l2(got, want, n_blk, m).max() <= TOL_BLOCK


def test_process_blocks_matches_captured_closure(golden, manifest):
    torch = pytest.importorskip("torch")
    for case in manifest["cases"]:
        if case["signal"] != "link":
            continue
        name = case["name"]
        c = golden["link_c17"] if case["algorithm"] == "essfm" else None
        cfg = case_config(case, c)
        eng = pb.get_engine(cfg, 56e9, 0)
        blocks = np.ascontiguousarray(golden[f"link_{name}_blk_in"].astype(np.complex64))
        d_in = torch.from_numpy(blocks.view(np.float32)).cuda()
        d_out = torch.empty_like(d_in)
        eng.native.process_blocks(d_in.data_ptr(), d_out.data_ptr(), blocks.shape[0])
        torch.cuda.synchronize()
        got = d_out.cpu().numpy().view(np.complex64)
        want = golden[f"link_{name}_blk_out"]
        for b in range(blocks.shape[0]):
            assert rel_l2(got[b], want[b]) <= TOL_BLOCK, (name, b, rel_l2(got[b], want[b]))


def test_batch_items_bit_equal_single(rng):
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(2048, 700), quiet_link(4, STD),
                       coeffs=pb.EssfmCoefficients(waveforms.gaussian_coeffs(17)))
    x = (0.03 * (rng.normal(size=(5, 2, 20000)) + 1j * rng.normal(size=(5, 2, 20000)))).astype(np.complex64)
    batch = _run(x, cfg)
    for i in range(5):
        np.testing.assert_array_equal(batch[i], _run(x[i], cfg)[0])


@pytest.mark.parametrize("n", [700, 1348, 1349, 2696, 4100])
def test_batch_item_index_every_blocks_per_item(rng, n):
    # blocks -> (item, block) (the kernel's multiply-high division): 1, 1, 2, 2
    # and 4 blocks per item (step 1348), batch of 7, each item == its single run
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(2048, 700), quiet_link(4, STD),
                       coeffs=pb.EssfmCoefficients(waveforms.gaussian_coeffs(17)))
    x = (0.03 * (rng.normal(size=(7, 2, n)) + 1j * rng.normal(size=(7, 2, n)))).astype(np.complex64)
    batch = _run(x, cfg)
    for i in range(7):
        np.testing.assert_array_equal(batch[i], _run(x[i], cfg)[0])


@pytest.mark.parametrize("parts", [2, 3, 8])
def test_block_range_shards_bit_equal_whole(rng, parts):
    # multi-GPU contract: chunks on multiples of N - M are bitwise equal
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(2048, 700), quiet_link(40, STD),
                       coeffs=pb.EssfmCoefficients(waveforms.gaussian_coeffs(17)))
    x = (0.03 * (rng.normal(size=(1, 2, 100000)) + 1j * rng.normal(size=(1, 2, 100000)))).astype(np.complex64)
    whole = _run(x, cfg)
    eng = pb.get_engine(cfg, 56e9, 0)
    out = np.zeros_like(x)
    for b0, b1 in pb.shard_blocks(eng.num_blocks(x.shape[-1]), parts):
        part = eng.run_host(x, block_range=(b0, b1))
        lo, hi = cfg.plan.output_span(b0, b1, x.shape[-1])
        out[..., lo:hi] = part[..., lo:hi]
    np.testing.assert_array_equal(out, whole)


def test_chunk_mode_bit_equal_whole(rng):
    torch = pytest.importorskip("torch")
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(2048, 700), quiet_link(40, STD),
                       coeffs=pb.EssfmCoefficients(waveforms.gaussian_coeffs(9)), arrangement="linear-first")
    n = 50000
    x = (0.03 * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n)))).astype(np.complex64)
    whole = _run(x, cfg)[0]
    eng = pb.get_engine(cfg, 56e9, 0)
    nb = eng.num_blocks(n)
    for b0, b1 in [(0, 5), (5, 17), (17, nb)]:
        lo, hi = cfg.plan.input_span(b0, b1)
        span = np.ascontiguousarray(pb.framing.gather_span(x, lo, hi))
        olo, ohi = cfg.plan.output_span(b0, b1, n)
        d_in = torch.from_numpy(span.view(np.float32)).cuda()
        d_out = torch.zeros((2, (ohi - olo) * 2), dtype=torch.float32, device="cuda")
        eng.native.run_chunk(d_in.data_ptr(), d_out.data_ptr(), n, 1, b0, b1, hi - lo, ohi - olo)
        torch.cuda.synchronize()
        got = d_out.cpu().numpy().view(np.complex64)
        np.testing.assert_array_equal(got, whole[:, olo:ohi])


def test_large_item_host_chunking_bit_equal(rng):
    # item larger than a staging slot -> dbp_run_host's halo'd block-range path
    cfg = pb.DbpConfig("ssfm", pb.OverlapPlan(1024, 256), quiet_link(8, STD), num_steps=3)
    n = 300000
    x = (0.03 * (rng.normal(size=(1, 2, n)) + 1j * rng.normal(size=(1, 2, n)))).astype(np.complex64)
    whole = _run(x, cfg)
    eng = pb.DbpEngine(cfg, 56e9, 0)
    eng.native.set_staging(1 << 20)   # 256 KiB per slot buffer < 4.8 MB item
    chunked = eng.run_host(x)
    eng.close()
    np.testing.assert_array_equal(chunked, whole)


def test_jobs_bit_identical(rng):
    x = (rng.normal(size=8192) + 1j * rng.normal(size=8192))
    sig = pb.DualPolSignal(x, x[::-1], 56e9)
    cfg = pb.DbpConfig("ssfm", pb.OverlapPlan(2048, 512), quiet_link(2, STD), num_steps=4)
    a = pb.backpropagate(sig, cfg, jobs=1)
    b = pb.backpropagate(sig, cfg, jobs=3)
    np.testing.assert_array_equal(a.stack(), b.stack())
    assert a.x.dtype == np.complex128 and len(a) == len(sig) and a.sample_rate == sig.sample_rate
    with pytest.raises(ValueError):
        pb.backpropagate(sig, cfg, jobs=0)


def test_warns_on_short_overlap(rng):
    # test_dbp.py:203-214
    x = rng.normal(size=4096) + 0j
    sig = pb.DualPolSignal(x, x, 56e9)
    with pytest.warns(UserWarning, match="channel memory"):
        pb.backpropagate(sig, pb.DbpConfig("ffe", pb.OverlapPlan(1024, 256), quiet_link(80, STD)))
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        pb.backpropagate(sig, pb.DbpConfig("ffe", pb.OverlapPlan(2048, 512), quiet_link(1, STD)))


@pytest.mark.parametrize("n_total", [1, 5, 1536, 1537, 4096, 5000])
def test_ffe_identity_filter_edge_lengths(rng, n_total):
    # zero dispersion: the block engine must reproduce any input length (test_spectral.py:72-77)
    span = pb.FiberParams(beta2=0.0, gamma=1.3, alpha_db_per_km=0.2, length=40.0)
    cfg = pb.DbpConfig("ffe", pb.OverlapPlan(2048, 512), quiet_link(1, span))
    x = (rng.normal(size=(2, n_total)) + 1j * rng.normal(size=(2, n_total))).astype(np.complex64)
    got = _run(x, cfg)[0]
    np.testing.assert_allclose(got, x, rtol=0, atol=2e-6 * np.max(np.abs(x)))


def test_decisions_and_q_match_oracle(golden, manifest):
    symbols = golden["link_tx_symbols"]
    ref_bits = waveforms.hard_decisions(symbols)
    for case in manifest["cases"]:
        if case["signal"] != "link" or case["name"] not in ("c0_sym", "c0_lf", "c2_ssfm20"):
            continue
        x, c, want = _case_inputs(golden, case)
        got = _run(x, case_config(case, c))[0]
        bits_gpu = waveforms.hard_decisions(waveforms.receive_symbols(got))
        bits_ref = waveforms.hard_decisions(waveforms.receive_symbols(want))
        assert np.array_equal(bits_gpu, bits_ref), case["name"]
        q_gpu = waveforms.q_factor_db(bits_gpu, ref_bits)
        q_ref = waveforms.q_factor_db(bits_ref, ref_bits)
        assert q_gpu == q_ref or abs(q_gpu - q_ref) <= 0.02


def test_reference_receiver_on_gpu_dbp_output(golden, manifest, golden_rx, manifest_rx):
    # identical qpsk_decide decisions and |dQ| <= 0.02 dB after the reference's own Rx
    # chain (butterfly_equalize -> carrier_recover -> qpsk_decide -> measure_ber, cli.py:677-685).
    # Reference side: the reference DBP output through the reference modem (golden_rx "link").
    # GPU side: the GPU DBP of the same received waveform through the GPU receiver (rx.py).
    case = next(c for c in manifest["cases"] if c["name"] == "c0_sym")
    ref_case = next(c for c in manifest_rx["cases"] if c["name"] == "link")
    x, c, _ = _case_inputs(golden, case)
    got = _run(x, case_config(case, c))[0]
    sym = golden["link_tx_symbols"]
    eq = pb.butterfly_equalize(pb.DualPolSignal(got[0], got[1], 56e9))
    rec = pb.carrier_recover(eq.stack(), 28e9, reference=sym)
    dec = pb.qpsk_decide(rec)
    np.testing.assert_array_equal(dec, golden_rx["link_dec"])
    met = pb.measure_ber(dec, pb.qpsk_decide(sym), skip=ref_case["skip_bits"])
    assert met.ber == ref_case["ber"] and met.bits_counted == ref_case["bits_counted"]
    assert abs(met.q_factor_db - ref_case["q_db"]) <= 0.02


def test_full_size_properties(rng):
    # BASELINE config-3 item size (2^18 samples): linearity of FFE and ESSFM(identity) == SSFM
    n = 1 << 18
    x = (0.03 * (rng.normal(size=(2, 2, n)) + 1j * rng.normal(size=(2, 2, n)))).astype(np.complex64)
    link = quiet_link(40, pb.FiberParams(-21.6826, 1.3, 0.2, 80.0))
    plan = pb.OverlapPlan(2048, 700)
    ffe = pb.DbpConfig("ffe", plan, link)
    a, b = _run(x, ffe)
    s = _run((x[0] + x[1])[None].astype(np.complex64), ffe)[0]
    assert rel_l2(s, a + b) < 1e-5
    plain = _run(x, pb.DbpConfig("ssfm", plan, link, num_steps=1))
    ident = _run(x, pb.DbpConfig("essfm", plan, link, coeffs=pb.EssfmCoefficients.identity(17)))
    np.testing.assert_array_equal(plain, ident)
    # energy: the inverse-dispersion filter is unitary up to framing
    assert abs(np.sum(np.abs(a) ** 2) / np.sum(np.abs(x[0]) ** 2) - 1.0) < 0.05


@pytest.mark.parametrize("power_dbm", [-4.0, 0.0, 4.0])
def test_config2_ssfm20_power_sweep(power_dbm):
    # BASELINE configs[2]: 20-step SSFM (dispersion then rotation), gamma' = 8/9 * 1.3,
    # launch power -4..+4 dBm; per-block rel-L2 <= 1e-5 (multi-step programs use the
    # polynomial sincos -- the SFU's correlated error would exceed the bar at +4 dBm)
    beta2 = waveforms.d_to_beta2(17.0)
    tx, _ = waveforms.qpsk_rrc(2 ** 12, 2, 0.1, seed=4, power_dbm=power_dbm)
    rx = waveforms.forward_link(tx, 56e9, beta2, 1.3 * 8 / 9, 0.2, 80.0, 40, 4).astype(np.complex64)
    span = pb.FiberParams(beta2, 1.3 * 8 / 9, 0.2, 80.0)
    cfg = pb.DbpConfig("ssfm", pb.OverlapPlan(2048, 700), quiet_link(40, span), num_steps=20,
                       arrangement="linear-first")
    got = _run(rx, cfg)[0]
    want = dbp_port.backpropagate_arrays(rx.astype(np.complex128), 56e9, port_config(cfg))
    assert dbp_port.per_block_rel_l2(got, want, 2048, 700).max() <= TOL_BLOCK


def test_coefficient_training_matches_reference(golden):
    # the reference's Gauss-Newton fit (train.py:86-188) with every
    # coefficient batch evaluated in one launch; float32 central differences
    link = quiet_link(40, pb.FiberParams(waveforms.d_to_beta2(17.0), 1.3, 0.2, 80.0))
    rx = golden["link_rx"]
    sig = pb.DualPolSignal(rx[0], rx[1], 56e9)
    tcfg = pb.TrainConfig(n_coeffs=4, target_steps_per_span=2, train_samples=8192, max_iterations=6)
    dcfg = pb.DbpConfig("essfm", pb.OverlapPlan(2048, 700), link, coeffs=pb.EssfmCoefficients.identity(4))
    res = pb.optimize_coefficients(sig, dcfg, tcfg)
    ref_initial, ref_final, ref_iters, _ = golden["train_mse"]
    print("gpu", res.initial_mse, res.final_mse, res.iterations, res.coefficients.c)
    print("ref", ref_initial, ref_final, ref_iters, golden["train_c"])
    assert abs(res.initial_mse - ref_initial) <= 1e-4 * ref_initial
    assert res.final_mse <= ref_final * 1.01
    np.testing.assert_allclose(res.coefficients.c, golden["train_c"], rtol=0, atol=2e-2)


def test_coeff_batch_items_match_single_runs(rng):
    # per-item coefficient sets (one launch) == separate ESSFM runs with each set
    link = quiet_link(8, STD)
    plan = pb.OverlapPlan(1024, 256)
    x = (0.03 * (rng.normal(size=(2, 6000)) + 1j * rng.normal(size=(2, 6000)))).astype(np.complex64)
    sets = np.stack([waveforms.gaussian_coeffs(5, w) for w in (1.0, 2.0, 3.5)])
    eng = pb.get_engine(pb.DbpConfig("essfm", plan, link, num_steps=2,
                                     coeffs=pb.EssfmCoefficients.identity(5)), 56e9, 0)
    out = np.empty((3, 2, 6000), dtype=np.complex64)
    with eng.native.lock:
        eng.native.set_coeff_batch(sets)
        eng.native.run_host_coeff_batch(np.ascontiguousarray(x), out, 6000)
    for i in range(3):
        single = _run(x, pb.DbpConfig("essfm", plan, link, num_steps=2, coeffs=pb.EssfmCoefficients(sets[i])))[0]
        assert rel_l2(out[i], single) < 1e-6


def test_random_configurations_match_oracle():
    # seeded sweep of random geometries / programs (cf. the reference's hypothesis
    # properties, test_dbp.py:90-114): every block length 16..8192, any overlap,
    # ragged lengths (n < N included), 1..6 steps, gains != 1, every arrangement,
    # N_c up to min(64, (N-1)/2) -- per-block rel-L2 <= 1e-5 against the oracle
    gen = np.random.default_rng(2718)
    for case in range(40):
        logn = int(gen.integers(4, 14))
        n_blk = 1 << logn
        m = int(gen.integers(0, n_blk))
        n = int(gen.integers(1, 3 * n_blk + 2))
        alg = ("ffe", "ssfm", "essfm")[case % 3]
        steps = int(gen.integers(1, 7))
        spans = int(gen.integers(1, 6))
        arr = pb.ARRANGEMENTS[int(gen.integers(0, 3))]
        coeffs = None
        if alg == "essfm":
            nc = int(gen.integers(0, min(64, (n_blk - 1) // 2) + 1))
            c = gen.normal(size=nc + 1) * 0.1
            c[0] = 1.0
            coeffs = pb.EssfmCoefficients(c)
        span = pb.FiberParams(-21.68, 1.3, 0.2, float(gen.uniform(20.0, 100.0)))
        cfg = pb.DbpConfig(alg, pb.OverlapPlan(n_blk, m), quiet_link(spans, span), num_steps=steps,
                           coeffs=coeffs, arrangement=arr)
        x = (0.02 * (gen.normal(size=(2, n)) + 1j * gen.normal(size=(2, n)))).astype(np.complex64)
        got = _run(x, cfg)[0]
        want = dbp_port.backpropagate_arrays(x.astype(np.complex128), 56e9, port_config(cfg))
        err = dbp_port.per_block_rel_l2(got, want, n_blk, m).max()
        assert err <= TOL_BLOCK, (case, alg, n_blk, m, n, steps, spans, arr, err)


def test_integration_stub_runs_and_matches(golden, manifest, tmp_path):
    # the ctypes binding INTEGRATION.md shows a fiberdbp maintainer adding, executed verbatim
    # (its two relative imports pointed at this package's equivalents) against the same case
    import re
    from pathlib import Path
    text = (Path(__file__).resolve().parent.parent / "INTEGRATION.md").read_text()
    stub = re.search(r"```python\n(import ctypes, numpy as np.*?)```", text, re.S).group(1)
    stub = stub.replace("from .dbp import _reverse_step_schedule",
                        "from paper_1507_00921_b200.backprop import _reverse_step_schedule")
    stub = stub.replace("from .spectral import fft_frequencies", "from paper_1507_00921_b200 import fft_frequencies")
    stub = stub.replace('ctypes.CDLL("libdbp_b200.so")', f'ctypes.CDLL("{_native.LIB_PATH}")')
    ns = {}
    exec(compile(stub, "INTEGRATION.md", "exec"), ns)
    case = next(c for c in manifest["cases"] if c["name"] == "c0_sym")
    x, c, want = _case_inputs(golden, case)
    cfg = case_config(case, c)
    got = ns["backpropagate_b200"](pb.DualPolSignal(x[0], x[1], 56e9), cfg).stack()
    errs = dbp_port.per_block_rel_l2(got, want, case["block_len"], case["overlap"])
    assert errs.max() <= TOL_BLOCK
    np.testing.assert_array_equal(got.astype(np.complex64), _run(x, cfg)[0])


@pytest.mark.gpu
@pytest.mark.parametrize("n_blk,m", [(4096, 700), (4096, 1400), (8192, 1024)])
def test_ffe_kernel_large_blocks_match_oracle(n_blk, m):
    # the FFE-only kernel instantiation (launch.h, N >= 4096): whole-signal cyclic
    # framing with edge blocks, a ragged length and a 2-item batch, per-block
    # rel-L2 <= 1e-5 against the oracle (dbp.py:185-191) and batch == single runs
    gen = np.random.default_rng(n_blk + m)
    span = pb.FiberParams(-21.68, 1.3, 0.2, 80.0)
    cfg = pb.DbpConfig("ffe", pb.OverlapPlan(n_blk, m), quiet_link(40, span))
    n = 5 * (n_blk - m) + 123
    x = (0.02 * (gen.normal(size=(2, 2, n)) + 1j * gen.normal(size=(2, 2, n)))).astype(np.complex64)
    got = _run(x, cfg)
    for i in range(2):
        want = dbp_port.backpropagate_arrays(x[i].astype(np.complex128), 56e9, port_config(cfg))
        assert dbp_port.per_block_rel_l2(got[i], want, n_blk, m).max() <= TOL_BLOCK
        np.testing.assert_array_equal(got[i], _run(x[i:i + 1], cfg)[0])


@pytest.mark.gpu
@pytest.mark.parametrize("alg,n_blk,m,steps,arr", [
    ("ssfm", 2048, 700, 20, "linear-first"), ("ssfm", 2048, 700, 3, "symmetric"),
    ("essfm0", 2048, 700, 1, "symmetric"), ("ssfm", 4096, 1400, 4, "nonlinear-first"),
    ("ssfm", 8192, 1024, 20, "linear-first")])
def test_nofir_kernel_matches_oracle(alg, n_blk, m, steps, arr):
    # the no-FIR split-step instantiation (launch.h, N >= 2048: SSFM and ESSFM
    # with N_c = 0): whole-signal framing with edge blocks, ragged length, 2-item
    # batch; per-block rel-L2 <= 1e-5 against the oracle (dbp.py:193-235) and
    # batch == single runs
    gen = np.random.default_rng(n_blk + steps)
    span = pb.FiberParams(-21.68, 1.3, 0.2, 80.0)
    coeffs = pb.EssfmCoefficients(np.array([0.9])) if alg == "essfm0" else None
    cfg = pb.DbpConfig("essfm" if alg == "essfm0" else "ssfm", pb.OverlapPlan(n_blk, m), quiet_link(40, span),
                       num_steps=steps, coeffs=coeffs, arrangement=arr)
    n = 4 * (n_blk - m) + 77
    x = (0.03 * (gen.normal(size=(2, 2, n)) + 1j * gen.normal(size=(2, 2, n)))).astype(np.complex64)
    got = _run(x, cfg)
    for i in range(2):
        want = dbp_port.backpropagate_arrays(x[i].astype(np.complex128), 56e9, port_config(cfg))
        assert dbp_port.per_block_rel_l2(got[i], want, n_blk, m).max() <= TOL_BLOCK
        np.testing.assert_array_equal(got[i], _run(x[i:i + 1], cfg)[0])


@pytest.mark.parametrize("batch", [1, 3])
def test_multi_device_split_bit_equal(rng, batch):
    # backpropagate_batch(devices=[...]) on one GPU listed twice: B < #devices splits the
    # waveform by block range (each shard staged as its halo'd span only), B >= #devices
    # by whole waveforms; both must equal the single-device run bit for bit
    # (blocks are independent, spectral.py:100-101)
    n = 7 * 1348 + 77
    x = (0.02 * (rng.normal(size=(batch, 2, n)) + 1j * rng.normal(size=(batch, 2, n)))).astype(np.complex64)
    span = pb.FiberParams(-21.6826, 1.3, 0.2, 80.0)
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(2048, 700), quiet_link(40, span), num_steps=1,
                       coeffs=pb.EssfmCoefficients(waveforms.gaussian_coeffs(17)))
    one = _run(x, cfg)
    for devs in ([0, 0], [0, 0, 0]):
        np.testing.assert_array_equal(_run(x, cfg, devices=devs), one)
    # and through the drop-in call
    sig = pb.DualPolSignal(x[0, 0], x[0, 1], 56e9)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        out = pb.backpropagate(sig, cfg, devices=[0, 0])
    np.testing.assert_array_equal(out.stack(), one[0])


@pytest.mark.parametrize("batch,n_total", [(1, (1 << 16)), (1, (1 << 19) + 5), (3, (1 << 18) + 11), (5, (1 << 16) + 123), (4, 1 << 18)])
def test_pageable_host_rows_bit_equal_pinned(rng, batch, n_total):
    # dbp_run_host on ordinary numpy (pageable) rows goes through pinned staging on the host
    # pool, whole items or block-range chunks with halos (run_host_staged); on page-locked
    # buffers it copies directly: same bits either way (spectral.py:100-101, blocks independent)
    from paper_1507_00921_b200 import _native
    span = pb.FiberParams(-21.6826, 1.3, 0.2, 80.0)
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(2048, 700), quiet_link(40, span), num_steps=1,
                       coeffs=pb.EssfmCoefficients(waveforms.gaussian_coeffs(17)))
    x = (0.02 * (rng.normal(size=(batch, 2, n_total)) + 1j * rng.normal(size=(batch, 2, n_total)))).astype(np.complex64)
    eng = pb.get_engine(cfg, 56e9)
    got = np.empty_like(x)
    eng.run_host(x, got)
    pin_in, pin_out = _native.PinnedBuffer(x.shape), _native.PinnedBuffer(x.shape)
    try:
        pin_in.array[...] = x
        eng.run_host(pin_in.array, pin_out.array)
        np.testing.assert_array_equal(got, pin_out.array)
        # mixed: pageable in, pinned out
        pin_out.array[...] = 0
        eng.run_host(x, pin_out.array)
        np.testing.assert_array_equal(got, pin_out.array)
    finally:
        pin_in.free()
        pin_out.free()


def test_in_place_host_rows(rng):
    # dbp_run_host in place (h_out == h_in) keeps the plain whole-item path and its result;
    # dbp_backpropagate_c128 refuses result rows that overlap its input (spectral.py:129:
    # the reference never mutates its input)
    n_total = (1 << 18) + 77
    span = pb.FiberParams(-21.6826, 1.3, 0.2, 80.0)
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(2048, 700), quiet_link(40, span), num_steps=1,
                       coeffs=pb.EssfmCoefficients(waveforms.gaussian_coeffs(17)))
    x = (0.02 * (rng.normal(size=(1, 2, n_total)) + 1j * rng.normal(size=(1, 2, n_total)))).astype(np.complex64)
    eng = pb.get_engine(cfg, 56e9)
    want = eng.run_host(x)
    buf = x.copy()
    eng.run_host(buf, buf)
    np.testing.assert_array_equal(buf, want)
    xs = x[0].astype(np.complex128)
    other = np.empty(n_total, np.complex128)
    with eng.native.lock:
        with pytest.raises(ValueError, match="overlap"):
            eng.native.backpropagate_c128(xs[0], xs[1], xs[0], other)
        with pytest.raises(ValueError, match="overlap"):
            eng.native.backpropagate_c128(xs[0], xs[1], other, other)


def test_dropin_results_are_distinct_arrays_across_calls(rng):
    # the recycled output rows (backprop._RowArena) never alias a result the caller still
    # holds, and a recycled row is fully rewritten (spectral.py:145: the output is a new array)
    n_total = 1 << 16
    span = pb.FiberParams(-21.6826, 1.3, 0.2, 80.0)
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(2048, 700), quiet_link(40, span), num_steps=1,
                       coeffs=pb.EssfmCoefficients(waveforms.gaussian_coeffs(17)))
    sigs = [pb.DualPolSignal(*(0.02 * (rng.normal(size=(2, n_total)) + 1j * rng.normal(size=(2, n_total)))), 56e9)
            for _ in range(3)]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        kept = [pb.backpropagate(s, cfg) for s in sigs]
        copies = [k.stack() for k in kept]
        for _ in range(4):                                  # dropped results free their rows ...
            pb.backpropagate(sigs[1], cfg)
        again = pb.backpropagate(sigs[0], cfg)              # ... and a recycled row holds only the new result
    rows = [r for k in kept + [again] for r in (k.x, k.y)]
    for i in range(len(rows)):
        for j in range(i + 1, len(rows)):
            assert not np.shares_memory(rows[i], rows[j])
    for k, c in zip(kept, copies):
        np.testing.assert_array_equal(k.stack(), c)         # untouched by the later calls
    np.testing.assert_array_equal(again.stack(), copies[0])


@pytest.mark.parametrize("n_total", [1, 5, 1348, 4099, (1 << 17), (1 << 22) + 777])
def test_dropin_complex128_path_bit_equal(rng, n_total):
    # backpropagate(sig, cfg) on complex128 rows (dbp_backpropagate_c128: host-thread casts,
    # pinned staging, block-range chunks with halos above 2^21 samples) == the batch path on
    # the complex64 cast, bit for bit, returned as complex128 (sigkit.py:56-68)
    x = 0.02 * (rng.normal(size=(2, n_total)) + 1j * rng.normal(size=(2, n_total)))
    span = pb.FiberParams(-21.6826, 1.3, 0.2, 80.0)
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(2048, 700), quiet_link(40, span), num_steps=1,
                       coeffs=pb.EssfmCoefficients(waveforms.gaussian_coeffs(17)))
    sig = pb.DualPolSignal(x[0], x[1], 56e9)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        out = pb.backpropagate(sig, cfg)
    assert out.x.dtype == np.complex128 and len(out) == n_total and out.sample_rate == 56e9
    want = _run(x.astype(np.complex64)[None], cfg)[0]
    np.testing.assert_array_equal(out.stack(), want.astype(np.complex128))


def test_failed_reconfiguration_leaves_the_plan_intact(rng):
    # a rejected dbp_plan_set_steps / set_linear must not leave a
    # half-updated plan (new program with the old schedule, new K with old K^1/2)
    span = pb.FiberParams(-21.6826, 1.3, 0.2, 80.0)
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(1024, 256), quiet_link(10, span), num_steps=2,
                       coeffs=pb.EssfmCoefficients(waveforms.gaussian_coeffs(9)))
    eng = pb.DbpEngine(cfg, 56e9, 0)
    x = (0.02 * (rng.normal(size=(1, 2, 5000)) + 1j * rng.normal(size=(1, 2, 5000)))).astype(np.complex64)
    before = eng.run_host(x)
    sched = eng.schedule
    bad = np.full(10, np.nan)
    with pytest.raises(ValueError, match="finite"):
        eng.native.set_steps("essfm", "linear-first", [w for _, w, _ in sched], [g for _, _, g in sched],
                             -1.3, bad)
    with pytest.raises(ValueError, match="finite"):
        eng.native.set_steps("ssfm", "symmetric", [np.nan] * 2, [1.0, 1.0], -1.3)
    with pytest.raises(ValueError, match="finite"):
        eng.native.set_linear(np.full(1024, np.nan + 0j), np.ones(1024, complex))
    np.testing.assert_array_equal(eng.run_host(x), before)
    eng.close()


@pytest.mark.parametrize("alg,n_blk,m,n", [
    ("ffe", 2048, 700, 1 << 17), ("ffe", 4096, 1400, 1 << 17), ("ffe", 4096, 4051, 10294),
    ("ffe", 4096, 4032, 1 << 15), ("essfm", 2048, 700, 1 << 17), ("ssfm", 4096, 1400, 1 << 17)])
def test_tma_and_split_barrier_paths_deterministic(alg, n_blk, m, n):
    # Regression for a write-after-read race of round 2: with the FFE block input
    # arriving through the exchange planes (TMA bulk load) under split (mbarrier)
    # write-after-read barriers (N = 2048, 4096), each warp's initial arrival was
    # made at kernel start, so a fast warp could write its first exchange over
    # rows a slow warp had not read yet (seen by the randomised sweep as a 6e-3
    # block error at N = 4096, M = 4051, and as run-to-run differences).  A batch
    # large enough to keep every SM busy is run three times and must reproduce
    # itself bit for bit; its first item must match the oracle per block.
    gen = np.random.default_rng(n_blk + m + n)
    span = pb.FiberParams(-21.68, 1.3, 0.2, 80.0)
    coeffs = pb.EssfmCoefficients(np.r_[1.0, 0.05 * gen.normal(size=17)]) if alg == "essfm" else None
    cfg = pb.DbpConfig(alg, pb.OverlapPlan(n_blk, m), quiet_link(8, span), num_steps=4 if alg != "ffe" else 1,
                       coeffs=coeffs, arrangement="symmetric")
    batch = max(2, (1 << 22) // n)
    x = (0.02 * (gen.normal(size=(batch, 2, n)) + 1j * gen.normal(size=(batch, 2, n)))).astype(np.complex64)
    first = _run(x, cfg)
    for _ in range(2):
        np.testing.assert_array_equal(_run(x, cfg), first)
    want = dbp_port.backpropagate_arrays(x[0].astype(np.complex128), 56e9, port_config(cfg))
    assert dbp_port.per_block_rel_l2(first[0], want, n_blk, m).max() <= TOL_BLOCK


def test_warp_ffe_kernel_matches_oracle_in_subprocess():
    # The warp-resident FFE kernel (dbp_warp_kernel.cuh, off by default) is
    # selected per process by env DBP_WARP_FFE=1: run the FFE parity tests --
    # golden FFE cases, the large-block FFE cases, the determinism repeats --
    # in a child process with it on.
    import os
    import subprocess
    import sys
    from pathlib import Path

    env = dict(os.environ, DBP_WARP_FFE="1")
    root = Path(__file__).resolve().parent.parent
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
                          "tests/test_gpu_parity.py", "-k",
                          "golden_cases or ffe_kernel_large or (deterministic and ffe) or ffe_is_linear "
                          "or ffe_identity_filter"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]


def test_polsplit_pairs_match_oracle_in_subprocess():
    # N = 8192 polarisation-split pairs (launch.h polsplit_mode): the FFE program
    # runs them by default; DBP_POLSPLIT=1 forces them for every program (the
    # split-step programs as 2-CTA clusters exchanging |v|^2 through distributed
    # shared memory).  Run the N = 8192 parity tests with them forced.
    import os
    import subprocess
    import sys
    from pathlib import Path

    env = dict(os.environ, DBP_POLSPLIT="1", DBP_R2="0")
    root = Path(__file__).resolve().parent.parent
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
                          "tests/test_gpu_parity.py", "-k",
                          "golden_cases or (ffe_kernel_large and 8192) or (nofir and 8192) "
                          "or (fir_paths and 8192) or random_configurations"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]


def test_r2_off_and_on_everywhere_match_oracle_in_subprocess():
    # N = 8192 split-step programs run the radix-2-around-4096 kernel
    # (dbp_r2_kernel.cuh) by default.  DBP_R2=0 brings back the pol-pair block
    # kernel, DBP_R2=1 also routes the FFE program through R2: run the N = 8192
    # parity tests both ways so every instantiation stays checked.
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    for val in ("0", "1"):
        env = dict(os.environ, DBP_R2=val)
        res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
                              "tests/test_gpu_parity.py", "-k",
                              "golden_cases or (ffe_kernel_large and 8192) or (nofir and 8192) "
                              "or (fir_paths and 8192) or random_configurations"],
                             cwd=root, env=env, capture_output=True, text=True, timeout=900)
        assert res.returncode == 0, (val, res.stdout[-3000:] + res.stderr[-2000:])


def test_r2t_matches_oracle_in_subprocess():
    # N = 8192 with the parked subsequence in tensor memory, two CTAs per SM
    # (dbp_r2t_kernel.cuh).  DBP_R2T=2 routes every program (FFE included)
    # through it: run the N = 8192 parity tests that way.
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, DBP_R2T="2")
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
                          "tests/test_gpu_parity.py", "-k",
                          "golden_cases or (ffe_kernel_large and 8192) or (nofir and 8192) "
                          "or (fir_paths and 8192) or random_configurations"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]


# ---------------------------------------------------------------------------
# Block lengths outside the fused kernel's [16, 8192]: the float64
# multi-kernel path (csrc/dbp_general.cuh).  The reference accepts any
# power-of-two block (spectral.py:72-76); same API, same parity bar.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n_blk,m", [(1, 0), (2, 1), (4, 2), (8, 3), (16384, 2048), (32768, 700)])
@pytest.mark.parametrize("alg,arr,steps", [("essfm", "symmetric", 1), ("ssfm", "linear-first", 3),
                                           ("essfm", "nonlinear-first", 2), ("ffe", "symmetric", 1)])
def test_general_block_lengths_match_oracle(n_blk, m, alg, arr, steps):
    rng = np.random.default_rng(n_blk * 7 + steps)
    n = 3 * n_blk + 77 if n_blk >= 16384 else 301
    span = pb.FiberParams(-21.68, 1.3, 0.2, 80.0)
    link = quiet_link(3, span)   # 3 spans: N_s = 2 puts a step boundary mid-span (gain != 1)
    nc = 0 if n_blk <= 2 else min(3, (n_blk - 1) // 2) if n_blk < 16384 else 17
    coeffs = None if alg != "essfm" else pb.EssfmCoefficients(np.r_[1.0, 0.05 * rng.normal(size=nc)])
    cfg = pb.DbpConfig(alg, pb.OverlapPlan(n_blk, m), link, num_steps=steps, coeffs=coeffs, arrangement=arr)
    x = (0.01 * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n)))).astype(np.complex64)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        got = pb.backpropagate(pb.DualPolSignal(x[0], x[1], 56e9), cfg).stack()
    want = dbp_port.backpropagate_arrays(x.astype(np.complex128), 56e9, port_config(cfg))
    if n_blk - m >= 16:
        err = dbp_port.per_block_rel_l2(got, want, n_blk, m).max()
    else:   # tiny kept segments: whole-signal bar (a 1-sample segment has no meaningful norm)
        err = rel_l2(got, want)
    assert err <= 1e-6, (n_blk, m, alg, arr, err)   # float64 inside: only the complex64 I/O rounding


@pytest.mark.parametrize("n_blk,m,n", [(16384, 3000, 4 * 16384 + 2), (32768, 12419, 117994)])
def test_general_block_lengths_through_the_host_pipelines(n_blk, m, n):
    # the staged host pipelines run consecutive chunks on two streams; the general path's
    # kernels share one workspace per plan, so its launches must take turns
    # (launch_general's ws_done event).  Found by tools/fuzz_parity.py --seed 4242:
    # garbage at N = 32768, n = 117994 before the event.  Repeated: a race is timing dependent.
    rng = np.random.default_rng(n)
    span = pb.FiberParams(-21.68, 1.3, 0.2, 60.0)
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(n_blk, m), quiet_link(2, span), num_steps=8,
                       coeffs=pb.EssfmCoefficients(np.r_[1.0, 0.05 * rng.normal(size=23)]),
                       arrangement="linear-first")
    x = (0.02 * (rng.normal(size=(2, 2, n)) + 1j * rng.normal(size=(2, 2, n)))).astype(np.complex64)
    want = [dbp_port.backpropagate_arrays(x[i].astype(np.complex128), 56e9, port_config(cfg)) for i in range(2)]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for _ in range(3):
            got = pb.backpropagate_batch(x, 56e9, cfg)                      # pageable complex64 rows
            for i in range(2):
                assert dbp_port.per_block_rel_l2(got[i], want[i], n_blk, m).max() <= 1e-6
            one = pb.backpropagate(pb.DualPolSignal(x[0, 0], x[0, 1], 56e9), cfg).stack()   # complex128 rows
            assert dbp_port.per_block_rel_l2(one, want[0], n_blk, m).max() <= 1e-6


def test_general_block_length_multi_chunk_and_chunk_mode_in_subprocess():
    # a small workspace budget (DBP_GENERAL_WS_MB) forces many block chunks;
    # the chunk-mode entry (dbp_run_chunk over two halves) must equal the
    # whole-signal run bit for bit, and the identity program must frame exactly
    import os
    import subprocess
    import sys
    from pathlib import Path

    code = r'''
import numpy as np, torch, warnings
import paper_1507_00921_b200 as pb
from oracle import dbp_port
from tests.helpers import quiet_link, port_config
rng = np.random.default_rng(5)
N, M, n = 16384, 1000, 16384 * 9 + 5
span = pb.FiberParams(-21.68, 1.3, 0.2, 80.0)
cfg = pb.DbpConfig("essfm", pb.OverlapPlan(N, M), quiet_link(40, span), num_steps=1,
                   coeffs=pb.EssfmCoefficients(np.r_[1.0, 0.1, -0.02]))
x = (0.02 * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n)))).astype(np.complex64)
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    eng = pb.get_engine(cfg, 56e9)
got = eng.run_host(x[None])[0]
want = dbp_port.backpropagate_arrays(x.astype(np.complex128), 56e9, port_config(cfg))
err = dbp_port.per_block_rel_l2(got, want, N, M).max()
assert err <= 1e-6, err
nb = eng.num_blocks(n)
h = nb // 2
parts = [eng.run_host(x[None], block_range=(0, h))[0], eng.run_host(x[None], block_range=(h, nb))[0]]
step = N - M
joined = np.concatenate([parts[0][:, :h * step], parts[1][:, h * step:]], axis=1)
assert np.array_equal(joined, got)
ident = pb.overlap_save_run(pb.DualPolSignal(x[0], x[1], 56e9), pb.OverlapPlan(N, M),
                            pb.identity_processor(pb.OverlapPlan(N, M), 56e9))
assert np.array_equal(ident.stack(), x.astype(np.complex128))
print("ok", err)
'''
    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, DBP_GENERAL_WS_MB="3")
    res = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0 and "ok" in res.stdout, res.stdout[-2000:] + res.stderr[-3000:]


def test_general_block_length_coefficient_batch_matches_oracle():
    # per-item coefficient sets (the training batch, dbp_run_host_coeff_batch)
    # on the general path: each set against the oracle with that set
    # (the batch entry carries float32 coefficients, so the oracle gets them rounded)
    rng = np.random.default_rng(11)
    N, M, n = 16384, 1500, 40000
    span = pb.FiberParams(-21.68, 1.3, 0.2, 80.0)
    sets = np.stack([np.r_[1.0, 0.1 * rng.normal(size=5)] for _ in range(3)])
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(N, M), quiet_link(10, span), num_steps=1,
                       coeffs=pb.EssfmCoefficients(sets[0]))
    x = (0.02 * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n)))).astype(np.complex64)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        eng = pb.DbpEngine(cfg, 56e9)
    try:
        eng.native.set_coeff_batch(sets)
        out = np.zeros((3, 2, n), np.complex64)
        eng.native.run_host_coeff_batch(x, out, n)
    finally:
        eng.close()
    for i in range(3):
        c32 = sets[i].astype(np.float32).astype(np.float64)
        ci = pb.DbpConfig("essfm", pb.OverlapPlan(N, M), quiet_link(10, span), num_steps=1,
                          coeffs=pb.EssfmCoefficients(c32))
        want = dbp_port.backpropagate_arrays(x.astype(np.complex128), 56e9, port_config(ci))
        assert dbp_port.per_block_rel_l2(out[i], want, N, M).max() <= 1e-6, i


@pytest.mark.parametrize("n_blk,m,alg", [(8192, 1400, "essfm"), (8192, 1023, "ssfm"), (8192, 1024, "ffe"),
                                         (4096, 701, "essfm"), (16384, 2000, "essfm")])
def test_chunk_mode_and_block_ranges_bit_equal_whole_every_kernel(rng, n_blk, m, alg):
    # the multi-GPU contract on the N = 8192 R2 kernel (its TMA / paired / 8-byte
    # output stores: odd M makes the kept ranges odd), the FFE pairs, the
    # 4096 kernel and the general path: chunk mode and host block ranges
    # reproduce the whole-signal result bit for bit
    torch = pytest.importorskip("torch")
    coeffs = pb.EssfmCoefficients(waveforms.gaussian_coeffs(9)) if alg == "essfm" else None
    cfg = pb.DbpConfig(alg, pb.OverlapPlan(n_blk, m), quiet_link(20, STD), num_steps=2 if alg == "ssfm" else 1,
                       coeffs=coeffs, arrangement="linear-first" if alg == "ssfm" else "symmetric")
    n = 5 * n_blk + 333
    x = (0.03 * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n)))).astype(np.complex64)
    whole = _run(x, cfg)[0]
    eng = pb.get_engine(cfg, 56e9, 0)
    nb = eng.num_blocks(n)
    cuts = [(0, 2), (2, nb - 1), (nb - 1, nb)]
    for b0, b1 in cuts:
        lo, hi = cfg.plan.input_span(b0, b1)
        span = np.ascontiguousarray(pb.framing.gather_span(x, lo, hi))
        olo, ohi = cfg.plan.output_span(b0, b1, n)
        d_in = torch.from_numpy(span.view(np.float32)).cuda()
        d_out = torch.zeros((2, (ohi - olo) * 2), dtype=torch.float32, device="cuda")
        eng.native.run_chunk(d_in.data_ptr(), d_out.data_ptr(), n, 1, b0, b1, hi - lo, ohi - olo)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(d_out.cpu().numpy().view(np.complex64), whole[:, olo:ohi])
        part = eng.run_host(x[None], block_range=(b0, b1))[0]
        np.testing.assert_array_equal(part[:, olo:ohi], whole[:, olo:ohi])
