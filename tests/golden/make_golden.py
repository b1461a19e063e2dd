"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (the reference is not present on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference ``fiberdbp`` package from $FIBERDBP_REF (default
/root/reference/pkg/src) and records inputs and outputs of the hot-path
functions -- ``backpropagate`` (dbp.py:160), the per-block ``process``
closure it hands to ``overlap_save_run`` (dbp.py:212-233, captured by
wrapping the module-global ``overlap_save_run`` looked up at dbp.py:235),
``nonlinear_substep_essfm`` (dbp.py:49), ``_reverse_step_schedule``
(dbp.py:112) and ``channel_memory_samples`` (dbp.py:35).  Every signal
input is first rounded to complex64 so the GPU (complex64) and the reference
(complex128) see identical samples.
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
sys.path.insert(0, str(REPO))

import fiberdbp  # noqa: E402
from fiberdbp import dbp as ref_dbp  # noqa: E402
from fiberdbp import (  # noqa: E402
    DbpConfig, DualPolSignal, EssfmCoefficients, FiberParams, LinkConfig,
    OverlapPlan, SsfmStepConfig, propagate_link,
)

from oracle.waveforms import add_awgn_osnr, d_to_beta2, gaussian_coeffs, qpsk_rrc  # noqa: E402

OUT = HERE / "golden_v1.npz"
MANIFEST = HERE / "golden_v1.json"


def c64(a):
    return np.asarray(a).astype(np.complex64)


def quiet_link(num_spans, span):
    return LinkConfig(span=span, num_spans=num_spans, amp_gain_db=None,
                      amp_noise_figure_db=None, pol_rotation=False)


def capture_blocks(sig, cfg, picks):
    """Run backpropagate while recording the per-block closure on chosen blocks."""
    seen = {}
    real_run = ref_dbp.overlap_save_run

    def spy(s, plan, proc, jobs=1):
        step, lead = plan.usable, plan.overlap // 2
        stack = s.stack()
        n = stack.shape[1]
        for b in picks:
            idx = (np.arange(plan.block_len) + b * step - lead) % n
            blk = stack[:, idx]
            seen[b] = (blk.copy(), proc(blk))
        return real_run(s, plan, proc, jobs=jobs)

    ref_dbp.overlap_save_run = spy
    try:
        out = ref_dbp.backpropagate(sig, cfg)
    finally:
        ref_dbp.overlap_save_run = real_run
    return out, seen


def main():
    t0 = time.time()
    arrays = {}
    cases = []
    rng = np.random.default_rng(20260101)

    # ---- channel memory known answers (test_dbp.py:31-37) ----
    mem = [(21.0, 3000.0, 50e9), (-21.0, 3000.0, 50e9), (21.0, 3200.0, 56e9),
           (-21.6826, 3200.0, 56e9), (21.0, 2000.0, 50e9)]
    arrays["memory_args"] = np.array(mem)
    arrays["memory_vals"] = np.array([ref_dbp.channel_memory_samples(*m) for m in mem])

    # ---- reverse schedules ----
    std = FiberParams(beta2=-21.0, gamma=1.3, alpha_db_per_km=0.2, length=40.0)
    sched_cases = [(std, 4, 1), (std, 3, 3), (std, 8, 1), (std, 8, 2), (std, 8, 3),
                   (std, 8, 5), (std, 8, 160), (std, 2, 7),
                   (FiberParams(-21.0, 1.3, 0.0, 50.0), 2, 5),
                   (FiberParams(-21.6826, 1.3, 0.2, 80.0), 40, 1),
                   (FiberParams(-21.6826, 1.3, 0.2, 80.0), 40, 20),
                   (FiberParams(-21.6826, 1.3, 0.2, 80.0), 40, 3)]
    for i, (span, ns, steps) in enumerate(sched_cases):
        sch = ref_dbp._reverse_step_schedule(quiet_link(ns, span), steps)
        arrays[f"sched{i}"] = np.array(sch)
        arrays[f"sched{i}_args"] = np.array([span.beta2, span.gamma, span.alpha_db_per_km,
                                             span.length, ns, steps], dtype=np.float64)

    # ---- ESSFM sub-step vs nested loop geometry (test_dbp.py:47-57) ----
    for nc in (0, 1, 2, 4):
        blk = 0.7 * (rng.normal(size=(2, 16)) + 1j * rng.normal(size=(2, 16)))
        c = rng.normal(size=nc + 1) * 0.3
        c[0] = 1.0
        arrays[f"sub{nc}_in"] = blk
        arrays[f"sub{nc}_c"] = c
        arrays[f"sub{nc}_out"] = ref_dbp.nonlinear_substep_essfm(blk, 1.7, 0.25, EssfmCoefficients(c))

    # ---- whole-path cases on white dual-pol noise (reference test geometry) ----
    noise_cases = [
        # name, algorithm, N, M, n, spans, steps, arrangement, nc
        ("ffe_a", "ffe", 1024, 256, 4096, 4, 1, "symmetric", None),
        ("ffe_tiny1", "ffe", 2048, 512, 1, 2, 1, "symmetric", None),
        ("ffe_tiny5", "ffe", 2048, 512, 5, 2, 1, "symmetric", None),
        ("ffe_1537", "ffe", 2048, 512, 1537, 2, 1, "symmetric", None),
        ("ssfm_sym", "ssfm", 512, 128, 1024, 3, 5, "symmetric", None),
        ("ssfm_lf", "ssfm", 512, 128, 1024, 2, 4, "linear-first", None),
        ("ssfm_nf", "ssfm", 512, 128, 1000, 3, 3, "nonlinear-first", None),
        ("essfm_sym", "essfm", 256, 64, 3000, 2, 2, "symmetric", 4),
        ("essfm_lf", "essfm", 1024, 256, 5000, 8, 3, "linear-first", 9),
        ("essfm_nf", "essfm", 128, 32, 300, 1, 1, "nonlinear-first", 2),
        ("essfm_odd", "essfm", 2048, 512, 4096, 2, 4, "symmetric", 13),
        ("ssfm_8192", "ssfm", 8192, 2048, 12000, 4, 2, "symmetric", None),
        ("essfm_4096", "essfm", 4096, 1024, 9000, 4, 1, "symmetric", 33),
        ("ffe_16", "ffe", 16, 4, 100, 1, 1, "symmetric", None),
        ("essfm_32", "essfm", 32, 8, 200, 1, 2, "linear-first", 3),
        ("ssfm_64", "ssfm", 64, 16, 333, 1, 1, "nonlinear-first", None),
    ]
    for name, alg, N, M, n, spans, steps, arr, nc in noise_cases:
        # split-step cases at a physical launch power (0 dBm, every third at +4 dBm):
        # at the reference tests' unit-variance power (~4 W) the accumulated nonlinear
        # phase is 1e2-1e3 rad and no complex64 evaluation is well conditioned
        power_dbm = None if alg == "ffe" else (4.0 if len(cases) % 3 == 0 else 0.0)
        amp = 1.0 if power_dbm is None else math.sqrt(10 ** ((power_dbm - 30) / 10) / 4.0)
        x = c64(amp * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n))))
        sig = DualPolSignal(x[0], x[1], 56e9)
        coeffs = None
        if alg == "essfm":
            c = rng.normal(size=nc + 1) * 0.2
            c[0] = 1.0
            coeffs = EssfmCoefficients(c)
        cfg = DbpConfig(alg, OverlapPlan(N, M), quiet_link(spans, std), num_steps=steps,
                        coeffs=coeffs, arrangement=arr)
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            out = ref_dbp.backpropagate(sig, cfg)
        arrays[f"bp_{name}_in"] = x
        arrays[f"bp_{name}_out"] = out.stack()
        if coeffs is not None:
            arrays[f"bp_{name}_c"] = coeffs.c
        cases.append(dict(name=name, algorithm=alg, block_len=N, overlap=M, n=n,
                          sample_rate=56e9, beta2=std.beta2, gamma=std.gamma,
                          alpha_db_per_km=std.alpha_db_per_km, span_km=std.length,
                          num_spans=spans, num_steps=steps, arrangement=arr,
                          n_coeffs=None if nc is None else nc, signal="white",
                          power_dbm=power_dbm))

    # ---- config-0-like link waveform (BASELINE configs[0..2] geometry, shortened) ----
    beta2 = d_to_beta2(17.0)
    span80 = FiberParams(beta2=beta2, gamma=1.3, alpha_db_per_km=0.2, length=80.0)
    link = quiet_link(40, span80)
    nsym = 2 ** 13
    tx, symbols = qpsk_rrc(nsym, sps=2, rolloff=0.1, seed=0, power_dbm=0.0)
    t1 = time.time()
    rx = propagate_link(DualPolSignal(tx[0], tx[1], 56e9), link, SsfmStepConfig(80), rng=None)
    print(f"forward link {time.time() - t1:.1f}s")
    rxs = c64(add_awgn_osnr(rx.stack(), 56e9, 14.0, seed=1))
    arrays["link_tx_symbols"] = symbols
    arrays["link_rx"] = rxs
    sig = DualPolSignal(rxs[0], rxs[1], 56e9)
    c17 = gaussian_coeffs(17)
    arrays["link_c17"] = c17
    span_nl89 = FiberParams(beta2=beta2, gamma=1.3 * 8.0 / 9.0, alpha_db_per_km=0.2, length=80.0)
    link_cases = [
        ("c0_sym", DbpConfig("essfm", OverlapPlan(2048, 700), link, 1, EssfmCoefficients(c17), "symmetric")),
        ("c0_lf", DbpConfig("essfm", OverlapPlan(2048, 700), link, 1, EssfmCoefficients(c17), "linear-first")),
        ("c1_1024", DbpConfig("ffe", OverlapPlan(1024, 700), link)),
        ("c1_2048", DbpConfig("ffe", OverlapPlan(2048, 700), link)),
        ("c1_4096", DbpConfig("ffe", OverlapPlan(4096, 700), link)),
        ("c2_ssfm20", DbpConfig("ssfm", OverlapPlan(2048, 700), quiet_link(40, span_nl89), 20,
                                None, "linear-first")),
    ]
    import warnings
    for name, cfg in link_cases:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            picks = (0, 5)
            out, seen = capture_blocks(sig, cfg, picks)
        arrays[f"link_{name}_out"] = out.stack()
        arrays[f"link_{name}_blk_in"] = c64(np.stack([seen[b][0] for b in picks]))
        arrays[f"link_{name}_blk_out"] = np.stack([seen[b][1] for b in picks])
        sp = cfg.link.span
        cases.append(dict(name=name, algorithm=cfg.algorithm, block_len=cfg.plan.block_len,
                          overlap=cfg.plan.overlap, n=rxs.shape[1], sample_rate=56e9,
                          beta2=sp.beta2, gamma=sp.gamma, alpha_db_per_km=sp.alpha_db_per_km,
                          span_km=sp.length, num_spans=cfg.link.num_spans,
                          num_steps=cfg.num_steps, arrangement=cfg.arrangement,
                          n_coeffs=17 if cfg.algorithm == "essfm" else None, signal="link",
                          picks=list(picks)))

    # ---- coefficient training (train.py:86-188) on the link waveform ----
    from fiberdbp import TrainConfig, optimize_coefficients
    tcfg = TrainConfig(n_coeffs=4, target_steps_per_span=2, train_samples=8192, max_iterations=6)
    dcfg = DbpConfig("essfm", OverlapPlan(2048, 700), link, num_steps=1,
                     coeffs=EssfmCoefficients.identity(4), arrangement="symmetric")
    t1 = time.time()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = optimize_coefficients(sig, dcfg, tcfg)
    print(f"training {time.time() - t1:.1f}s iterations {res.iterations} mse {res.initial_mse:.4e} -> {res.final_mse:.4e}")
    arrays["train_c"] = res.coefficients.c
    arrays["train_mse"] = np.array([res.initial_mse, res.final_mse, res.iterations, float(res.converged)])

    np.savez_compressed(OUT, **arrays)
    MANIFEST.write_text(json.dumps(dict(
        generator="tests/golden/make_golden.py", reference="fiberdbp " + fiberdbp.__version__,
        numpy=np.__version__, cases=cases,
        sched_cases=len(sched_cases)), indent=1))
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB) in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
