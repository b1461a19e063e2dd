"""The paper's experiment end to end on one GPU: Q factor vs launch power.

    python tools/q_vs_power.py [--symbols 16] [--out profiles/r1/q_vs_power.json]

Every stage runs in this package (cf. the reference's ``ber-sweep``,
cli.py:599-695): seeded dual-pol QPSK with RRC(0.1) pulses at 2 samples /
symbol (28 GBd) -> ``propagate_link_batch`` over 40 x 80 km SMF (D = 17,
0.2 dB/km, gamma 1.3, EDFAs with 5 dB noise figure, Haar polarisation
rotations, 1 km steps; all launch powers as one batch) -> DBP variants
(CD-only FFE, SSFM with 1 and 40 steps, ESSFM with 1 step and N_c = 17
coefficients fitted per power by ``optimize_coefficients``) -> the
receiver chain ``receive_batch`` (CMA, carrier recovery, decisions, BER).
Reports Q (dB) per power and variant plus the time of every stage: the whole
experiment runs twice (the second pass must reproduce the first exactly) and
the stage times are the second pass's, the first pass's total -- one-time
set-up included -- is ``first_pass_total_s``; ``--no-warmup`` runs once.
"""

from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

LIGHT = 299792458.0


def d_to_beta2(d_ps_nm_km: float, wavelength_nm: float = 1550.0) -> float:
    lam = wavelength_nm * 1e-9
    return -d_ps_nm_km * 1e-6 * lam ** 2 / (2.0 * math.pi * LIGHT) * 1e3 * 1e24


def rrc_tx(num_symbols: int, seed: int, sps: int = 2, rolloff: float = 0.1):
    """Unit-power dual-pol QPSK with root-raised-cosine pulses (circular)."""
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2, size=(2, 2, num_symbols))
    sym = ((1.0 - 2.0 * bits[:, 0]) + 1j * (1.0 - 2.0 * bits[:, 1])) / math.sqrt(2.0)
    n = num_symbols * sps
    f = np.abs(np.fft.fftfreq(n, 1.0 / sps))
    lo, hi = (1.0 - rolloff) / 2.0, (1.0 + rolloff) / 2.0
    h = np.where(f <= lo, 1.0, 0.0)
    mid = (f > lo) & (f <= hi)
    h[mid] = np.sqrt(0.5 * (1.0 + np.cos(np.pi / rolloff * (f[mid] - lo))))
    up = np.zeros((2, n), dtype=np.complex128)
    up[:, ::sps] = sym
    wave = np.fft.ifft(np.fft.fft(up, axis=1) * h, axis=1)
    wave /= math.sqrt(np.mean(np.abs(wave[0]) ** 2 + np.abs(wave[1]) ** 2))
    return wave, sym


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--symbols", type=int, default=16, help="log2 symbols per polarisation")
    ap.add_argument("--powers", default="-4,-3,-2,-1,0,1,2,3,4")
    ap.add_argument("--steps-per-span", type=int, default=80)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-warmup", action="store_true",
                    help="one pass only, timings include the cold starts")
    a = ap.parse_args()
    import paper_1507_00921_b200 as pb

    powers = [float(p) for p in a.powers.split(",")]
    m = 1 << a.symbols
    fs = 56e9
    span = pb.FiberParams(beta2=d_to_beta2(17.0), gamma=1.3, alpha_db_per_km=0.2, length=80.0)
    link = pb.LinkConfig(span=span, num_spans=40, amp_noise_figure_db=5.0, pol_rotation=True)
    tx, sym = rrc_tx(m, seed=0)
    batch = np.stack([tx * math.sqrt(10 ** ((p - 30) / 10)) for p in powers]).astype(np.complex64)

    quiet = pb.LinkConfig(span=span, num_spans=40, amp_gain_db=None, amp_noise_figure_db=None, pol_rotation=False)
    plan = pb.OverlapPlan(2048, 700)
    tcfg = pb.TrainConfig(n_coeffs=17, target_steps_per_span=4, train_samples=16384, max_iterations=10)

    def one_pass():
        timings = {}
        t0 = time.perf_counter()
        rx = pb.propagate_link_batch(batch, fs, link, pb.SsfmStepConfig(a.steps_per_span),
                                     [np.random.SeedSequence([7, i]) for i in range(len(powers))])
        timings["link_s"] = time.perf_counter() - t0
        variants = {
            "cdc": pb.DbpConfig("ffe", plan, quiet),
            "ssfm_1": pb.DbpConfig("ssfm", plan, quiet, num_steps=1),
            "ssfm_40": pb.DbpConfig("ssfm", plan, quiet, num_steps=40),
        }
        q = {name: [] for name in list(variants) + ["essfm_1_nc17"]}
        ber = {name: [] for name in q}
        timings["dbp_s"] = 0.0
        timings["train_s"] = 0.0
        timings["rx_s"] = 0.0
        for name, cfg in variants.items():
            t0 = time.perf_counter()
            out = pb.backpropagate_batch(rx, fs, cfg)
            timings["dbp_s"] += time.perf_counter() - t0
            t0 = time.perf_counter()
            mets = pb.receive_batch(out, 28e9, sym)
            timings["rx_s"] += time.perf_counter() - t0
            q[name] = [None if isinstance(r, Exception) else r.q_factor_db for r in mets]
            ber[name] = [None if isinstance(r, Exception) else r.ber for r in mets]
        # ESSFM: one step, N_c = 17 coefficients fitted per launch power (train.py:86-188)
        outs = []
        coeffs = []
        for i in range(len(powers)):
            sig = pb.DualPolSignal(rx[i, 0], rx[i, 1], fs)
            geometry = pb.DbpConfig("essfm", plan, quiet, num_steps=1, coeffs=pb.EssfmCoefficients.identity(17))
            t0 = time.perf_counter()
            res = pb.optimize_coefficients(sig, geometry, tcfg)
            timings["train_s"] += time.perf_counter() - t0
            coeffs.append(res.coefficients.c.tolist())
            cfg = pb.DbpConfig("essfm", plan, quiet, num_steps=1, coeffs=res.coefficients)
            t0 = time.perf_counter()
            outs.append(pb.backpropagate_batch(rx[i:i + 1], fs, cfg)[0])
            timings["dbp_s"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        mets = pb.receive_batch(np.stack(outs), 28e9, sym)
        timings["rx_s"] += time.perf_counter() - t0
        q["essfm_1_nc17"] = [None if isinstance(r, Exception) else r.q_factor_db for r in mets]
        ber["essfm_1_nc17"] = [None if isinstance(r, Exception) else r.ber for r in mets]
        return q, ber, coeffs, timings

    # pass 1 pays the one-time costs (simulator tables for this length, DBP
    # engines, lazily loaded CUDA modules, cuFFT plans, receiver buffers);
    # pass 2 repeats the identical experiment and gives the steady-state stage times
    t0 = time.perf_counter()
    q, ber, coeffs, timings = one_pass()
    first = time.perf_counter() - t0
    if not a.no_warmup:
        q2, ber2, coeffs2, timings = one_pass()
        assert q2 == q and coeffs2 == coeffs, "the repeated pass must reproduce the first"
        timings["first_pass_total_s"] = first
    print("launch dBm " + " ".join(f"{p:>6.1f}" for p in powers))
    for name in q:
        print(f"{name:12s} " + " ".join("   n/a" if v is None else f"{min(v, 99.0):6.2f}" for v in q[name]))
    print(json.dumps(timings))
    if a.out:
        Path(a.out).write_text(json.dumps(dict(
            experiment="Q vs launch power, 40x80 km SMF, 28 GBd PM-QPSK RRC 0.1, EDFA NF 5 dB, "
                       f"2^{a.symbols} symbols/pol, {a.steps_per_span} SSFM steps/span",
            powers_dbm=powers, q_db=q, ber=ber, essfm_coefficients=coeffs, timings=timings), indent=1))


if __name__ == "__main__":
    main()
