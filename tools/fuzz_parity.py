"""Randomised parity sweep of the GPU paths against the CPU oracle (evidence run).

    python tools/fuzz_parity.py [--dbp 600] [--general 0] [--sim 60] [--rx 24] [--out profiles/r1/fuzz_parity.json]

DBP: random block length 16..8192, overlap, ragged length, algorithm,
arrangement, 1..8 steps, 1..8 spans of 20..100 km, N_c 0..64, batch 1..3,
launch power -6..+6 dBm -- per-block relative L2 vs oracle/dbp_port.py
(where the kept segment N - M is below 16 samples, per block against
max(segment norm, signal RMS x sqrt(segment size)): the L2 norm of a
1-sample segment is dominated by whether that sample is near zero).
Simulator: random n 2^8..2^18, 1..6 steps, loss / gamma / dispersion, with
and without nonlinearity -- whole-waveform rel-L2 vs oracle/channel_port.py.
Receiver: random polarisation mixes, noise and frequency offsets -- the
equaliser output and the error counts vs oracle/rx_port.py.  Prints one JSON
summary (worst errors, counts of tolerance violations).
"""
import argparse
import json
import math
import sys
import time
import warnings
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dbp", type=int, default=1500)
    ap.add_argument("--general", type=int, default=0,
                    help="extra DBP items at N = 1 .. 8, 16384, 32768 (the general block-length path)")
    ap.add_argument("--sim", type=int, default=60)
    ap.add_argument("--rx", type=int, default=24)
    ap.add_argument("--seed", type=int, default=20261020)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import paper_1507_00921_b200 as pb
    from oracle import channel_port as cp
    from oracle import dbp_port, rx_port
    gen = np.random.default_rng(a.seed)
    t0 = time.time()
    res = {"dbp": {"cases": 0, "worst": 0.0, "violations": 0, "worst_case": None},
           "sim": {"cases": 0, "worst_ratio": 0.0, "violations": 0},
           "rx": {"cases": 0, "worst_eq_diff": 0.0, "count_mismatches": 0}}
    for case in range(a.dbp + a.general):
        if case < a.dbp:
            logn = int(gen.integers(4, 14))
        else:   # block lengths outside the fused kernel (the float64 general path)
            logn = (0, 1, 2, 3, 14, 15)[int(gen.integers(0, 6))]
            res["dbp"]["general_cases"] = res["dbp"].get("general_cases", 0) + 1
        nb = 1 << logn
        m = int(gen.integers(0, nb))
        n = int(gen.integers(1, 4 * nb + 2))
        alg = ("ffe", "ssfm", "essfm")[int(gen.integers(0, 3))]
        steps = int(gen.integers(1, 9))
        spans = int(gen.integers(1, 9))
        arr = pb.ARRANGEMENTS[int(gen.integers(0, 3))]
        coeffs = None
        if alg == "essfm":
            nc = int(gen.integers(0, min(64, (nb - 1) // 2) + 1))
            c = gen.normal(size=nc + 1) * 0.1
            c[0] = 1.0
            coeffs = pb.EssfmCoefficients(c)
        span = pb.FiberParams(-21.68, 1.3, 0.2, float(gen.uniform(20.0, 100.0)))
        link = pb.LinkConfig(span=span, num_spans=spans, amp_gain_db=None, amp_noise_figure_db=None,
                             pol_rotation=False)
        cfg = pb.DbpConfig(alg, pb.OverlapPlan(nb, m), link, num_steps=steps, coeffs=coeffs, arrangement=arr)
        dbm = float(gen.uniform(-6.0, 6.0))
        amp = math.sqrt(10 ** ((dbm - 30) / 10) / 4.0)
        batch = int(gen.integers(1, 4))
        x = (amp * (gen.normal(size=(batch, 2, n)) + 1j * gen.normal(size=(batch, 2, n)))).astype(np.complex64)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            got = pb.backpropagate_batch(x, 56e9, cfg)
        for i in range(batch):
            want = dbp_port.backpropagate_arrays(x[i].astype(np.complex128), 56e9, dbp_port.PortConfig.from_objects(cfg))
            errs = dbp_port.per_block_rel_l2(got[i], want, nb, m)
            # a kept segment of < 16 samples (overlap within 16 of N) can be all but
            # zero, so its own norm is no scale: those segments are measured per
            # block against max(their norm, the signal RMS x sqrt(segment length))
            if nb - m >= 16:
                err = float(errs.max())
            else:
                step = nb - m
                rms = float(np.sqrt(np.mean(np.abs(want) ** 2)))
                err = 0.0
                for b0 in range(0, n, step):
                    d = got[i][:, b0:b0 + step] - want[:, b0:b0 + step]
                    ref = max(float(np.linalg.norm(want[:, b0:b0 + step])), rms * math.sqrt(d.size))
                    err = max(err, float(np.linalg.norm(d)) / ref)
                res["dbp"]["tiny_step_cases"] = res["dbp"].get("tiny_step_cases", 0) + 1
            res["dbp"]["cases"] += 1
            if err > res["dbp"]["worst"]:
                res["dbp"]["worst"] = err
                res["dbp"]["worst_case"] = dict(alg=alg, N=nb, M=m, n=n, steps=steps, spans=spans, arrangement=arr,
                                                nc=None if coeffs is None else len(coeffs.c) - 1, dbm=round(dbm, 2))
            res["dbp"]["violations"] += int(err > 1e-5)
    for case in range(a.sim):
        lg = int(gen.integers(8, 19))
        n = 1 << lg
        steps = int(gen.integers(1, 7))
        nl = bool(gen.integers(0, 2))
        fiber = pb.FiberParams(float(gen.uniform(-25.0, 25.0)), float(gen.uniform(0.0, 2.0)),
                               float(gen.uniform(0.0, 0.3)), float(gen.uniform(10.0, 100.0)))
        dbm = float(gen.uniform(-4.0, 6.0))
        amp = math.sqrt(10 ** ((dbm - 30) / 10) / 4.0)
        x = (amp * (gen.normal(size=(2, n)) + 1j * gen.normal(size=(2, n)))).astype(np.complex64)
        got = pb.propagate_span(pb.DualPolSignal(x[0], x[1], 56e9), fiber, pb.SsfmStepConfig(steps, nl)).stack()
        want = cp.span(x.astype(np.complex128), 56e9, fiber.beta2, fiber.gamma, fiber.alpha_db_per_km,
                       fiber.length, steps, nl)
        err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
        tol = 2e-6 + 6e-8 * steps
        res["sim"]["cases"] += 1
        res["sim"]["worst_ratio"] = max(res["sim"]["worst_ratio"], err / tol)
        res["sim"]["violations"] += int(err > tol)
    from oracle.waveforms import qpsk_rrc
    for case in range(a.rx):
        tx, sym = qpsk_rrc(1 << 12, seed=int(gen.integers(0, 1 << 30)))
        th, ph = float(gen.uniform(0, math.pi)), float(gen.uniform(0, 2 * math.pi))
        jones = np.array([[math.cos(th), math.sin(th) * np.exp(1j * ph)], [-math.sin(th) * np.exp(-1j * ph), math.cos(th)]])
        y = jones @ tx
        snr = float(gen.uniform(0.02, 0.25))
        y = y + snr * math.sqrt(np.mean(np.abs(y) ** 2)) * (gen.normal(size=y.shape) + 1j * gen.normal(size=y.shape))
        eq = pb.butterfly_equalize(pb.DualPolSignal(y[0], y[1], 56e9)).stack()
        weq, _, _ = rx_port.equalize(y)
        res["rx"]["cases"] += 1
        res["rx"]["worst_eq_diff"] = max(res["rx"]["worst_eq_diff"], float(np.max(np.abs(eq - weq))))
        (met,) = pb.receive_batch(y, 28e9, sym)
        rec, _, _ = rx_port.carrier(weq, 28e9, sym)
        errors, counted = rx_port.count_errors(rx_port.decide(rec), rx_port.decide(sym))
        if isinstance(met, Exception) or met.ber != errors / (2 * counted):
            res["rx"]["count_mismatches"] += 1
    res["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(res))
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
