"""SURVEY 8f-1 measurement: ESSFM coefficient fit on the GPU vs the CPU restatement.

    python tools/train_bench.py [--n-coeffs 17] [--iterations 10]

Workload: the reference TrainConfig defaults except N_c / iteration count
(16384 training samples, fine target 4 steps per span) on a seeded 0 dBm
PM-QPSK RRC-0.1 waveform forward-propagated over 40 x 80 km (oracle forward
SSFM, 8 steps per span) with N = 2048 / M = 700, ESSFM 1 step, symmetric.
CPU leg: oracle/train_port.py (train.py:86-188 on the float64 numpy port),
one process.  Prints one JSON line.
"""
import argparse
import json
import sys
import time
import warnings
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-coeffs", type=int, default=17)
    ap.add_argument("--iterations", type=int, default=10)
    ap.add_argument("--train-samples", type=int, default=16384)
    a = ap.parse_args()
    import paper_1507_00921_b200 as pb
    from oracle import dbp_port, train_port, waveforms

    warnings.simplefilter("ignore")
    beta2 = waveforms.d_to_beta2(17.0)
    tx, _ = waveforms.qpsk_rrc(a.train_samples // 2, 2, 0.1, seed=11, power_dbm=0.0)
    rx = waveforms.forward_link(tx, 56e9, beta2, 1.3, 0.2, 80.0, 40, 8).astype(np.complex64)
    span = pb.FiberParams(beta2, 1.3, 0.2, 80.0)
    link = pb.LinkConfig(span, 40, amp_noise_figure_db=None, pol_rotation=False)
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(2048, 700), link,
                       coeffs=pb.EssfmCoefficients.identity(a.n_coeffs))
    tcfg = pb.TrainConfig(n_coeffs=a.n_coeffs, target_steps_per_span=4, train_samples=a.train_samples,
                          max_iterations=a.iterations, tolerance=1e-12)
    sig = pb.DualPolSignal(rx[0], rx[1], 56e9)
    pb.optimize_coefficients(sig, cfg, pb.TrainConfig(n_coeffs=a.n_coeffs, target_steps_per_span=4,
                                                      train_samples=a.train_samples, max_iterations=1))
    t0 = time.perf_counter()
    res = pb.optimize_coefficients(sig, cfg, tcfg)
    gpu_s = time.perf_counter() - t0

    pcfg = dbp_port.PortConfig.from_objects(cfg)
    t0 = time.perf_counter()
    c, err, initial, _, iters = train_port.fit(rx.astype(np.complex128), 56e9, pcfg, a.n_coeffs, 4,
                                               a.train_samples, a.iterations, tolerance=1e-12)
    cpu_s = time.perf_counter() - t0
    print(json.dumps({
        "metric": "ESSFM coefficient fit wall time (s)", "n_coeffs": a.n_coeffs, "iterations": a.iterations,
        "train_samples": a.train_samples,
        "gpu": {"seconds": gpu_s, "iterations": res.iterations, "initial_mse": res.initial_mse,
                "final_mse": res.final_mse},
        "cpu_port": {"seconds": cpu_s, "iterations": iters, "initial_mse": initial, "final_mse": err,
                     "cores": 1},
        "speedup": cpu_s / gpu_s,
        "coeff_max_abs_diff": float(np.max(np.abs(res.coefficients.c - c))),
    }), flush=True)


if __name__ == "__main__":
    main()
