"""Repeat each stage of tools/q_vs_power.py a few times (steady-state timing check)."""
import math, sys, time, warnings
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent)); sys.path.insert(0, str(Path(__file__).resolve().parent))
import numpy as np
import paper_1507_00921_b200 as pb
from q_vs_power import d_to_beta2, rrc_tx

powers = [-4.0, -3.0, -2.0, -1.0, 0.0, 1.0, 2.0, 3.0, 4.0]
fs = 56e9
span = pb.FiberParams(beta2=d_to_beta2(17.0), gamma=1.3, alpha_db_per_km=0.2, length=80.0)
link = pb.LinkConfig(span=span, num_spans=40, amp_noise_figure_db=5.0, pol_rotation=True)
quiet = pb.LinkConfig(span=span, num_spans=40, amp_gain_db=None, amp_noise_figure_db=None, pol_rotation=False)
tx, sym = rrc_tx(1 << 16, seed=0)
batch = np.stack([tx * math.sqrt(10 ** ((p - 30) / 10)) for p in powers]).astype(np.complex64)
plan = pb.OverlapPlan(2048, 700)
for k in range(3):
    t = time.perf_counter()
    rx = pb.propagate_link_batch(batch, fs, link, pb.SsfmStepConfig(80), [np.random.SeedSequence([7, i]) for i in range(9)])
    print("link", round(time.perf_counter() - t, 3))
cdc = pb.DbpConfig("ffe", plan, quiet)
for k in range(3):
    t = time.perf_counter(); out = pb.backpropagate_batch(rx, fs, cdc); t1 = time.perf_counter()
    pb.receive_batch(out, 28e9, sym); t2 = time.perf_counter()
    print("dbp", round(t1 - t, 4), "rx", round(t2 - t1, 4))
tcfg = pb.TrainConfig(n_coeffs=17, target_steps_per_span=4, train_samples=16384, max_iterations=10)
geometry = pb.DbpConfig("essfm", plan, quiet, num_steps=1, coeffs=pb.EssfmCoefficients.identity(17))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    for k in range(2):
        ts = []
        for i in range(9):
            t = time.perf_counter()
            pb.optimize_coefficients(pb.DualPolSignal(rx[i, 0], rx[i, 1], fs), geometry, tcfg)
            ts.append(round(time.perf_counter() - t, 4))
        print("fits", ts)
