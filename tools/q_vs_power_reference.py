"""Reference (CPU) run of tools/q_vs_power.py at chosen powers -- cross-check of the GPU pipeline.

Runs in the build container only (imports /root/reference):
    PYTHONDONTWRITEBYTECODE=1 python tools/q_vs_power_reference.py --powers 0,2
Same transmitter, the reference's own propagate_link with the same seed
sequence per power, reference backpropagate (CDC, ESSFM N_c = 17 fitted by
the reference optimize_coefficients) and the reference receiver chain.
"""
import argparse
import json
import math
import os
import sys
import time
import warnings
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, os.environ.get("FIBERDBP_REF", "/root/reference/pkg/src"))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import fiberdbp as ref  # noqa: E402
from fiberdbp import modem  # noqa: E402

from q_vs_power import d_to_beta2, rrc_tx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--symbols", type=int, default=16)
    ap.add_argument("--powers", default="0,2")
    ap.add_argument("--all-powers", default="-4,-3,-2,-1,0,1,2,3,4")
    ap.add_argument("--steps-per-span", type=int, default=80)
    a = ap.parse_args()
    allp = [float(p) for p in a.all_powers.split(",")]
    m = 1 << a.symbols
    fs = 56e9
    span = ref.FiberParams(beta2=d_to_beta2(17.0), gamma=1.3, alpha_db_per_km=0.2, length=80.0)
    link = ref.LinkConfig(span=span, num_spans=40, amp_noise_figure_db=5.0, pol_rotation=True)
    quiet = ref.LinkConfig(span=span, num_spans=40, amp_gain_db=None, amp_noise_figure_db=None, pol_rotation=False)
    plan = ref.OverlapPlan(2048, 700)
    tx, sym = rrc_tx(m, seed=0)
    out = {}
    for p in [float(v) for v in a.powers.split(",")]:
        i = allp.index(p)
        x = (tx * math.sqrt(10 ** ((p - 30) / 10))).astype(np.complex64).astype(np.complex128)
        t0 = time.time()
        rx = ref.propagate_link(ref.DualPolSignal(x[0], x[1], fs), link, ref.SsfmStepConfig(a.steps_per_span),
                                rng=np.random.SeedSequence([7, i]))
        t_link = time.time() - t0
        rx = ref.DualPolSignal(rx.x.astype(np.complex64), rx.y.astype(np.complex64), fs)

        def q_of(sig):
            eq = modem.butterfly_equalize(sig)
            rec = modem.carrier_recover(eq.stack(), 28e9, reference=sym)
            return modem.measure_ber(modem.qpsk_decide(rec), modem.qpsk_decide(sym)).q_factor_db

        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            q_cdc = q_of(ref.backpropagate(rx, ref.DbpConfig("ffe", plan, quiet)))
            geo = ref.DbpConfig("essfm", plan, quiet, num_steps=1, coeffs=ref.EssfmCoefficients.identity(17))
            t0 = time.time()
            res = ref.optimize_coefficients(rx, geo, ref.TrainConfig(n_coeffs=17, target_steps_per_span=4,
                                                                      train_samples=16384, max_iterations=10))
            t_train = time.time() - t0
            q_essfm = q_of(ref.backpropagate(rx, ref.DbpConfig("essfm", plan, quiet, num_steps=1,
                                                               coeffs=res.coefficients)))
        out[p] = dict(q_cdc=q_cdc, q_essfm=q_essfm, link_s=t_link, train_s=t_train)
        print(p, json.dumps(out[p]), flush=True)


if __name__ == "__main__":
    main()
