"""Golden fixtures for the forward link simulator, made by the REFERENCE.

Run in the build container (the reference is not present on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_forward.py

Records inputs and outputs of ``fiberdbp.channel`` -- ``propagate_span``
(channel.py:74-94), ``amplify_with_ase`` (:97-128), ``haar_random_unitary``
(:131-138), ``random_polarization_rotation`` (:150-153) and
``propagate_link`` (:174-207) with ASE and Haar rotations drawn from the
reference's seeded child streams.  Inputs are rounded to complex64 first.
"""

from __future__ import annotations

import json
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
from fiberdbp import DualPolSignal, FiberParams, LinkConfig, SsfmStepConfig  # noqa: E402
from fiberdbp import channel as ref_ch  # noqa: E402

from oracle.waveforms import d_to_beta2, qpsk_rrc  # noqa: E402

OUT = HERE / "golden_fwd_v1.npz"
MANIFEST = HERE / "golden_fwd_v1.json"


def c64(a):
    return np.asarray(a).astype(np.complex64)


def main():
    t0 = time.time()
    arrays, cases = {}, []
    beta2 = d_to_beta2(17.0)
    span80 = FiberParams(beta2=beta2, gamma=1.3, alpha_db_per_km=0.2, length=80.0)
    lossless = FiberParams(beta2=beta2, gamma=1.3, alpha_db_per_km=0.0, length=50.0)

    def wave(nsym, seed, dbm):
        tx, _ = qpsk_rrc(nsym, sps=2, rolloff=0.1, seed=seed, power_dbm=dbm)
        return c64(tx)

    # ---- single spans ----
    span_cases = [
        ("span_nl", 2048, 11, 4.0, span80, SsfmStepConfig(20)),
        ("span_lin", 2048, 12, 4.0, span80, SsfmStepConfig(20, nonlinear_enabled=False)),
        ("span_lossless", 2048, 13, 6.0, lossless, SsfmStepConfig(7)),
        ("span_one_step", 128, 14, 8.0, span80, SsfmStepConfig(1)),
    ]
    for name, nsym, seed, dbm, fiber, cfg in span_cases:
        x = wave(nsym, seed, dbm)
        out = ref_ch.propagate_span(DualPolSignal(x[0], x[1], 56e9), fiber, cfg)
        arrays[f"{name}_in"], arrays[f"{name}_out"] = x, out.stack()
        cases.append(dict(name=name, kind="span", sample_rate=56e9, beta2=fiber.beta2, gamma=fiber.gamma,
                          alpha_db_per_km=fiber.alpha_db_per_km, length=fiber.length,
                          steps_per_span=cfg.steps_per_span, nonlinear=cfg.nonlinear_enabled))

    # ---- amplifier, Haar unitary, rotation ----
    x = wave(1024, 21, 0.0)
    sig = DualPolSignal(x[0], x[1], 56e9)
    arrays["amp_in"] = x
    arrays["amp_out"] = ref_ch.amplify_with_ase(sig, 16.0, 5.0, 1550.0, rng=3).stack()
    arrays["amp_quiet_out"] = ref_ch.amplify_with_ase(sig, 16.0, None).stack()
    arrays["haar11"] = ref_ch.haar_random_unitary(11)
    arrays["rot_out"] = ref_ch.random_polarization_rotation(sig, rng=5).stack()

    # ---- links with ASE and polarisation rotations ----
    link_cases = [
        ("link_ase_rot", 2048, 31, 2.0, LinkConfig(span=span80, num_spans=3), SsfmStepConfig(10), 7),
        ("link_gain_nf", 2048, 32, 0.0, LinkConfig(span=span80, num_spans=2, amp_gain_db=20.0,
                                                   amp_noise_figure_db=6.0, pol_rotation=False,
                                                   center_wavelength_nm=1560.0), SsfmStepConfig(5), 99),
        ("link_rot_only", 1024, 33, 3.0, LinkConfig(span=span80, num_spans=4, amp_noise_figure_db=None),
         SsfmStepConfig(8), 5),
    ]
    for name, nsym, seed, dbm, link, cfg, rs in link_cases:
        x = wave(nsym, seed, dbm)
        out = ref_ch.propagate_link(DualPolSignal(x[0], x[1], 56e9), link, cfg, rng=rs)
        arrays[f"{name}_in"], arrays[f"{name}_out"] = x, out.stack()
        cases.append(dict(name=name, kind="link", sample_rate=56e9, beta2=link.span.beta2,
                          gamma=link.span.gamma, alpha_db_per_km=link.span.alpha_db_per_km,
                          length=link.span.length, num_spans=link.num_spans, amp_gain_db=link.amp_gain_db,
                          amp_noise_figure_db=link.amp_noise_figure_db, pol_rotation=link.pol_rotation,
                          center_wavelength_nm=link.center_wavelength_nm,
                          steps_per_span=cfg.steps_per_span, nonlinear=cfg.nonlinear_enabled, rng=rs))

    # ---- the golden_v1 link waveform before its AWGN (40 x 80 km, 80 steps/span) ----
    x = wave(2 ** 13, 0, 0.0)
    link = LinkConfig(span=span80, num_spans=40, amp_gain_db=None, amp_noise_figure_db=None, pol_rotation=False)
    t1 = time.time()
    out = ref_ch.propagate_link(DualPolSignal(x[0], x[1], 56e9), link, SsfmStepConfig(80), rng=None)
    print(f"config-0 forward link {time.time() - t1:.1f}s")
    arrays["link_c0_in"], arrays["link_c0_out"] = x, c64(out.stack())
    cases.append(dict(name="link_c0", kind="link", sample_rate=56e9, beta2=beta2, gamma=1.3,
                      alpha_db_per_km=0.2, length=80.0, num_spans=40, amp_gain_db=None,
                      amp_noise_figure_db=None, pol_rotation=False, center_wavelength_nm=1550.0,
                      steps_per_span=80, nonlinear=True, rng=None))

    np.savez_compressed(OUT, **arrays)
    MANIFEST.write_text(json.dumps(dict(generator="tests/golden/make_golden_forward.py",
                                        reference="fiberdbp " + fiberdbp.__version__,
                                        numpy=np.__version__, cases=cases), indent=1))
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB) in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
