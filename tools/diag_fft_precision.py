#!/usr/bin/env python
"""Worst per-block rel-L2 of the GPU DBP against the oracle vs step count.

    DBP_FFT=dit python tools/diag_fft_precision.py      # fused-twiddle FFT
    DBP_FFT=adjoint python tools/diag_fft_precision.py  # exact-adjoint FFT

One JSON line per (N, M, steps, arrangement, algorithm, amplitude): seeded
complex Gaussian dual-pol input, 40 x 80 km link, oracle/dbp_port.py float64.
"""
import json
import os
import sys
import warnings
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1507_00921_b200 as pb  # noqa: E402
from oracle import dbp_port, waveforms  # noqa: E402


def main():
    span = pb.FiberParams(-21.68, 1.3, 0.2, 80.0)
    link = pb.LinkConfig(span, 40, amp_noise_figure_db=None, pol_rotation=False)
    rows = []
    for n_blk, m in ((2048, 700), (4096, 1400), (8192, 1024), (1024, 768)):
        for steps in (1, 2, 3, 4, 8, 20):
            for arr in ("symmetric", "linear-first"):
                for alg, nc in (("ssfm", 0), ("essfm", 17)):
                    for amp in (0.01, 0.03):
                        gen = np.random.default_rng(n_blk + steps)
                        n = 6 * (n_blk - m) + 77
                        x = (amp * (gen.normal(size=(2, n)) + 1j * gen.normal(size=(2, n)))).astype(np.complex64)
                        coeffs = pb.EssfmCoefficients(waveforms.gaussian_coeffs(nc)) if alg == "essfm" else None
                        cfg = pb.DbpConfig(alg, pb.OverlapPlan(n_blk, m), link, num_steps=steps, coeffs=coeffs,
                                           arrangement=arr)
                        with warnings.catch_warnings():
                            warnings.simplefilter("ignore")
                            got = pb.backpropagate_batch(x[None], 56e9, cfg)[0]
                        want = dbp_port.backpropagate_arrays(x.astype(np.complex128), 56e9,
                                                             dbp_port.PortConfig.from_objects(cfg))
                        err = float(dbp_port.per_block_rel_l2(got, want, n_blk, m).max())
                        row = dict(fft=os.environ.get("DBP_FFT", "default"), N=n_blk, M=m, steps=steps,
                                   arrangement=arr, algorithm=alg, nc=nc, amp=amp, worst=err)
                        print(json.dumps(row), flush=True)
                        rows.append(row)
    return 0


if __name__ == "__main__":
    sys.exit(main())
