"""Error growth of the GPU link simulator against the float64 oracle (diagnostics).

python tools/diag_sim.py [--fp32-numpy]   (the flag runs a complex64 numpy restatement instead of the GPU)
"""
import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import channel_port as cp  # noqa: E402
from oracle.dbp_port import LN10_OVER_10, bin_frequencies, effective_len  # noqa: E402
from oracle.waveforms import d_to_beta2, qpsk_rrc  # noqa: E402


def numpy32_span(x, fs, beta2, gamma, adb, length, steps, nonlinear):
    n = x.shape[1]
    f = bin_frequencies(n, fs)
    alpha = LN10_OVER_10 * adb
    dz = length / steps
    dze = effective_len(alpha, dz) if alpha > 0 else dz
    lin = np.exp(1j * (-2 * np.pi ** 2 * (beta2 * 1e-24) * f ** 2 * dz)).astype(np.complex64)
    loss = np.float32(np.exp(-alpha * dz / 2))
    cur = x.astype(np.complex64)
    for _ in range(steps):
        cur = np.fft.ifft(np.fft.fft(cur, axis=1) * lin, axis=1).astype(np.complex64)
        if nonlinear:
            p = (np.abs(cur[0]) ** 2 + np.abs(cur[1]) ** 2).astype(np.float32)
            cur = (cur * np.exp(-1j * np.float32(gamma * dze) * p).astype(np.complex64)).astype(np.complex64)
        cur = (cur * loss).astype(np.complex64)
    return cur


def main():
    use_np = "--fp32-numpy" in sys.argv
    if not use_np:
        import paper_1507_00921_b200 as pb
    beta2 = d_to_beta2(17.0)
    tx, _ = qpsk_rrc(2 ** 13, seed=0, power_dbm=0.0)
    x = tx.astype(np.complex64)
    for nl in (False, True):
        for spans in (1, 5, 40):
            steps = 80
            want = x.astype(np.complex128)
            for _ in range(spans):
                want = cp.span(want, 56e9, beta2, 1.3, 0.2, 80.0, steps, nl) * 10 ** (0.2 * 80 / 20)
            if use_np:
                got = x
                for _ in range(spans):
                    got = numpy32_span(got, 56e9, beta2, 1.3, 0.2, 80.0, steps, nl) * np.float32(10 ** (0.8))
            else:
                link = pb.LinkConfig(span=pb.FiberParams(beta2, 1.3, 0.2, 80.0), num_spans=spans,
                                     amp_noise_figure_db=None, pol_rotation=False)
                got = pb.propagate_link(pb.DualPolSignal(x[0], x[1], 56e9), link,
                                        pb.SsfmStepConfig(steps, nl)).stack()
            d = got - want
            scale = np.vdot(want, got) / np.vdot(want, want)
            err = np.linalg.norm(d) / np.linalg.norm(want)
            print(f"{'np32' if use_np else 'gpu '} nl={int(nl)} spans={spans:2d} rel-L2 {err:.2e}  "
                  f"gain-err {abs(scale) - 1:+.2e} phase-err {np.angle(scale):+.2e}  "
                  f"after common-scale {np.linalg.norm(got / scale - want) / np.linalg.norm(want):.2e}")


if __name__ == "__main__":
    main()
