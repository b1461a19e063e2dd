"""Per-block rel-L2 of the GPU path vs the oracle across launch powers (config 2 / config 0 geometry)."""
import sys, warnings
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1507_00921_b200 as pb
from oracle import dbp_port, waveforms

warnings.simplefilter("ignore")
beta2 = waveforms.d_to_beta2(17.0)
n_sym = 2 ** 13
for p_dbm in (-4.0, 0.0, 2.0, 4.0, 6.0):
    tx, _ = waveforms.qpsk_rrc(n_sym, 2, 0.1, seed=3, power_dbm=p_dbm)
    rx = waveforms.forward_link(tx, 56e9, beta2, 1.3 * 8 / 9, 0.2, 80.0, 40, 8)
    x = rx.astype(np.complex64)
    for alg, ns, arr, nc in (("ssfm", 20, "linear-first", 0), ("essfm", 1, "symmetric", 17), ("ssfm", 40, "symmetric", 0)):
        span = pb.FiberParams(beta2, 1.3 * 8 / 9, 0.2, 80.0)
        link = pb.LinkConfig(span, 40, amp_noise_figure_db=None, pol_rotation=False)
        c = pb.EssfmCoefficients(waveforms.gaussian_coeffs(nc)) if alg == "essfm" else None
        cfg = pb.DbpConfig(alg, pb.OverlapPlan(2048, 700), link, num_steps=ns, coeffs=c, arrangement=arr)
        got = pb.backpropagate_batch(x, 56e9, cfg)[0]
        want = dbp_port.backpropagate_arrays(x.astype(np.complex128), 56e9, dbp_port.PortConfig.from_objects(cfg))
        e = dbp_port.per_block_rel_l2(got, want, 2048, 700)
        print(f"P={p_dbm:+.0f} dBm {alg:5s} Ns={ns:2d} {arr:12s} worst={e.max():.3e} median={np.median(e):.3e}", flush=True)
