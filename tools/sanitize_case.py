"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys
import warnings
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1507_00921_b200 as pb  # noqa: E402

warnings.simplefilter("ignore")
rng = np.random.default_rng(0)
span = pb.FiberParams(-21.68, 1.3, 0.2, 80.0)
link = pb.LinkConfig(span, 4, amp_noise_figure_db=None, pol_rotation=False)
cases = [
    ("essfm", 2048, 700, 1, 17, "symmetric", 5000),
    ("essfm", 1024, 300, 2, 9, "linear-first", 3000),
    ("ssfm", 8192, 2048, 2, 0, "nonlinear-first", 9000),
    ("ffe", 4096, 1024, 1, 0, "symmetric", 4100),
    ("essfm", 16, 4, 1, 3, "symmetric", 37),
    ("essfm", 256, 60, 3, 23, "symmetric", 700),
    # the float64 general path (N outside [16, 8192])
    ("essfm", 8, 3, 2, 3, "linear-first", 29),
    ("essfm", 16384, 2000, 1, 17, "symmetric", 20000),
]
for alg, n_blk, m, steps, nc, arr, n in cases:
    c = None
    if alg == "essfm":
        cc = rng.normal(size=nc + 1) * 0.1
        cc[0] = 1.0
        c = pb.EssfmCoefficients(cc)
    cfg = pb.DbpConfig(alg, pb.OverlapPlan(n_blk, m), link, num_steps=steps, coeffs=c, arrangement=arr)
    x = (0.02 * (rng.normal(size=(2, 2, n)) + 1j * rng.normal(size=(2, 2, n)))).astype(np.complex64)
    y = pb.backpropagate_batch(x, 56e9, cfg)
    eng = pb.get_engine(cfg, 56e9, 0)
    part = eng.run_host(x, block_range=(1, max(2, eng.num_blocks(n) - 1))) if eng.num_blocks(n) > 2 else y
    assert np.all(np.isfinite(y))
    print(alg, n_blk, m, steps, nc, arr, n, "ok", flush=True)
sig = pb.DualPolSignal(x[0, 0], x[0, 1], 56e9)
res = pb.optimize_coefficients(sig, pb.DbpConfig("essfm", pb.OverlapPlan(256, 60), link,
                                                 coeffs=pb.EssfmCoefficients.identity(3)),
                               pb.TrainConfig(n_coeffs=3, target_steps_per_span=1, train_samples=700,
                                              max_iterations=1))
print("train ok", res.iterations)
