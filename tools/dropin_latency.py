"""Latency breakdown of the drop-in call backpropagate(sig, cfg) at small sizes (GPU box)."""
import sys
import time
import warnings
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1507_00921_b200 as pb  # noqa: E402
from oracle import waveforms  # noqa: E402

warnings.simplefilter("ignore")
span = pb.FiberParams(beta2=waveforms.d_to_beta2(17.0), gamma=1.3, alpha_db_per_km=0.2, length=80.0)
link = pb.LinkConfig(span, 40, amp_noise_figure_db=None, pol_rotation=False)
cfg = pb.DbpConfig("essfm", pb.OverlapPlan(2048, 700), link, num_steps=1,
                   coeffs=pb.EssfmCoefficients(waveforms.gaussian_coeffs(17)))
for lg in (12, 14, 17, 20, 24):
    n = 1 << lg
    rng = np.random.default_rng(0)
    x = 0.02 * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n)))
    sig = pb.DualPolSignal(x[0], x[1], 56e9)
    eng = pb.get_engine(cfg, 56e9)
    x64 = x.astype(np.complex64)[None]
    out64 = np.zeros_like(x64)
    ox, oy = np.empty(n, np.complex128), np.empty(n, np.complex128)

    def t(f, k=(300 if lg < 19 else 30) if lg < 22 else 5):
        f()
        t0 = time.perf_counter()
        for _ in range(k):
            f()
        return (time.perf_counter() - t0) / k * 1e6

    a = t(lambda: pb.backpropagate(sig, cfg))
    b = t(lambda: eng.native.backpropagate_c128(sig.x, sig.y, ox, oy))
    c = t(lambda: eng.run_host(x64, out64))
    print(f"n=2^{lg}: backpropagate {a:8.1f} us  native c128 (preallocated out) {b:8.1f} us  run_host c64 {c:8.1f} us"
          f"  -> {n / a / 1e3:.3f} GS/s drop-in (dual-pol samples)")

# a batch of pageable complex64 waveforms through backpropagate_batch (configs[3] shape, reduced batch)
rng = np.random.default_rng(1)
xb = (0.02 * (rng.normal(size=(32, 2, 1 << 18)) + 1j * rng.normal(size=(32, 2, 1 << 18)))).astype(np.complex64)
ob = np.empty_like(xb)
eng = pb.get_engine(cfg, 56e9)
eng.run_host(xb, ob)
t0 = time.perf_counter()
for _ in range(5):
    eng.run_host(xb, ob)
sec = (time.perf_counter() - t0) / 5
print(f"batch 32 x 2^18 pageable complex64 run_host: {sec * 1e3:.2f} ms -> {32 * (1 << 18) / sec / 1e9:.3f} GS/s")
pb.backpropagate_batch(xb, 56e9, cfg)
t0 = time.perf_counter()
for _ in range(5):
    res = pb.backpropagate_batch(xb, 56e9, cfg)
sec = (time.perf_counter() - t0) / 5
print(f"batch 32 x 2^18 pageable complex64 backpropagate_batch (result allocated by the call): {sec * 1e3:.2f} ms -> "
      f"{32 * (1 << 18) / sec / 1e9:.3f} GS/s")
