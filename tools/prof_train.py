import cProfile, pstats, sys, time, math, io
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import numpy as np
import paper_1507_00921_b200 as pb
from q_vs_power import d_to_beta2, rrc_tx
span = pb.FiberParams(beta2=d_to_beta2(17.0), gamma=1.3, alpha_db_per_km=0.2, length=80.0)
quiet = pb.LinkConfig(span=span, num_spans=40, amp_gain_db=None, amp_noise_figure_db=None, pol_rotation=False)
tx, sym = rrc_tx(1 << 16, seed=0)
x = (tx * math.sqrt(1e-3)).astype(np.complex64)
link = pb.LinkConfig(span=span, num_spans=40, amp_noise_figure_db=5.0, pol_rotation=True)
rx = pb.propagate_link_batch(x[None], 56e9, link, pb.SsfmStepConfig(80), [np.random.SeedSequence([7, 0])])
sig = pb.DualPolSignal(rx[0, 0], rx[0, 1], 56e9)
plan = pb.OverlapPlan(2048, 700)
tcfg = pb.TrainConfig(n_coeffs=17, target_steps_per_span=4, train_samples=16384, max_iterations=10)
geometry = pb.DbpConfig("essfm", plan, quiet, num_steps=1, coeffs=pb.EssfmCoefficients.identity(17))
pb.optimize_coefficients(sig, geometry, tcfg)   # warm
for k in range(2):
    t = time.perf_counter(); r = pb.optimize_coefficients(sig, geometry, tcfg); print("fit", time.perf_counter() - t, r.iterations)
pr = cProfile.Profile(); pr.enable(); pb.optimize_coefficients(sig, geometry, tcfg); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumtime").print_stats(25); print(s.getvalue()[:6000])
