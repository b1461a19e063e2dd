"""Random host-pipeline cases: pageable complex64 rows (dbp_run_host staged through pinned
memory) and complex128 rows (dbp_backpropagate_c128) against the same plan's device-resident
run (dbp_run on a torch buffer) -- bit for bit, at signal lengths tools/fuzz_parity.py does
not reach (2^16 .. 2^20 samples: block-range chunks, whole items, mixed batches)."""
import argparse
import json
import sys
import time
import warnings
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1507_00921_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=120)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--out", default=None)
a = ap.parse_args()
warnings.simplefilter("ignore")
gen = np.random.default_rng(a.seed)
t0 = time.time()
res = {"cases": 0, "mismatches": 0, "bad": []}
for case in range(a.cases):
    logn = int(gen.integers(9, 16))                     # 512 .. 32768 (the last two: the general path)
    nb = 1 << logn
    m = int(gen.integers(0, nb - nb // 8))
    n = int(gen.integers(1 << 16, (1 << 20) + 1)) if gen.random() < 0.8 else int(gen.integers(1, 1 << 16))
    batch = int(gen.integers(1, 7))
    if batch * n > 3 << 20:
        batch = max(1, (3 << 20) // n)
    alg = ("ffe", "ssfm", "essfm")[int(gen.integers(0, 3))]
    steps = int(gen.integers(1, 4))
    arr = pb.ARRANGEMENTS[int(gen.integers(0, 3))]
    coeffs = None
    if alg == "essfm":
        nc = (1, 9, 17, 33, 5)[int(gen.integers(0, 5))]
        coeffs = pb.EssfmCoefficients(np.r_[1.0, 0.05 * gen.normal(size=nc)])
    span = pb.FiberParams(-21.68, 1.3, 0.2, 80.0)
    link = pb.LinkConfig(span, int(gen.integers(1, 5)), amp_noise_figure_db=None, pol_rotation=False)
    cfg = pb.DbpConfig(alg, pb.OverlapPlan(nb, m), link, num_steps=steps, coeffs=coeffs, arrangement=arr)
    x = (0.02 * (gen.normal(size=(batch, 2, n)) + 1j * gen.normal(size=(batch, 2, n)))).astype(np.complex64)
    eng = pb.get_engine(cfg, 56e9)
    d_in = torch.from_numpy(x.view(np.float32)).cuda()
    d_out = torch.empty_like(d_in)
    with eng.native.lock:
        eng.native.run_device(d_in.data_ptr(), d_out.data_ptr(), n, batch, 0, eng.num_blocks(n),
                              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    want = d_out.cpu().numpy().view(np.complex64).reshape(batch, 2, n)
    got = eng.run_host(x)                                # pageable rows
    ok = np.array_equal(got, want)
    one = pb.backpropagate(pb.DualPolSignal(x[0, 0], x[0, 1], 56e9), cfg).stack()   # complex128 rows
    ok = ok and np.array_equal(one, want[0].astype(np.complex128))
    res["cases"] += 1
    if not ok:
        res["mismatches"] += 1
        res["bad"].append(dict(alg=alg, N=nb, M=m, n=n, batch=batch, steps=steps, arrangement=arr))
res["seconds"] = round(time.time() - t0, 1)
print(json.dumps(res))
if a.out:
    Path(a.out).write_text(json.dumps(res, indent=1))
