"""Print the worst per-block rel-L2 of every golden case and a few variants (GPU diagnostic)."""
import json, sys, warnings
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1507_00921_b200 as pb
from oracle import dbp_port
from tests.helpers import case_config, port_config, quiet_link

g = np.load("tests/golden/golden_v1.npz"); man = json.load(open("tests/golden/golden_v1.json"))
warnings.simplefilter("ignore")
for case in man["cases"]:
    name = case["name"]
    if case["signal"] == "white":
        x = g[f"bp_{name}_in"]; c = g[f"bp_{name}_c"] if f"bp_{name}_c" in g.files else None; want = g[f"bp_{name}_out"]
    else:
        x = g["link_rx"]; c = g["link_c17"] if case["algorithm"] == "essfm" else None; want = g[f"link_{name}_out"]
    cfg = case_config(case, c)
    got = pb.backpropagate_batch(x, 56e9, cfg)[0]
    e = dbp_port.per_block_rel_l2(got, want, case["block_len"], case["overlap"])
    print(f"{name:12s} N={case['block_len']:5d} alg={case['algorithm']:5s} arr={case['arrangement']:15s} Ns={case['num_steps']} worst={e.max():.3e}")
rng = np.random.default_rng(0)
STD = pb.FiberParams(-21.0, 1.3, 0.2, 40.0)
for N in (16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192):
    for alg, arr, steps, spans in [("ssfm", "symmetric", 1, 1), ("ssfm", "symmetric", 2, 2), ("ssfm", "linear-first", 1, 1), ("ssfm", "symmetric", 3, 2), ("ffe", "symmetric", 1, 1)]:
        n = 3 * N
        x = (0.05 * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n)))).astype(np.complex64)
        cfg = pb.DbpConfig(alg, pb.OverlapPlan(N, N // 4), quiet_link(spans, STD), num_steps=steps, arrangement=arr)
        got = pb.backpropagate_batch(x, 56e9, cfg)[0]
        want = dbp_port.backpropagate_arrays(x.astype(np.complex128), 56e9, port_config(cfg))
        e = dbp_port.per_block_rel_l2(got, want, N, N // 4)
        print(f"N={N:5d} {alg} {arr:13s} Ns={steps} spans={spans} worst={e.max():.3e}")
