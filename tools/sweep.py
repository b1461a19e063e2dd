"""Throughput sweep over BASELINE configs[1..3] (device-resident, CUDA-event timed).

    python tools/sweep.py [--waveforms 128] [--reps 20] > profiles/r1/sweep.json

Config 3: N in {1024, 2048, 4096, 8192} with the overlap >= the 3200 km
dispersion memory (1367 samples -> M = 1400; N = 1024 cannot hold it, M = 768
is the signal-band memory of a 30.8 GHz RRC-0.1 channel), N_s in {1, 2, 4},
N_c in {1, 9, 17, 33}, symmetric.  Plus the config-0 geometry (2048/700) in
both arrangements, config 1 FFE at N in {1024, 2048, 4096} (M = 700) and
config 2 SSFM-20 linear-first.  One JSON object per line.
"""

import argparse
import json
import math
import sys
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--waveforms", type=int, default=128)
    ap.add_argument("--log2-samples", type=int, default=18)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()

    import torch

    import bench
    import paper_1507_00921_b200 as pb
    from paper_1507_00921_b200 import _native

    warnings.simplefilter("ignore")
    n = 1 << a.log2_samples
    B = a.waveforms
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(7)
    amp = math.sqrt(1e-3 / 4.0)
    d_in = torch.randn((B, 2, n, 2), generator=gen, device="cuda:0") * amp
    d_out = torch.empty_like(d_in)
    stream = torch.cuda.Stream()
    peak_tf = max(_native.probe_fp32_peak(0, 8192)[0], _native.probe_fp32x2_peak(0, 8192)[0])

    points = []
    overl = {1024: 768, 2048: 1400, 4096: 1400, 8192: 1400}
    for blk in (1024, 2048, 4096, 8192):
        for ns in (1, 2, 4):
            for nc in (1, 9, 17, 33):
                points.append(("essfm", blk, overl[blk], ns, nc, "symmetric", "config3"))
    for arr in ("symmetric", "linear-first"):
        points.append(("essfm", 2048, 700, 1, 17, arr, "config0"))
    for blk in (1024, 2048, 4096):
        points.append(("ffe", blk, 700, 1, 0, "symmetric", "config1"))
    points.append(("ssfm", 2048, 700, 20, 0, "linear-first", "config2"))
    points.append(("ssfm", 8192, 1024, 20, 0, "linear-first", "config2"))
    if a.quick:
        points = [p for p in points if p[6] != "config3" or (p[3] == 1 and p[4] == 17)]

    for alg, blk, m, ns, nc, arr, tag in points:
        args = bench.parse_args(["--algorithm", alg, "--block-len", str(blk), "--overlap", str(m),
                                 "--num-steps", str(ns), "--nc", str(max(nc, 0)), "--arrangement", arr])
        if alg == "ssfm":
            args.nc = 0
        cfg = bench.make_cfg(args)
        eng = pb.get_engine(cfg, bench.SAMPLE_RATE, 0)
        nb = eng.num_blocks(n)
        for _ in range(3):
            eng.native.run_device(d_in.data_ptr(), d_out.data_ptr(), n, B, 0, nb, stream.cuda_stream)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.reps):
            eng.native.run_device(d_in.data_ptr(), d_out.data_ptr(), n, B, 0, nb, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        gss = B * n / (ms * 1e-3) / 1e9
        f_s, b_s = bench.work_per_sample(args, gains_not_one=any(g != 1.0 for _, _, g in eng.schedule))
        row = {"config": tag, "algorithm": alg, "block_len": blk, "overlap": m, "num_steps": ns,
               "n_coeffs": nc, "arrangement": arr, "gsamples_per_s": gss, "ms_per_launch": ms,
               "flops_per_sample": f_s, "tflops": f_s * gss / 1e3, "fp32_frac": f_s * gss / 1e3 / peak_tf,
               "hbm_gbs": b_s * gss, "hbm_frac": b_s * gss / 6555.5, "fp32_peak_tflops": peak_tf,
               "waveforms": B, "samples_per_waveform": n}
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
