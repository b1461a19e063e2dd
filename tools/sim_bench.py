"""Throughput of the GPU link simulator against the CPU oracle.

python tools/sim_bench.py [--out profiles/r1/sim_bench.json]

Metric: dual-polarisation sample-steps per second (one SSFM step over one
complex sample of both polarisations), 80 km spans of 80 steps (1 km, the
reference experiments' step size), batch 1 waveform, fully device resident;
each ``dbp_sim_span`` call is timed on the host around the blocking call
(the call ends with a stream synchronize).  Algorithmic traffic per
single-polarisation sample per step: column layout (2^11 <= n <= 2^21) 64
bytes (row kernel B: data r+w 16, double-float dispersion table 16, W_n
table 8; column kernel CA: 16 + W_n 8); transposed layout 96 bytes (the
same plus two transposes, 32).  CPU baseline: oracle/channel_port.span (numpy
complex128 pocketfft, one thread) on a bounded sample.
"""
import argparse
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--logs", default="14,17,20,21,22")
    ap.add_argument("--steps", type=int, default=80)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--batches", default="1")
    args = ap.parse_args()
    import paper_1507_00921_b200 as pb
    from paper_1507_00921_b200 import _native
    from paper_1507_00921_b200.forward import _SimCache
    from oracle import channel_port as cp
    from oracle.waveforms import d_to_beta2

    beta2 = d_to_beta2(17.0)
    fiber = pb.FiberParams(beta2, 1.3, 0.2, 80.0)
    cfg = pb.SsfmStepConfig(args.steps)
    from paper_1507_00921_b200.forward import _span_args
    dz, dz_eff, loss = _span_args(fiber, cfg)
    rows = []
    peaks = json.loads(Path("MEASURED_PEAKS.json").read_text()) if Path("MEASURED_PEAKS.json").exists() else {}
    for lg in [int(v) for v in args.logs.split(",")]:
      for batch in [int(v) for v in args.batches.split(",")]:
        n = 1 << lg
        if batch * n > (1 << 24):
            continue
        rng = np.random.default_rng(lg)
        x = ((rng.normal(size=(batch, 2, n)) + 1j * rng.normal(size=(batch, 2, n))) * 0.02).astype(np.complex64)
        sim = _SimCache.get(0, lg, batch)
        sim.upload(x)
        sim.span(batch, 56e9, beta2, 1.3, dz, dz_eff, loss, args.steps, True)   # warm-up + tables
        times = []
        for _ in range(args.reps):
            t0 = time.perf_counter()
            sim.span(batch, 56e9, beta2, 1.3, dz, dz_eff, loss, args.steps, True)
            times.append(time.perf_counter() - t0)
        t = float(np.median(times))
        per_step = t / args.steps
        rate = batch * n * args.steps / t
        forced_t = os.environ.get("DBP_SIM_TRANSPOSE") == "1"
        block = lg <= 12 and not forced_t and os.environ.get("DBP_SIM_NO_BLOCK") != "1"
        column = not block and 11 <= lg <= 21 and not forced_t
        # block mode keeps the waveform on-chip for the whole span: 16 B per pol-sample per span
        # (load + store) plus the 16-byte table per step
        traffic = ((16.0 + 16.0 * args.steps) / args.steps if block else 64.0 if column else 96.0) * 2 * n * batch
        rows.append(dict(log2_n=lg, batch=batch, layout="block" if block else "column" if column else "transposed",
                         bytes_per_pol_sample_step=round(traffic / (2 * n * batch), 2), ms_per_span=t * 1e3, us_per_step=per_step * 1e6,
                         sample_steps_per_s=rate, effective_GBps=traffic / per_step / 1e9))
        print(json.dumps(rows[-1]))
    # CPU oracle on a bounded sample: 2^17 samples, 4 steps
    n = 1 << 17
    rng = np.random.default_rng(0)
    x = (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n))) * 0.02
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < 10.0:
        cp.span(x, 56e9, beta2, 1.3, 0.2, 80.0 * 4 / args.steps, 4)
        reps += 1
    tc = (time.perf_counter() - t0) / reps
    cpu = dict(value=n * 4 / tc, unit="sample-steps/s", cores=1, kind="port",
               sample=f"oracle/channel_port.span, 2^17 samples x 4 steps, {reps} reps")
    print(json.dumps(dict(cpu_baseline=cpu)))
    out = dict(metric="link simulator throughput", unit="dual-pol sample-steps/s", steps_per_span=args.steps,
               span_km=80.0, rows=rows, cpu_baseline=cpu,
               hbm_peak_GBps=peaks.get("hbm_gbs"))
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
