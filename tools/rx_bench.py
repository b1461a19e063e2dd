"""Throughput of the GPU receiver DSP against the CPU restatement.

python tools/rx_bench.py [--out profiles/r1/rx_bench.json]

Workload: the receiver chain of cli.py:677-685 (CMA 15 taps, 2 passes ->
carrier recovery with the reference search -> decisions -> BER) on B
waveforms of 2^16 symbols x 2 samples/symbol (BASELINE configs' symbol
count), noisy RRC QPSK with a per-waveform polarisation rotation.  GPU: one
``receive_batch`` call (host buffers in, metrics out), median of 3.  CPU:
oracle/rx_port.py (the CMA loop numba-jitted, as the reference does) on one
waveform, one core.
"""
import argparse
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--batches", default="1,16,64,148,296")
    ap.add_argument("--log-symbols", type=int, default=16)
    args = ap.parse_args()
    import paper_1507_00921_b200 as pb
    from oracle import rx_port
    from oracle.waveforms import qpsk_rrc
    m = 1 << args.log_symbols
    tx, sym = qpsk_rrc(m, seed=3)
    rng = np.random.default_rng(1)
    bmax = max(int(b) for b in args.batches.split(","))
    xs = np.empty((bmax, 2, 2 * m), dtype=np.complex64)
    p = math.sqrt(np.mean(np.abs(tx) ** 2))
    for i in range(bmax):
        th = 0.37 * i
        j = np.array([[math.cos(th), math.sin(th)], [-math.sin(th), math.cos(th)]])
        xs[i] = j @ tx + 0.05 * p * (rng.normal(size=tx.shape) + 1j * rng.normal(size=tx.shape))
    rows = []
    for b in [int(v) for v in args.batches.split(",")]:
        pb.receive_batch(xs[:b], 28e9, sym)   # warm-up (plans, buffers)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            mets = pb.receive_batch(xs[:b], 28e9, sym)
            ts.append(time.perf_counter() - t0)
        t = float(np.median(ts))
        assert all(not isinstance(x, Exception) for x in mets)
        rows.append(dict(batch=b, seconds=t, waveforms_per_s=b / t, symbols_per_s=2 * m * b / t,
                         ber_mean=float(np.mean([x.ber for x in mets]))))
        print(json.dumps(rows[-1]))
    rx_port.equalize(xs[0, :, :64].astype(np.complex128))   # jit warm-up
    t0 = time.perf_counter()
    eq, _, _ = rx_port.equalize(xs[0].astype(np.complex128))
    rec, _, _ = rx_port.carrier(eq, 28e9, sym)
    errors, counted = rx_port.count_errors(rx_port.decide(rec), rx_port.decide(sym))
    tc = time.perf_counter() - t0
    cpu = dict(value=1.0 / tc, unit="waveforms/s", cores=1, kind="port",
               sample=f"oracle/rx_port (numba CMA) on 1 waveform of 2^{args.log_symbols} symbols",
               seconds=tc, ber=errors / (2 * counted), jitted=rx_port.JITTED)
    print(json.dumps(dict(cpu_baseline=cpu)))
    if args.out:
        Path(args.out).write_text(json.dumps(dict(metric="receiver chain throughput", unit="waveforms/s",
                                                  symbols_per_waveform=m, rows=rows, cpu_baseline=cpu), indent=1))


if __name__ == "__main__":
    main()
