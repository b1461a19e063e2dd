"""Process-parallel oracle runs for the large parity tests -- TEST INFRASTRUCTURE ONLY.

``backpropagate_many`` runs ``dbp_port.backpropagate_arrays`` on several
independent waveforms in a spawn-context process pool (numpy's FFT is
single-threaded; the reference parallelises the same way, cli.py:811-816).
"""

from __future__ import annotations

import multiprocessing as mp
import os
from concurrent.futures import ProcessPoolExecutor


def _one(args):
    import numpy as np
    from oracle.dbp_port import PortConfig, backpropagate_arrays
    x, rate, kwargs = args
    return backpropagate_arrays(np.asarray(x, dtype=np.complex128), rate, PortConfig(**kwargs))


def port_kwargs(cfg) -> dict:
    """PortConfig keyword arguments from a reference-style DbpConfig."""
    span = cfg.link.span
    return dict(algorithm=cfg.algorithm, block_len=cfg.plan.block_len, overlap=cfg.plan.overlap,
                beta2=span.beta2, gamma=span.gamma, alpha_db_per_km=span.alpha_db_per_km, span_km=span.length,
                num_spans=cfg.link.num_spans, num_steps=cfg.num_steps,
                coeffs=None if cfg.coeffs is None else [float(c) for c in cfg.coeffs.c],
                arrangement=cfg.arrangement)


def backpropagate_many(jobs, workers: int | None = None):
    """jobs: list of (samples (2, n), rate_hz, port kwargs) -> list of float64 outputs."""
    workers = max(1, min(len(jobs), workers or os.cpu_count() or 1))
    if workers == 1:
        return [_one(j) for j in jobs]
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn")) as pool:
        return list(pool.map(_one, jobs))
