"""CPU baseline runner for bench.py -- TEST/MEASUREMENT INFRASTRUCTURE ONLY.

Times the oracle port (a restatement of the reference's float64 numpy DBP,
pkg/src/fiberdbp/dbp.py:160-235) on the host cores: one process per core,
each running whole waveforms through ``backpropagate_arrays`` with numpy's
single-threaded pocketfft, mirroring the reference's own process-level
parallelism (pkg/src/fiberdbp/cli.py:811-816).  Inputs are seeded complex
Gaussian dual-pol waveforms at the bench's launch power.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np

from .dbp_port import PortConfig, backpropagate_arrays


def make_waveform(seed: int, n: int, power_dbm: float) -> np.ndarray:
    rng = np.random.default_rng(seed)
    amp = math.sqrt(10.0 ** ((power_dbm - 30.0) / 10.0) / 4.0)
    x = amp * (rng.standard_normal((2, n)) + 1j * rng.standard_normal((2, n)))
    return x.astype(np.complex64).astype(np.complex128)


def _work(args):
    seed, n, power_dbm, cfg_kwargs, rate = args
    x = make_waveform(seed, n, power_dbm)
    cfg = PortConfig(**cfg_kwargs)
    t0 = time.perf_counter()
    backpropagate_arrays(x, rate, cfg)
    return time.perf_counter() - t0


def _init_worker():
    os.environ.setdefault("OMP_NUM_THREADS", "1")


class CpuBaseline:
    """A pool of ``cores`` single-threaded workers timing the oracle port."""

    def __init__(self, cfg_kwargs: dict, rate: float, n: int, power_dbm: float, cores: int | None = None):
        import multiprocessing as mp

        self.cores = int(cores or os.cpu_count() or 1)
        self.cfg_kwargs = dict(cfg_kwargs)
        self.rate = float(rate)
        self.n = int(n)
        self.power_dbm = float(power_dbm)
        ctx = mp.get_context("spawn")
        self.pool = ctx.Pool(self.cores, initializer=_init_worker)
        # warm every worker (imports, numpy FFT plan caches)
        self.pool.map(_work, [(i, min(self.n, 1 << 14), self.power_dbm, self.cfg_kwargs, self.rate)
                              for i in range(self.cores)])

    def step(self, waveforms: int, seed0: int = 0) -> tuple[float, float]:
        """Process ``waveforms`` waveforms across the pool; returns (wall s, samples)."""
        jobs = [(seed0 + i, self.n, self.power_dbm, self.cfg_kwargs, self.rate) for i in range(waveforms)]
        t0 = time.perf_counter()
        self.job_seconds = self.pool.map(_work, jobs, chunksize=1)
        return time.perf_counter() - t0, float(waveforms * self.n)

    def one_core_rate(self) -> float:
        """Samples/s of one core: the median per-waveform time of the last step (each job is one process)."""
        return float(self.n / np.median(self.job_seconds))

    def close(self):
        self.pool.close()
        self.pool.join()
