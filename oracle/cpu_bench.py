"""CPU baseline runner for bench.py -- TEST/MEASUREMENT INFRASTRUCTURE ONLY.

Times the reference's own DBP on the host cores: one single-threaded process
per core, each running whole waveforms through ``fiberdbp.dbp.backpropagate``
(pkg/src/fiberdbp/dbp.py:160), mirroring the reference's process-level
parallelism (pkg/src/fiberdbp/cli.py:811-816).

``kind="reference"`` imports the UNMODIFIED reference package from
``oracle/_ref`` (installed by ``oracle/install_ref.sh``; it travels to the
GPU box with the snapshot).  ``kind="port"`` times the oracle restatement
``oracle/dbp_port.py`` (bit-identical outputs, ~17% slower) and is used only
when ``oracle/_ref`` is absent.  Inputs are seeded complex Gaussian dual-pol
waveforms at the bench's launch power.
"""

from __future__ import annotations

import math
import os
import sys
import time
import warnings
from pathlib import Path

import numpy as np

REF_DIR = Path(__file__).resolve().parent / "_ref"


def reference_available() -> bool:
    return (REF_DIR / "fiberdbp" / "dbp.py").exists()


def make_waveform(seed: int, n: int, power_dbm: float) -> np.ndarray:
    rng = np.random.default_rng(seed)
    amp = math.sqrt(10.0 ** ((power_dbm - 30.0) / 10.0) / 4.0)
    x = amp * (rng.standard_normal((2, n)) + 1j * rng.standard_normal((2, n)))
    return x.astype(np.complex64).astype(np.complex128)


_REF_CACHE: dict = {}


def _reference_runner(cfg_kwargs: dict, rate: float):
    """(fiberdbp module, DbpConfig) built from the port kwargs, cached per worker."""
    key = repr(sorted((k, repr(v)) for k, v in cfg_kwargs.items()))
    if key not in _REF_CACHE:
        if str(REF_DIR) not in sys.path:
            sys.path.insert(0, str(REF_DIR))
        import fiberdbp
        from fiberdbp import dbp as ref_dbp

        k = cfg_kwargs
        span = fiberdbp.FiberParams(k["beta2"], k["gamma"], k["alpha_db_per_km"], k["span_km"])
        link = fiberdbp.LinkConfig(span, k["num_spans"], amp_noise_figure_db=None, pol_rotation=False)
        coeffs = fiberdbp.EssfmCoefficients(np.asarray(k["coeffs"])) if k.get("coeffs") is not None else None
        cfg = fiberdbp.DbpConfig(k["algorithm"], fiberdbp.OverlapPlan(k["block_len"], k["overlap"]), link,
                                 num_steps=k["num_steps"], coeffs=coeffs, arrangement=k["arrangement"])
        _REF_CACHE[key] = (fiberdbp, ref_dbp, cfg)
    return _REF_CACHE[key]


def run_reference_once(x: np.ndarray, rate: float, cfg_kwargs: dict) -> np.ndarray:
    """fiberdbp.dbp.backpropagate on one (2, n) complex128 waveform (jobs=1)."""
    fiberdbp, ref_dbp, cfg = _reference_runner(cfg_kwargs, rate)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")   # the short-overlap UserWarning (dbp.py:175-181)
        out = ref_dbp.backpropagate(fiberdbp.DualPolSignal(x[0], x[1], rate), cfg)
    return out.stack()


def _work(args):
    seed, n, power_dbm, cfg_kwargs, rate, kind = args
    x = make_waveform(seed, n, power_dbm)
    if kind == "reference":
        t0 = time.perf_counter()
        run_reference_once(x, rate, cfg_kwargs)
        return time.perf_counter() - t0
    from .dbp_port import PortConfig, backpropagate_arrays
    cfg = PortConfig(**cfg_kwargs)
    t0 = time.perf_counter()
    backpropagate_arrays(x, rate, cfg)
    return time.perf_counter() - t0


def _init_worker():
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_cpu_bench")


class CpuBaseline:
    """A pool of ``cores`` single-threaded workers timing the reference DBP."""

    def __init__(self, cfg_kwargs: dict, rate: float, n: int, power_dbm: float, cores: int | None = None,
                 kind: str | None = None):
        import multiprocessing as mp

        self.kind = kind or ("reference" if reference_available() else "port")
        if self.kind == "reference" and not reference_available():
            raise RuntimeError("oracle/_ref is missing: run oracle/install_ref.sh")
        self.cores = int(cores or os.cpu_count() or 1)
        self.cfg_kwargs = dict(cfg_kwargs)
        if self.cfg_kwargs.get("coeffs") is not None:
            self.cfg_kwargs["coeffs"] = [float(c) for c in self.cfg_kwargs["coeffs"]]
        self.rate = float(rate)
        self.n = int(n)
        self.power_dbm = float(power_dbm)
        ctx = mp.get_context("spawn")
        os.environ.setdefault("OMP_NUM_THREADS", "1")
        self.pool = ctx.Pool(self.cores, initializer=_init_worker)
        # warm every worker (imports, numpy FFT plan caches)
        self.pool.map(_work, [(i, min(self.n, 1 << 14), self.power_dbm, self.cfg_kwargs, self.rate, self.kind)
                              for i in range(self.cores)])

    def describe(self) -> str:
        if self.kind == "reference":
            return ("fiberdbp.dbp.backpropagate (the unmodified reference, oracle/_ref), float64 numpy "
                    f"(pocketfft), {self.cores} single-threaded processes")
        return f"oracle/dbp_port.py float64 numpy (pocketfft), {self.cores} single-threaded processes"

    def step(self, waveforms: int, seed0: int = 0) -> tuple[float, float]:
        """Process ``waveforms`` waveforms across the pool; returns (wall s, samples)."""
        jobs = [(seed0 + i, self.n, self.power_dbm, self.cfg_kwargs, self.rate, self.kind)
                for i in range(waveforms)]
        t0 = time.perf_counter()
        self.job_seconds = self.pool.map(_work, jobs, chunksize=1)
        return time.perf_counter() - t0, float(waveforms * self.n)

    def one_core_rate(self) -> float:
        """Samples/s of one core: the median per-waveform time of the last step (each job is one process)."""
        return float(self.n / np.median(self.job_seconds))

    def close(self):
        self.pool.close()
        self.pool.join()
