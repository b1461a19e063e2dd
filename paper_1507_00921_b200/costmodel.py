"""Operation counts and the B200 roofline of the block equalisers.

Two models side by side:

* the reference's analytic cost model (``fiberdbp.costmodel``, costmodel.py:1-166),
  restated so a caller of ``cost_per_sample`` / ``optimize_block_length`` /
  ``sweep_link_length`` / ``cost_table_csv`` finds them here with the same
  arguments, results and ``ValueError``s: real multiplications and additions
  per output sample under the paper's radix-2 bookkeeping (8 N log2 N of each
  per step and polarisation pair, complex multiply = 4 + 2, phase
  exponentials from a table), latency proxied by the cascaded FFT pairs and
  power by the multiplication count;
* the B200 model this package is measured against (SURVEY
  8d): FP32 flops per output sample in the FFTW convention (5 N log2 N per
  complex transform, complex multiply = 6, sincos on the SFU excluded),
  algorithmic HBM bytes per output sample (the block read including its
  overlap plus the kept centre written, complex64, both polarisations), and
  the roofline throughput 1 / max(F / P_fp32, B / BW).  ``bench.py`` takes
  its roofline numbers from here.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable, Sequence

from .backprop import ALGORITHMS, estimate_channel_memory

# nominal FP32 rate of one B200 at 1965 MHz (148 SMs x 128 lanes x 2) and the
# pool's measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs)
B200_FP32_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12
B200_HBM_GBS = 6548.2


def _check_plan(block_len: int, overlap: int) -> None:
    if block_len < 1 or block_len & (block_len - 1):
        raise ValueError(f"block_len must be a power of two, got {block_len}")
    if not 0 <= overlap < block_len:
        raise ValueError("overlap must satisfy 0 <= overlap < block_len")


# ---------------------------------------------------------------------------
# the reference's model (costmodel.py:31-166)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class CostReport:
    """Operation counts of one equaliser configuration (costmodel.py:31-54)."""

    algorithm: str
    block_len: int
    overlap: int
    n_coeffs: int
    num_steps: int
    mults_per_sample: float
    adds_per_sample: float
    latency_proxy: int

    @property
    def mults_rounded(self) -> int:
        return round(self.mults_per_sample)

    @property
    def adds_rounded(self) -> int:
        return round(self.adds_per_sample)

    @property
    def power_proxy(self) -> float:
        return self.mults_per_sample


def cost_per_sample(algorithm: str, block_len: int, overlap: int, n_coeffs: int = 0,
                    num_steps: int = 1) -> CostReport:
    """Closed-form counts per output sample (costmodel.py:57-102).

    FFE: N (8 log2 N + 8) mults and N (8 log2 N + 4) adds per N - M outputs;
    SSFM / ESSFM per step: N (8 log2 N + 21 + Nc) mults and
    N (8 log2 N + 11 + 2 Nc) adds (Nc = 0 for SSFM), times N_s.
    """
    if algorithm not in ALGORITHMS:
        raise ValueError(f"algorithm must be one of {ALGORITHMS}, got {algorithm!r}")
    _check_plan(block_len, overlap)
    if n_coeffs < 0:
        raise ValueError("n_coeffs must be >= 0")
    if num_steps < 1:
        raise ValueError("num_steps must be >= 1")
    per_block = block_len / (block_len - overlap)
    fft_ops = 8.0 * math.log2(block_len)
    if algorithm == "ffe":
        return CostReport("ffe", block_len, overlap, 0, 1, per_block * (fft_ops + 8.0),
                          per_block * (fft_ops + 4.0), latency_proxy=1)
    nc = n_coeffs if algorithm == "essfm" else 0
    return CostReport(algorithm, block_len, overlap, nc, num_steps,
                      num_steps * per_block * (fft_ops + 21.0 + nc),
                      num_steps * per_block * (fft_ops + 11.0 + 2.0 * nc), latency_proxy=num_steps)


def optimize_block_length(algorithm: str, overlap: int, n_coeffs: int = 0,
                          candidates: Iterable[int] = ()) -> tuple[int, CostReport]:
    """The candidate N with the fewest per-step mults per sample, ties to the
    smaller block (costmodel.py:105-126)."""
    cands = sorted({int(c) for c in candidates})
    if not cands:
        raise ValueError("candidate set must be non-empty")
    if cands[0] <= overlap:
        raise ValueError("all candidates must exceed the overlap")
    reports = [(n, cost_per_sample(algorithm, n, overlap, n_coeffs=n_coeffs)) for n in cands]
    return min(reports, key=lambda nr: (nr[1].mults_per_sample, nr[0]))


def sweep_link_length(algorithms: Sequence[str], lengths_km: Sequence[float], beta2_mag: float,
                      bandwidth_hz: float, n_coeffs: int = 0) -> list[CostReport]:
    """Per-step cost against link length, overlap = the estimated channel
    memory and N = 8 x overlap (costmodel.py:129-151)."""
    if any(length <= 0.0 for length in lengths_km):
        raise ValueError("lengths must be positive")
    out = []
    for length in lengths_km:
        m = estimate_channel_memory(beta2_mag, length, bandwidth_hz)
        out.extend(cost_per_sample(alg, 8 * m, m, n_coeffs=n_coeffs) for alg in algorithms)
    return out


def cost_table_csv(reports: Sequence[CostReport]) -> str:
    """CSV rendering; relative_pct against the largest mult count (costmodel.py:154-166)."""
    if not reports:
        raise ValueError("no reports to render")
    top = max(r.mults_per_sample for r in reports)
    rows = ["algorithm,N,M,Nc,Ns,mults_per_sample,adds_per_sample,latency_proxy,relative_pct"]
    rows += [f"{r.algorithm},{r.block_len},{r.overlap},{r.n_coeffs},{r.num_steps},{r.mults_per_sample:.2f},"
             f"{r.adds_per_sample:.2f},{r.latency_proxy},{100.0 * r.mults_per_sample / top:.1f}" for r in reports]
    return "\n".join(rows) + "\n"


# ---------------------------------------------------------------------------
# the B200 roofline
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class RooflineReport:
    """FP32 work and HBM traffic per output sample and the B200 bound."""

    algorithm: str
    arrangement: str
    block_len: int
    overlap: int
    n_coeffs: int
    num_steps: int
    flops_per_sample: float        # FFTW convention
    bytes_per_sample: float        # algorithmic HBM bytes (complex64, both polarisations)
    bound: str                     # "fp32" or "hbm"
    roofline_gsps: float           # 1 / max(F / P, B / BW), Gsamples/s per GPU

    @property
    def intensity(self) -> float:
        """Arithmetic intensity, flops per HBM byte."""
        return self.flops_per_sample / self.bytes_per_sample


def work_per_sample(algorithm: str, block_len: int, overlap: int, n_coeffs: int = 0, num_steps: int = 1,
                    arrangement: str = "symmetric", gains_not_one: bool = False) -> tuple[float, float]:
    """(FP32 flops, HBM bytes) per output sample of one overlap-save program.

    Per block: 20 N log2 N + 12 N per transform pair (two 5 N log2 N complex
    FFTs of each polarisation and the dispersion multiply), N (3 Nc + 21) per
    nonlinear step (intensity 7, FIR 3 Nc + 1, scale 1, two rotations 12),
    4 N per step with a gain != 1; pairs = N_s + 1 (symmetric), N_s
    (linear-first / nonlinear-first) or 1 (FFE).  Bytes: 16 (2 N - M) per
    N - M outputs (block read with its overlap, kept centre written).
    """
    _check_plan(block_len, overlap)
    n, m = block_len, overlap
    lg = math.log2(n)
    if algorithm == "ffe":
        pairs, ns, nc = 1, 0, 0
    else:
        ns = num_steps
        pairs = ns + 1 if arrangement == "symmetric" else ns
        nc = n_coeffs if algorithm == "essfm" else 0
    flops = 20 * pairs * n * lg + 12 * pairs * n + ns * n * (3 * nc + 21) + (4 * n * ns if gains_not_one else 0)
    return flops / (n - m), 16.0 * (2 * n - m) / (n - m)


def b200_roofline(algorithm: str, block_len: int, overlap: int, n_coeffs: int = 0, num_steps: int = 1,
                  arrangement: str = "symmetric", gains_not_one: bool = False,
                  fp32_tflops: float = B200_FP32_TFLOPS, hbm_gbs: float = B200_HBM_GBS) -> RooflineReport:
    """The per-GPU roofline of one configuration."""
    if algorithm not in ALGORITHMS:
        raise ValueError(f"algorithm must be one of {ALGORITHMS}, got {algorithm!r}")
    f, b = work_per_sample(algorithm, block_len, overlap, n_coeffs, num_steps, arrangement, gains_not_one)
    t_fp, t_hbm = f / (fp32_tflops * 1e12), b / (hbm_gbs * 1e9)
    return RooflineReport(algorithm, arrangement if algorithm != "ffe" else "-", block_len, overlap,
                          n_coeffs if algorithm == "essfm" else 0, num_steps if algorithm != "ffe" else 1,
                          f, b, "fp32" if t_fp >= t_hbm else "hbm", 1e-9 / max(t_fp, t_hbm))


def optimize_block_length_b200(algorithm: str, overlap: int, n_coeffs: int = 0, num_steps: int = 1,
                               arrangement: str = "symmetric",
                               candidates: Iterable[int] = (1024, 2048, 4096, 8192)) -> tuple[int, RooflineReport]:
    """The candidate N with the highest B200 roofline throughput (ties to the smaller block)."""
    cands = sorted({int(c) for c in candidates})
    if not cands:
        raise ValueError("candidate set must be non-empty")
    if cands[0] <= overlap:
        raise ValueError("all candidates must exceed the overlap")
    reports = [(n, b200_roofline(algorithm, n, overlap, n_coeffs, num_steps, arrangement)) for n in cands]
    return max(reports, key=lambda nr: (nr[1].roofline_gsps, -nr[0]))
