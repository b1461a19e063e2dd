"""CPU oracle for the DBP hot path -- TEST INFRASTRUCTURE ONLY.

This module is a float64/complex128 numpy restatement of the reference
``fiberdbp`` digital-backpropagation path (overlap-and-save framing, the
FFE / SSFM / ESSFM block operators and the reverse step schedule).  It is the
checker the GPU product is compared against and the "port" CPU baseline that
``bench.py --impl reference`` times.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import it;
the product package (``paper_1507_00921_b200``) never does.

Parity pin: ``tests/test_oracle_golden.py`` checks every function here
against fixtures in ``tests/golden/`` that ``tests/golden/make_golden.py``
produced by importing the reference package itself, and against the
reference tests' own known answers (channel-memory values, schedule
identities, nested-loop ESSFM oracle).

All citations are ``path:line`` under the reference's ``pkg/src/fiberdbp``.
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

ALGORITHMS = ("ffe", "ssfm", "essfm")                      # dbp.py:25
ARRANGEMENTS = ("symmetric", "linear-first", "nonlinear-first")  # dbp.py:32

LN10_OVER_10 = math.log(10.0) / 10.0                        # sigkit.py:21,34-36


# ---------------------------------------------------------------------------
# scalar helpers
# ---------------------------------------------------------------------------

def memory_in_samples(beta2: float, length_km: float, rate_hz: float) -> float:
    """2 pi |beta2| L B^2 with beta2 in ps^2/km (dbp.py:35-41)."""
    if length_km <= 0.0:
        raise ValueError("length must be positive")
    if rate_hz <= 0.0:
        raise ValueError("bandwidth must be positive")
    return 2.0 * math.pi * abs(beta2) * 1e-24 * length_km * rate_hz ** 2


def pow2_ceil(v: float) -> int:
    """Smallest power of two >= v, at least 1 (spectral.py:24-29)."""
    p = 1
    while p < v:
        p <<= 1
    return p


def bin_frequencies(n: int, rate_hz: float) -> np.ndarray:
    """numpy fftfreq grid in Hz (spectral.py:51-60)."""
    k = np.arange(n)
    k = np.where(k < (n + 1) // 2, k, k - n)
    return k * (rate_hz / n)


def effective_len(alpha: float, dz: float) -> float:
    """(1 - exp(-alpha dz)) / alpha with the small-argument series (sigkit.py:186-212)."""
    if alpha == 0.0:
        return dz
    u = alpha * dz
    if u < 1e-8:
        return dz * (1.0 - u / 2.0 + u * u / 6.0)
    return (1.0 - math.exp(-u)) / alpha


# ---------------------------------------------------------------------------
# reverse step schedule (dbp.py:112-157)
# ---------------------------------------------------------------------------

def step_table(alpha_db_per_km: float, span_km: float, n_spans: int, num_steps: int):
    """Per reverse step (dz, weight, gain) in processing order.

    Segment j covers span coordinates [(j-1) S / Ns, j S / Ns] (exact
    rationals); the weight is the forward power-profile integral over the
    segment divided by the profile just after its far end, the gain is
    sqrt(profile(a) / profile(b)).  Profile is 1 at amplifier outputs
    (integer span coordinates) and exp(-alpha * local distance) inside.
    """
    alpha = LN10_OVER_10 * alpha_db_per_km
    dz = span_km * n_spans / num_steps

    def level_after(pos: Fraction) -> float:
        if pos.denominator == 1:
            return 1.0
        local = float(pos - math.floor(pos)) * span_km
        return math.exp(-alpha * local)

    def integral(lo_pos: Fraction, hi_pos: Fraction) -> float:
        acc = 0.0
        span_idx = math.floor(lo_pos)
        while span_idx < hi_pos:
            a = max(lo_pos, Fraction(span_idx))
            b = min(hi_pos, Fraction(span_idx + 1))
            za = float(a - span_idx) * span_km
            zb = float(b - span_idx) * span_km
            acc += (math.exp(-alpha * za) - math.exp(-alpha * zb)) / alpha if alpha > 0.0 else zb - za
            span_idx += 1
        return acc

    rows = []
    for j in range(num_steps, 0, -1):
        lo_pos = Fraction((j - 1) * n_spans, num_steps)
        hi_pos = Fraction(j * n_spans, num_steps)
        end_level = level_after(hi_pos)
        rows.append((dz, integral(lo_pos, hi_pos) / end_level,
                     math.sqrt(level_after(lo_pos) / end_level)))
    return rows


# ---------------------------------------------------------------------------
# block operators
# ---------------------------------------------------------------------------

def dispersion_response(n: int, rate_hz: float, beta2: float, length_km: float) -> np.ndarray:
    """exp(+j 2 pi^2 beta2 f^2 L), the inverse-dispersion filter (dbp.py:186, 196-197)."""
    f = bin_frequencies(n, rate_hz)
    return np.exp(1j * 2.0 * np.pi ** 2 * (beta2 * 1e-24) * f ** 2 * length_km)


def filter_block(block: np.ndarray, response: np.ndarray) -> np.ndarray:
    """ifft(fft(block) * H) along the sample axis (dbp.py:188-189; spectral.py:37-48)."""
    return np.fft.ifft(np.fft.fft(block, axis=-1) * response, axis=-1)


def filtered_intensity(block: np.ndarray, c: np.ndarray) -> np.ndarray:
    """c0 I_k + sum_i c_i (I_{k-i} + I_{k+i}), cyclic inside the block (dbp.py:71-74)."""
    power = np.abs(block[0]) ** 2 + np.abs(block[1]) ** 2
    n = power.size
    k = np.arange(n)
    acc = c[0] * power
    for i in range(1, c.size):
        acc = acc + c[i] * (power[(k - i) % n] + power[(k + i) % n])
    return acc


def rotate_essfm(block: np.ndarray, gamma: float, dz_eff: float, c: np.ndarray) -> np.ndarray:
    """block * exp(-j gamma dz_eff F) with F the filtered intensity (dbp.py:49-75)."""
    block = np.asarray(block)
    if block.ndim != 2 or block.shape[0] != 2:
        raise ValueError("expected a (2, n) dual-polarization block")
    c = np.asarray(c, dtype=np.float64)
    if block.shape[1] <= 2 * (c.size - 1):
        raise ValueError(
            f"block length {block.shape[1]} too short for {c.size - 1} side coefficients")
    return block * np.exp(-1j * gamma * dz_eff * filtered_intensity(block, c))


def rotate_ssfm(block: np.ndarray, gamma: float, dz_eff: float) -> np.ndarray:
    """block * exp(-j gamma dz_eff (|x|^2 + |y|^2)) (channel.py:61-71)."""
    block = np.asarray(block)
    if block.ndim != 2 or block.shape[0] != 2:
        raise ValueError("expected a (2, n) dual-polarization block")
    power = np.abs(block[0]) ** 2 + np.abs(block[1]) ** 2
    return block * np.exp(-1j * gamma * dz_eff * power)


# ---------------------------------------------------------------------------
# overlap-and-save framing (spectral.py:87-145)
# ---------------------------------------------------------------------------

def count_blocks(n_total: int, block_len: int, overlap: int) -> int:
    step = block_len - overlap
    return -(-n_total // step)


def cut_blocks(samples: np.ndarray, block_len: int, overlap: int) -> np.ndarray:
    """(2, n) circular signal -> (nb, 2, N) blocks; block b starts at b*step - M//2."""
    n_total = samples.shape[1]
    step = block_len - overlap
    lead = overlap // 2
    nb = count_blocks(n_total, block_len, overlap)
    starts = np.arange(nb) * step - lead
    idx = (starts[:, None] + np.arange(block_len)[None, :]) % n_total
    return np.ascontiguousarray(np.transpose(samples[:, idx], (1, 0, 2)))


def join_blocks(blocks: np.ndarray, n_total: int, overlap: int) -> np.ndarray:
    """Keep [M//2, M//2 + step) of each processed block and trim to n (spectral.py:138-145)."""
    nb, _, block_len = blocks.shape
    step = block_len - overlap
    lead = overlap // 2
    kept = blocks[:, :, lead:lead + step]                    # (nb, 2, step)
    return np.transpose(kept, (1, 0, 2)).reshape(2, nb * step)[:, :n_total]


# ---------------------------------------------------------------------------
# the whole path (dbp.py:160-235)
# ---------------------------------------------------------------------------

class PortConfig:
    """Plain-value mirror of ``DbpConfig`` + ``LinkConfig`` fields the path reads."""

    def __init__(self, algorithm, block_len, overlap, beta2, gamma, alpha_db_per_km,
                 span_km, num_spans, num_steps=1, coeffs=None, arrangement="symmetric"):
        if algorithm not in ALGORITHMS:
            raise ValueError(f"algorithm must be one of {ALGORITHMS}, got {algorithm!r}")
        if arrangement not in ARRANGEMENTS:
            raise ValueError(f"arrangement must be one of {ARRANGEMENTS}, got {arrangement!r}")
        if num_steps < 1:
            raise ValueError("num_steps must be >= 1")
        self.algorithm = algorithm
        self.block_len = int(block_len)
        self.overlap = int(overlap)
        self.beta2 = float(beta2)
        self.gamma = float(gamma)
        self.alpha_db_per_km = float(alpha_db_per_km)
        self.span_km = float(span_km)
        self.num_spans = int(num_spans)
        self.num_steps = int(num_steps)
        self.coeffs = None if coeffs is None else np.asarray(coeffs, dtype=np.float64)
        self.arrangement = arrangement
        if algorithm == "essfm" and self.coeffs is None:
            raise ValueError("essfm requires a coefficient set")

    @classmethod
    def from_objects(cls, cfg) -> "PortConfig":
        """Build from any object exposing the reference ``DbpConfig`` fields."""
        span = cfg.link.span
        coeffs = None if cfg.coeffs is None else np.asarray(cfg.coeffs.c)
        return cls(cfg.algorithm, cfg.plan.block_len, cfg.plan.overlap, span.beta2,
                   span.gamma, span.alpha_db_per_km, span.length, cfg.link.num_spans,
                   cfg.num_steps, coeffs, cfg.arrangement)

    @property
    def total_length(self) -> float:
        return self.span_km * self.num_spans


def block_operator(cfg: PortConfig, rate_hz: float):
    """The per-block closure ``process`` of dbp.py:185-233, as a function of one (2, N) block."""
    n = cfg.block_len
    if cfg.algorithm == "ffe":
        h_total = dispersion_response(n, rate_hz, cfg.beta2, cfg.total_length)
        return lambda blk: filter_block(blk, h_total)

    rows = step_table(cfg.alpha_db_per_km, cfg.span_km, cfg.num_spans, cfg.num_steps)
    dz = rows[0][0]
    h_full = dispersion_response(n, rate_hz, cfg.beta2, dz)
    h_half = dispersion_response(n, rate_hz, cfg.beta2, 0.5 * dz)
    neg_gamma = -cfg.gamma
    if cfg.algorithm == "essfm":
        c = cfg.coeffs

        def nl(blk, w):
            return rotate_essfm(blk, neg_gamma, w, c)
    else:
        def nl(blk, w):
            return rotate_ssfm(blk, neg_gamma, w)

    last = len(rows) - 1
    arrangement = cfg.arrangement

    def run(blk):
        cur = blk
        if arrangement == "symmetric":
            cur = filter_block(cur, h_half)
            for j, (_, w, g) in enumerate(rows):
                cur = nl(cur, w)
                if g != 1.0:
                    cur = cur * g
                cur = filter_block(cur, h_half if j == last else h_full)
            return cur
        for _, w, g in rows:
            if arrangement == "linear-first":
                cur = nl(filter_block(cur, h_full), w)
            else:
                cur = filter_block(nl(cur, w), h_full)
            if g != 1.0:
                cur = cur * g
        return cur

    return run


def backpropagate_arrays(samples: np.ndarray, rate_hz: float, cfg: PortConfig) -> np.ndarray:
    """(2, n) complex -> (2, n) complex128 through overlap-and-save (dbp.py:160-235)."""
    samples = np.asarray(samples, dtype=np.complex128)
    op = block_operator(cfg, rate_hz)
    blocks = cut_blocks(samples, cfg.block_len, cfg.overlap)
    done = np.stack([op(b) for b in blocks]) if len(blocks) else blocks
    return join_blocks(done, samples.shape[1], cfg.overlap)


def process_blocks(blocks: np.ndarray, rate_hz: float, cfg: PortConfig) -> np.ndarray:
    """Apply the block operator to each (2, N) block of a (nb, 2, N) stack."""
    op = block_operator(cfg, rate_hz)
    return np.stack([op(np.asarray(b, dtype=np.complex128)) for b in blocks])


# ---------------------------------------------------------------------------
# parity metrics
# ---------------------------------------------------------------------------

def per_block_rel_l2(got: np.ndarray, want: np.ndarray, block_len: int, overlap: int) -> np.ndarray:
    """Relative L2 error of each kept ``step`` segment (the north-star parity unit)."""
    step = block_len - overlap
    n = want.shape[-1]
    out = []
    for s in range(0, n, step):
        w = want[..., s:s + step]
        g = got[..., s:s + step]
        den = np.sqrt(np.sum(np.abs(w) ** 2))
        out.append(np.sqrt(np.sum(np.abs(g - w) ** 2)) / (den if den > 0 else 1.0))
    return np.asarray(out)
