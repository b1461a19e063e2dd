"""Overlap-and-save geometry and FFT-grid helpers of the DBP path.

Mirrors the reference's ``fiberdbp.spectral`` names (spectral.py:24-81):
``OverlapPlan``, ``fft_frequencies``, ``is_power_of_two``,
``next_power_of_two``.  The block engine itself (the reference's
``overlap_save_run``, spectral.py:87-145) lives on the GPU; this module only
holds the host-side index arithmetic that the kernels, the chunked host
pipeline and the multi-GPU shard planner share.

Framing contract (spectral.py:122-145): step = N - M, lead = M // 2,
num_blocks = ceil(n / step); block b covers global samples
[b*step - lead, b*step - lead + N) of the circularly extended signal and
contributes its samples [lead, lead + step) to output [b*step, (b+1)*step),
trimmed to n.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def is_power_of_two(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


def next_power_of_two(x: float) -> int:
    """Smallest power of two >= x, minimum 1 (spectral.py:24-29)."""
    p = 1
    while p < x:
        p *= 2
    return p


def fft_frequencies(n: int, sample_rate: float) -> np.ndarray:
    """Bin frequencies in Hz in FFT order (spectral.py:51-60)."""
    if not is_power_of_two(n):
        raise ValueError(f"block length must be a power of two, got {n}")
    if sample_rate <= 0.0:
        raise ValueError("sample_rate must be positive")
    return np.fft.fftfreq(n, d=1.0 / sample_rate)


@dataclass(frozen=True)
class OverlapPlan:
    """Blocks of ``block_len`` samples advancing by ``block_len - overlap`` (spectral.py:63-81)."""

    block_len: int
    overlap: int

    def __post_init__(self):
        if not is_power_of_two(self.block_len):
            raise ValueError(f"block_len must be a power of two, got {self.block_len}")
        if not (0 <= self.overlap < self.block_len):
            raise ValueError("overlap must satisfy 0 <= overlap < block_len")

    @property
    def usable(self) -> int:
        return self.block_len - self.overlap

    @property
    def lead(self) -> int:
        return self.overlap // 2

    def num_blocks(self, n_total: int) -> int:
        return -(-int(n_total) // self.usable)

    def input_span(self, block_begin: int, block_end: int) -> tuple[int, int]:
        """Global (possibly negative / >= n) sample range [lo, hi) blocks [b0, b1) read."""
        lo = block_begin * self.usable - self.lead
        return lo, lo + (block_end - block_begin) * self.usable + self.overlap

    def output_span(self, block_begin: int, block_end: int, n_total: int) -> tuple[int, int]:
        """Output sample range [lo, hi) blocks [b0, b1) produce, trimmed to n."""
        return block_begin * self.usable, min(block_end * self.usable, int(n_total))


def shard_blocks(num_blocks: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous block ranges b_g = floor(g * nb / parts): every chunk boundary
    is a multiple of N - M, so sharded outputs are bitwise equal to one device."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    edges = [(g * num_blocks) // parts for g in range(parts + 1)]
    return [(edges[g], edges[g + 1]) for g in range(parts)]


def gather_span(samples: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """samples[..., lo:hi] of the circularly extended signal (any lo, hi)."""
    n = samples.shape[-1]
    idx = np.arange(lo, hi) % n
    return samples[..., idx]
