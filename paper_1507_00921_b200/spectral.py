"""Alias module: ``fiberdbp.spectral`` names (pkg/src/fiberdbp/spectral.py) on the GPU.

``fft`` / ``ifft`` are float64 transforms on the library's own Stockham FFT
(``dbp_fft_c2c``, csrc/fft64.cuh) with the
reference's power-of-two check; ``overlap_save_run`` runs GPU block
processors (``block_processor(cfg, sample_rate)``) through the fused kernel.
"""
from __future__ import annotations

import numpy as np

from . import _native
from .backprop import BlockProcessor, DeviceBlockProcessor, GpuBlockProcessor, block_processor, overlap_save_run  # noqa: F401
from .framing import OverlapPlan, fft_frequencies, is_power_of_two, next_power_of_two  # noqa: F401
from .params import DualPolSignal  # noqa: F401


def _check_block_length(n: int):
    if not is_power_of_two(n):
        raise ValueError(f"block length must be a power of two, got {n}")


def fft(block) -> np.ndarray:
    """Forward DFT along the last axis (spectral.py:37-41); length a power of two."""
    block = np.asarray(block)
    _check_block_length(block.shape[-1])
    return _native.fft_c2c(block, inverse=False)


def ifft(block) -> np.ndarray:
    """Inverse DFT along the last axis, 1/n scaled (spectral.py:44-48)."""
    block = np.asarray(block)
    _check_block_length(block.shape[-1])
    return _native.fft_c2c(block, inverse=True)
