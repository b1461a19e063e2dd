"""Alias module: ``fiberdbp.spectral`` geometry names (pkg/src/fiberdbp/spectral.py)."""
from .framing import OverlapPlan, fft_frequencies, is_power_of_two, next_power_of_two  # noqa: F401
