"""Alias module: ``fiberdbp.dbp`` names (pkg/src/fiberdbp/dbp.py) on the GPU path."""
from .backprop import (  # noqa: F401
    ALGORITHMS, ARRANGEMENTS, DbpConfig, _reverse_step_schedule, backpropagate, block_processor,
    channel_memory_samples, estimate_channel_memory, nonlinear_substep_essfm, nonlinear_substep_ssfm,
    overlap_save_run,
)
from .framing import OverlapPlan, fft_frequencies, next_power_of_two  # noqa: F401
from .params import DualPolSignal, EssfmCoefficients, LinkConfig  # noqa: F401
from .spectral import fft, ifft  # noqa: F401
from .forward import linear_substep  # noqa: F401
