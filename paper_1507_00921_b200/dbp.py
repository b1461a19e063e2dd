"""Alias module: ``fiberdbp.dbp`` names (pkg/src/fiberdbp/dbp.py) on the GPU path."""
from .backprop import (  # noqa: F401
    ALGORITHMS, ARRANGEMENTS, DbpConfig, _reverse_step_schedule, backpropagate,
    channel_memory_samples, estimate_channel_memory, nonlinear_substep_essfm,
)
from .backprop import nonlinear_substep_ssfm  # noqa: F401
