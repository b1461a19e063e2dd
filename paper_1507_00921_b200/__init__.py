"""B200-native drop-in for the digital-backpropagation hot path of arXiv 1507.00921.

Mirrors the reference package's (``fiberdbp``) DBP API -- ``backpropagate``,
``DbpConfig``, ``OverlapPlan`` and the signal / link value types -- and runs
the overlap-save block engine with the SSFM / ESSFM / FFE operators as one
fused sm_100a CUDA kernel behind the C ABI in ``include/dbp_b200.h``
(``libdbp_b200.so``, loaded through ctypes).  There is no CPU fallback.
"""

from .params import (
    DualPolSignal,
    EssfmCoefficients,
    FiberParams,
    LinkConfig,
    alpha_from_db_per_km,
    dbm_to_watts,
    effective_length,
    scale_to_power,
    signal_power,
    watts_to_dbm,
)
from .framing import OverlapPlan, fft_frequencies, is_power_of_two, next_power_of_two, shard_blocks
from .backprop import (
    ALGORITHMS,
    ARRANGEMENTS,
    DbpConfig,
    DbpEngine,
    backpropagate,
    backpropagate_batch,
    channel_memory_samples,
    estimate_channel_memory,
    get_engine,
    nonlinear_substep_essfm,
    nonlinear_substep_ssfm,
    overlap_save_run,
    block_processor,
    identity_processor,
    filter_processor,
    BlockProcessor,
    GpuBlockProcessor,
    DeviceBlockProcessor,
)
from .spectral import fft, ifft

from .forward import (
    SsfmStepConfig,
    amplify_with_ase,
    apply_jones_matrix,
    apply_laser_phase_noise,
    linear_substep,
    haar_random_unitary,
    propagate_link,
    propagate_link_batch,
    propagate_span,
    random_polarization_rotation,
)
from .rx import (
    AlignmentError,
    FrequencyOffsetError,
    RxMetrics,
    butterfly_equalize,
    butterfly_equalize_batch,
    carrier_recover,
    carrier_recover_batch,
    evm_percent,
    measure_ber,
    qpsk_decide,
    qpsk_map,
    receive_batch,
)
from .training import TrainConfig, TrainResult, load_coefficients, mse, optimize_coefficients, save_coefficients
from . import costmodel

__version__ = "0.1.0"

__all__ = [
    "DualPolSignal", "EssfmCoefficients", "FiberParams", "LinkConfig", "alpha_from_db_per_km",
    "dbm_to_watts", "effective_length", "scale_to_power", "signal_power", "watts_to_dbm",
    "OverlapPlan", "fft_frequencies", "is_power_of_two", "next_power_of_two", "shard_blocks",
    "ALGORITHMS", "ARRANGEMENTS", "DbpConfig", "DbpEngine", "backpropagate", "backpropagate_batch",
    "channel_memory_samples", "estimate_channel_memory", "get_engine", "nonlinear_substep_essfm",
    "nonlinear_substep_ssfm", "TrainConfig", "TrainResult", "load_coefficients", "mse",
    "optimize_coefficients", "save_coefficients", "SsfmStepConfig", "amplify_with_ase",
    "apply_jones_matrix", "haar_random_unitary", "propagate_link", "propagate_link_batch", "propagate_span",
    "random_polarization_rotation", "apply_laser_phase_noise", "linear_substep", "overlap_save_run", "block_processor",
    "identity_processor", "filter_processor", "BlockProcessor", "GpuBlockProcessor", "DeviceBlockProcessor", "fft", "ifft", "AlignmentError", "FrequencyOffsetError", "RxMetrics", "butterfly_equalize",
    "butterfly_equalize_batch", "carrier_recover", "carrier_recover_batch", "evm_percent", "measure_ber",
    "qpsk_decide", "qpsk_map", "receive_batch", "__version__",
]
