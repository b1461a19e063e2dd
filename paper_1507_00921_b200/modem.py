"""Alias module: ``fiberdbp.modem`` receiver names (pkg/src/fiberdbp/modem.py) on the GPU receiver."""
from .params import DualPolSignal  # noqa: F401
from .rx import (  # noqa: F401
    AlignmentError, FrequencyOffsetError, RxMetrics, butterfly_equalize, butterfly_equalize_batch,
    carrier_recover, carrier_recover_batch, evm_percent, measure_ber, qpsk_decide, qpsk_map, receive_batch,
)
