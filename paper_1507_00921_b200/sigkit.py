"""Alias module: ``fiberdbp.sigkit`` value types (pkg/src/fiberdbp/sigkit.py)."""
from .params import (  # noqa: F401
    DualPolSignal, EssfmCoefficients, FiberParams, LinkConfig, alpha_from_db_per_km,
    dbm_to_watts, effective_length, scale_to_power, signal_power, watts_to_dbm,
)
