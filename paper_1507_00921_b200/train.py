"""Alias module: ``fiberdbp.train`` names (pkg/src/fiberdbp/train.py) with GPU evaluation."""
from .training import (  # noqa: F401
    TrainConfig, TrainResult, load_coefficients, mse, optimize_coefficients, save_coefficients,
)
