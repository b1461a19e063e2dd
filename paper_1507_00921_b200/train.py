"""Alias module: ``fiberdbp.train`` names (pkg/src/fiberdbp/train.py) on the GPU fit."""
from .backprop import DbpConfig, backpropagate  # noqa: F401
from .params import DualPolSignal, EssfmCoefficients  # noqa: F401
from .training import (  # noqa: F401
    TrainConfig, TrainResult, load_coefficients, mse, optimize_coefficients, save_coefficients,
)
