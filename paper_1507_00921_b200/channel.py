"""Alias module: ``fiberdbp.channel`` names (pkg/src/fiberdbp/channel.py) on the GPU simulator."""
from .backprop import nonlinear_substep_ssfm  # noqa: F401
from .forward import (  # noqa: F401
    SsfmStepConfig, amplify_with_ase, apply_jones_matrix, haar_random_unitary, propagate_link,
    propagate_link_batch, propagate_span, random_polarization_rotation,
)
