"""Alias module: ``fiberdbp.channel`` names (pkg/src/fiberdbp/channel.py) on the GPU simulator."""
from .backprop import nonlinear_substep_ssfm  # noqa: F401
from .forward import (  # noqa: F401
    PLANCK, SPEED_OF_LIGHT, SsfmStepConfig, amplify_with_ase, apply_jones_matrix, apply_laser_phase_noise,
    haar_random_unitary, linear_substep, propagate_link, propagate_link_batch, propagate_span,
    random_polarization_rotation,
)
from .framing import fft_frequencies  # noqa: F401
from .params import DualPolSignal, FiberParams, LinkConfig, effective_length  # noqa: F401
from .spectral import fft, ifft  # noqa: F401
