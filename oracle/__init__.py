"""CPU oracle for the B200 DBP hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this package.  The product package never does.  See dbp_port.py for
the restatement of the reference algorithm and its parity pin.
"""

from . import dbp_port, waveforms  # noqa: F401
