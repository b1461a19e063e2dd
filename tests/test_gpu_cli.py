"""The reference's experiment runner with ``--backend gpu``:
the same spec through fiberdbp.cli on the CPU (unchanged reference, from
oracle/_ref) and with the GPU backend; every row ok, the GPU kernels ran, and
the BER / Q of each (variant, power) cell agree with the reference."""

import math
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parent.parent / "oracle" / "_ref"

SPEC = """
scenario = ber-sweep
launch_powers_dbm = 1.5, 3
num_blocks = 1
seeds = 3
[link]
span_length_km = 40
num_spans = 30
amp_noise_figure_db = 5
[tx]
num_symbols = 4096
pulse = rc
rolloff = 0.2
[channel]
steps_per_span = 8
[train]
n_coeffs = 8
train_samples = 4096
max_iterations = 6
[dbp]
block_len = 1024
overlap = 256
[variant.ffe]
algorithm = ffe
[variant.essfm1]
algorithm = essfm
num_steps = 1
n_coeffs = 8
"""


@pytest.fixture(scope="module")
def ref_cli():
    if not (REF / "fiberdbp" / "cli.py").exists():
        pytest.skip("oracle/_ref not installed (oracle/install_ref.sh)")
    sys.path.insert(0, str(REF))
    from fiberdbp import cli
    return cli


def _rows(path):
    lines = Path(path).read_text().strip().splitlines()
    head = lines[0].split(",")
    return [dict(zip(head, ln.split(","))) for ln in lines[1:]]


@pytest.mark.filterwarnings("ignore::UserWarning")
def test_ber_sweep_gpu_backend_matches_reference(ref_cli, tmp_path):
    from paper_1507_00921_b200 import _native
    from paper_1507_00921_b200 import cli as gpu_cli
    spec = tmp_path / "run.cfg"
    spec.write_text(SPEC)
    cpu_out, gpu_out = tmp_path / "cpu.csv", tmp_path / "gpu.csv"
    assert gpu_cli.main(["--backend", "cpu", "sweep", "--spec", str(spec), "--out", str(cpu_out)]) == 0
    before = _native.launch_count()
    assert gpu_cli.main(["--backend", "gpu", "sweep", "--spec", str(spec), "--out", str(gpu_out),
                         "--jobs", "4"]) == 0
    assert _native.launch_count() > before          # the GPU implementations ran
    # the reference module is left as it was
    from fiberdbp import dbp
    assert ref_cli.backpropagate is dbp.backpropagate
    cpu, gpu = _rows(cpu_out), _rows(gpu_out)
    assert len(cpu) == len(gpu) == 4
    for a, b in zip(cpu, gpu):
        assert (a["algorithm"], a["power_dbm"]) == (b["algorithm"], b["power_dbm"])
        assert a["status"] == b["status"] == "ok", (a, b)
        ba, bb = float(a["ber"]), float(b["ber"])
        # float32 link simulation + DBP + coefficient fit + receiver against the float64
        # reference over 30 x 40 km: the cells agree to a handful of bit errors
        assert abs(ba - bb) <= max(1e-3, 0.25 * ba), (a, b)
        if ba > 1e-3:
            assert abs(float(a["q_db"]) - float(b["q_db"])) <= 0.5, (a, b)
        ma, mb = float(a["mse"]), float(b["mse"])
        assert abs(ma - mb) <= 0.05 * ma + 1e-6, (a, b)
        print(a["algorithm"], a["power_dbm"], "cpu", a["ber"], a["q_db"], a["mse"], "gpu", b["ber"], b["q_db"], b["mse"])
