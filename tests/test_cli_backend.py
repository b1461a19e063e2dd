"""--backend gpu wiring for the reference's experiment runner (no GPU needed):
the GPU bindings cover exactly the compute names fiberdbp.cli imports, and
install / uninstall leave the reference module as it was."""

import sys
from pathlib import Path

import pytest

from paper_1507_00921_b200 import cli as gpu_cli

REF = Path(__file__).resolve().parent.parent / "oracle" / "_ref"


@pytest.fixture(scope="module")
def ref_cli():
    if not (REF / "fiberdbp" / "cli.py").exists():
        pytest.skip("oracle/_ref not installed (oracle/install_ref.sh)")
    sys.path.insert(0, str(REF))
    from fiberdbp import cli
    return cli


def test_bindings_cover_the_runner_compute(ref_cli):
    import fiberdbp
    for name, fn in gpu_cli.GPU_BINDINGS.items():
        assert hasattr(ref_cli, name), name
        assert fn.__name__ == getattr(ref_cli, name).__name__ == name
        assert fn.__module__.startswith("paper_1507_00921_b200")
    # DBP, link, fit and receiver are all rebound; the cost model is not
    assert {"backpropagate", "propagate_link", "optimize_coefficients", "measure_ber"} <= set(gpu_cli.GPU_BINDINGS)
    assert "cost_per_sample" not in gpu_cli.GPU_BINDINGS
    assert fiberdbp.backpropagate is ref_cli.backpropagate


def test_install_uninstall_round_trip(ref_cli):
    before = {n: getattr(ref_cli, n) for n in gpu_cli.GPU_BINDINGS}
    saved = gpu_cli.install_gpu_backend(ref_cli)
    try:
        for n, fn in gpu_cli.GPU_BINDINGS.items():
            assert getattr(ref_cli, n) is fn
    finally:
        gpu_cli.uninstall_gpu_backend(ref_cli, saved)
    for n, fn in before.items():
        assert getattr(ref_cli, n) is fn


def test_jobs_flag_stripped_for_the_gpu_backend():
    assert gpu_cli._strip_jobs(["sweep", "--jobs", "4", "--spec", "a"]) == ["sweep", "--spec", "a"]
    assert gpu_cli._strip_jobs(["sweep", "--jobs=8"]) == ["sweep"]


def test_cpu_backend_runs_the_reference_cost_scenario(ref_cli, tmp_path):
    # the closed-form cost scenario needs no device on either backend
    out = tmp_path / "cost.csv"
    assert gpu_cli.main(["--backend", "cpu", "cost", "--scenario", "inset-table", "--out", str(out)]) == 0
    assert out.read_text().startswith("# format_version=")
