"""``--backend gpu`` for the reference's experiment runner.

    python -m paper_1507_00921_b200.cli --backend gpu sweep --spec run.cfg
    python -m paper_1507_00921_b200.cli --backend gpu train --spec run.cfg
    python -m paper_1507_00921_b200.cli --backend cpu sweep --spec run.cfg    # the reference as is

The reference's own command line (``fiberdbp.cli``: argument parsing, spec
files with their environment overrides, the Monte-Carlo ber-sweep and the
train-coeffs scenario, CSV output; cli.py:599-695, 828-861, 866-925) runs
unchanged, with its per-waveform compute -- laser phase noise, the link
simulation, digital backpropagation, the coefficient fit and the receiver --
bound to this package's GPU implementations.  cli.py imports those names as
module globals (cli.py:36-49) and calls them with the reference's own value
objects, which the GPU functions accept (same names, signatures and error
behaviour), so the switch is a rebinding of the module's globals.  The cost
scenarios (cost-fig1 / cost-fig2 / inset-table) are closed-form tables and
run as they are on either backend.

A drop-in needs the reference package it replaces: ``fiberdbp`` must be
importable.  ``--jobs`` is forced to 1 on the GPU backend (the reference's
process pool would fork CUDA contexts; one GPU process is faster anyway).
"""

from __future__ import annotations

import argparse
import sys

from . import backprop, forward, rx, training

# fiberdbp.cli global -> GPU implementation (cli.py:36-49)
GPU_BINDINGS = {
    "backpropagate": backprop.backpropagate,
    "propagate_link": forward.propagate_link,
    "apply_laser_phase_noise": forward.apply_laser_phase_noise,
    "optimize_coefficients": training.optimize_coefficients,
    "butterfly_equalize": rx.butterfly_equalize,
    "carrier_recover": rx.carrier_recover,
    "qpsk_decide": rx.qpsk_decide,
    "measure_ber": rx.measure_ber,
    "evm_percent": rx.evm_percent,
}


def install_gpu_backend(cli_module) -> dict:
    """Rebind the reference CLI module's compute globals to the GPU ones;
    returns the previous bindings (for ``uninstall_gpu_backend``)."""
    missing = [name for name in GPU_BINDINGS if not hasattr(cli_module, name)]
    if missing:
        raise RuntimeError(f"{cli_module.__name__} lacks {missing}: not the reference experiment runner")
    saved = {name: getattr(cli_module, name) for name in GPU_BINDINGS}
    for name, fn in GPU_BINDINGS.items():
        setattr(cli_module, name, fn)
    return saved


def uninstall_gpu_backend(cli_module, saved: dict) -> None:
    for name, fn in saved.items():
        setattr(cli_module, name, fn)


def _strip_jobs(argv: list[str]) -> list[str]:
    out, skip = [], False
    for i, a in enumerate(argv):
        if skip:
            skip = False
            continue
        if a == "--jobs":
            skip = True
            continue
        if a.startswith("--jobs="):
            continue
        out.append(a)
    return out


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_1507_00921_b200.cli", add_help=False,
                                 description="the reference experiment runner with a GPU backend")
    ap.add_argument("--backend", choices=("gpu", "cpu"), default="gpu")
    args, rest = ap.parse_known_args(sys.argv[1:] if argv is None else argv)
    try:
        from fiberdbp import cli as ref_cli
    except ImportError as exc:   # the drop-in replaces the reference's compute, not the reference
        print(f"error: the reference package fiberdbp is not importable ({exc})", file=sys.stderr)
        return 2
    if args.backend == "cpu":
        return ref_cli.main(rest)
    saved = install_gpu_backend(ref_cli)
    try:
        return ref_cli.main(_strip_jobs(rest))
    finally:
        uninstall_gpu_backend(ref_cli, saved)


if __name__ == "__main__":
    sys.exit(main())
