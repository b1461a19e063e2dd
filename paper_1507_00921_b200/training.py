"""ESSFM coefficient fitting on the GPU (the path's heaviest caller).

Mirrors ``fiberdbp.train`` (pkg/src/fiberdbp/train.py): ``mse``,
``TrainConfig``, ``TrainResult``, ``optimize_coefficients``,
``save_coefficients``, ``load_coefficients`` -- same fields, same
validation, same damped Gauss-Newton with step-halving line search.  What
changes is how the residuals are evaluated: the reference runs one
``backpropagate`` per coefficient vector (N_c+1 for every Jacobian,
train.py:153-158, plus one per line-search trial, train.py:161-178); here
every batch of coefficient vectors is ONE launch of the fused kernel over
the same waveform (``dbp_run_host_coeff_batch``: per-item coefficient sets,
shared input), the Jacobian uses all 2(N_c+1) central-difference
perturbations at once and the line search evaluates eight step scales per
launch, accepting the first improving scale in the reference's halving
order.  The outputs of every coefficient set stay on the device: the
squared residual norms (line search) and the Gauss-Newton normal equations
J^T J, J^T r (float64) are reduced there (``dbp_fit_sumsq`` /
``dbp_fit_normal``, csrc/fit_capi.cu), so an iteration moves (N_c+2)(N_c+1)
numbers over PCIe instead of the outputs.

Float32 note: the reference's forward difference with h = 1e-6
(train.py:148) is below the float32 noise floor of a DBP output (~1e-7
relative), so the GPU fit uses central differences with h = 1e-3
(truncation O(h^2) ~ 1e-6); the acceptance rule, stopping rule and the
least-squares solve (float64 numpy ``lstsq`` on the host) are unchanged.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from . import _native
from .backprop import DbpConfig, backpropagate_batch, get_engine
from .params import DualPolSignal, EssfmCoefficients


def _as_stack(sig) -> np.ndarray:
    if hasattr(sig, "stack") and callable(sig.stack):
        return sig.stack()
    arr = np.asarray(sig)
    return arr[np.newaxis, :] if arr.ndim == 1 else arr


def mse(a, b) -> float:
    """mean(|a - b|^2) / mean(|b|^2) over both polarisations (train.py:32-44)."""
    sa, sb = _as_stack(a), _as_stack(b)
    if sa.shape != sb.shape:
        raise ValueError(f"shape mismatch: {sa.shape} vs {sb.shape}")
    den = np.mean(np.abs(sb) ** 2)
    if den == 0.0:
        raise ValueError("reference is identically zero")
    return float(np.mean(np.abs(sa - sb) ** 2) / den)


@dataclass(frozen=True)
class TrainConfig:
    """Coefficient-fit settings (train.py:47-74)."""

    n_coeffs: int = 32
    target_steps_per_span: int = 4
    train_samples: int = 16384
    max_iterations: int = 30
    tolerance: float = 1e-9
    rng_seed: int = 0

    def __post_init__(self):
        if self.n_coeffs < 0:
            raise ValueError("n_coeffs must be >= 0")
        if self.target_steps_per_span < 1:
            raise ValueError("target_steps_per_span must be >= 1")
        if self.train_samples < 10 * (self.n_coeffs + 1):
            raise ValueError("train_samples must be at least 10x the unknown count")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")
        if not (self.tolerance > 0.0):
            raise ValueError("tolerance must be positive")


@dataclass(frozen=True)
class TrainResult:
    coefficients: EssfmCoefficients
    final_mse: float
    initial_mse: float
    converged: bool
    iterations: int


class _DeviceEvaluator:
    """DBP outputs of many coefficient vectors on one waveform, kept on the device.

    ``run`` is one launch for a batch of sets (dbp_run_coeff_batch); ``sumsq``
    and ``normal`` reduce the residuals (out - target)[window] * scale on the
    device (dbp_fit_sumsq / dbp_fit_normal); ``keep`` makes one set's output
    the base the next Jacobian's residual r refers to.
    """

    def __init__(self, prefix: np.ndarray, sample_rate: float, dbp_cfg: DbpConfig, n_coeffs: int,
                 target: np.ndarray, window: slice, device: int, max_sets: int):
        import torch

        geo = DbpConfig("essfm", dbp_cfg.plan, dbp_cfg.link, num_steps=dbp_cfg.num_steps,
                        coeffs=EssfmCoefficients.identity(n_coeffs), arrangement=dbp_cfg.arrangement)
        self.engine = get_engine(geo, sample_rate, device)
        self.n = prefix.shape[1]
        dev = torch.device("cuda", device)

        def upload(a):
            return torch.from_numpy(np.ascontiguousarray(a.astype(np.complex64)).view(np.float32)).to(dev)

        self.d_in = upload(prefix)
        self.d_target = upload(target)
        self.d_out = torch.empty((max_sets, 2, 2 * self.n), dtype=torch.float32, device=dev)
        self.d_base = torch.empty((2, 2 * self.n), dtype=torch.float32, device=dev)
        self.stream = torch.cuda.Stream(device=dev)
        self.w0, self.w1 = window.start, window.stop
        t_win = target[:, window].astype(np.complex128)
        self.scale = 1.0 / np.sqrt(np.sum(np.abs(t_win) ** 2))
        self.max_sets = max_sets
        self.launches = 0

    def run(self, sets: np.ndarray) -> int:
        sets = np.atleast_2d(np.asarray(sets, dtype=np.float64))
        if sets.shape[0] > self.max_sets:
            raise ValueError("too many coefficient sets for the evaluator")
        plan = self.engine.native
        with plan.lock:
            plan.set_coeff_batch(sets)
            plan.run_coeff_batch(self.d_in.data_ptr(), self.d_out.data_ptr(), self.n, self.stream.cuda_stream)
        self.launches += 1
        return sets.shape[0]

    def sumsq(self, n_sets: int) -> np.ndarray:
        return _native.fit_sumsq(self.d_out.data_ptr(), n_sets, self.n, self.d_target.data_ptr(), self.w0, self.w1,
                                 self.scale, self.stream.cuda_stream)

    def normal(self, n_params: int, fd_step: float):
        return _native.fit_normal(self.d_out.data_ptr(), n_params, self.n, self.d_target.data_ptr(),
                                  self.d_base.data_ptr(), self.w0, self.w1, self.scale, fd_step,
                                  self.stream.cuda_stream)

    def keep(self, k: int):
        with torch_stream(self.stream):
            self.d_base.copy_(self.d_out[k], non_blocking=True)


def torch_stream(stream):
    import torch
    return torch.cuda.stream(stream)


def optimize_coefficients(received: DualPolSignal, dbp_cfg: DbpConfig, train_cfg: TrainConfig, *,
                          device: int | None = None, fd_step: float = 1e-3,
                          line_search_batch: int = 8) -> TrainResult:
    """Fit ESSFM coefficients to a fine-step SSFM target on the GPU (train.py:86-188)."""
    dev = 0 if device is None else int(device)
    n_train = min(train_cfg.train_samples, len(received))
    prefix = np.stack([np.asarray(received.x[:n_train]), np.asarray(received.y[:n_train])])
    target_cfg = DbpConfig("ssfm", dbp_cfg.plan, dbp_cfg.link,
                           num_steps=train_cfg.target_steps_per_span * dbp_cfg.link.num_spans,
                           arrangement=dbp_cfg.arrangement)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        target = backpropagate_batch(prefix, received.sample_rate, target_cfg, device=dev)[0]
    target = target.astype(np.complex128)

    edge = dbp_cfg.plan.overlap // 2
    if n_train <= 4 * edge:
        edge = 0
    window = slice(edge, n_train - edge if edge else n_train)
    if np.sum(np.abs(target[:, window]) ** 2) == 0.0:
        raise ValueError("fine-step target is identically zero on the fit window")

    n_params = train_cfg.n_coeffs + 1
    ev = _DeviceEvaluator(prefix, received.sample_rate, dbp_cfg, train_cfg.n_coeffs, target, window, dev,
                          max_sets=max(2 * n_params, line_search_batch))
    c = EssfmCoefficients.identity(train_cfg.n_coeffs).c.copy()
    ev.run(c)
    err = float(ev.sumsq(1)[0])
    ev.keep(0)
    initial_err = err
    eye = np.eye(c.size) * fd_step

    converged = False
    iterations = 0
    for _ in range(train_cfg.max_iterations):
        ev.run(np.concatenate([c + eye, c - eye]))                  # 2 (Nc+1) sets, one launch
        ata, atr = ev.normal(c.size, fd_step)                        # J^T J, J^T r on the device
        step, *_ = np.linalg.lstsq(ata, -atr, rcond=None)

        scales = []
        s = 1.0
        while s >= 1e-8:
            scales.append(s)
            s *= 0.5
        accepted = False
        for i0 in range(0, len(scales), line_search_batch):
            trial = scales[i0:i0 + line_search_batch]
            cand = np.stack([c + sc * step for sc in trial])
            ev.run(cand)
            errs = ev.sumsq(len(trial))
            hit = np.nonzero(errs < err)[0]
            if hit.size:
                k = int(hit[0])                      # first improving scale in halving order
                improvement = (err - errs[k]) / err
                c, err = cand[k], float(errs[k])
                ev.keep(k)
                iterations += 1
                accepted = True
                if improvement < train_cfg.tolerance:
                    converged = True
                break
        if not accepted:
            converged = True
            break
        if converged:
            break

    return TrainResult(coefficients=EssfmCoefficients(c), final_mse=err, initial_mse=initial_err,
                       converged=converged, iterations=iterations)


def save_coefficients(path, coeffs: EssfmCoefficients):
    """Text format: line 1 N_c, then c_0 .. c_Nc one per line (train.py:191-198)."""
    lines = [str(coeffs.n_coeffs)] + [repr(float(v)) for v in coeffs.c]
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def load_coefficients(path) -> EssfmCoefficients:
    """Read a file written by save_coefficients (train.py:201-217)."""
    with open(path) as fh:
        raw = [ln.strip() for ln in fh if ln.strip()]
    if not raw:
        raise ValueError(f"{path}: empty coefficient file")
    try:
        n_c = int(raw[0])
    except ValueError as exc:
        raise ValueError(f"{path}: first line must be the side-coefficient count") from exc
    values = raw[1:]
    if len(values) != n_c + 1:
        raise ValueError(f"{path}: expected {n_c + 1} coefficients, found {len(values)}")
    try:
        c = np.array([float(v) for v in values])
    except ValueError as exc:
        raise ValueError(f"{path}: malformed coefficient value") from exc
    return EssfmCoefficients(c)
