"""CPU restatement of the reference coefficient fit -- TEST/MEASUREMENT INFRASTRUCTURE ONLY.

Damped Gauss-Newton with a forward-difference Jacobian and a step-halving
line search, exactly as pkg/src/fiberdbp/train.py:86-188, evaluated with the
oracle port (oracle/dbp_port.py) instead of ``fiberdbp.backpropagate``.
Pinned by tests/test_oracle_golden.py against the reference's own fit
(tests/golden: train_c, train_mse); used as the CPU baseline of
tools/train_bench.py.
"""

from __future__ import annotations

import numpy as np

from .dbp_port import PortConfig, backpropagate_arrays


def fit(samples: np.ndarray, rate_hz: float, cfg: PortConfig, n_coeffs: int,
        target_steps_per_span: int, train_samples: int, max_iterations: int,
        tolerance: float = 1e-9, fd_step: float = 1e-6):
    """Returns (coefficients, final_err, initial_err, converged, iterations)."""
    n_train = min(train_samples, samples.shape[1])
    prefix = np.asarray(samples[:, :n_train], dtype=np.complex128)
    tcfg = PortConfig("ssfm", cfg.block_len, cfg.overlap, cfg.beta2, cfg.gamma, cfg.alpha_db_per_km,
                      cfg.span_km, cfg.num_spans, target_steps_per_span * cfg.num_spans,
                      None, cfg.arrangement)
    target = backpropagate_arrays(prefix, rate_hz, tcfg)                 # train.py:110-117
    edge = cfg.overlap // 2                                             # train.py:121-125
    if n_train <= 4 * edge:
        edge = 0
    win = slice(edge, n_train - edge if edge else n_train)
    t_win = target[:, win]
    norm = np.sum(np.abs(t_win) ** 2)

    def residual(c):                                                    # train.py:130-143
        ecfg = PortConfig("essfm", cfg.block_len, cfg.overlap, cfg.beta2, cfg.gamma,
                          cfg.alpha_db_per_km, cfg.span_km, cfg.num_spans, cfg.num_steps,
                          np.asarray(c), cfg.arrangement)
        d = (backpropagate_arrays(prefix, rate_hz, ecfg) - target)[:, win] / np.sqrt(norm)
        return np.concatenate([d.real.ravel(), d.imag.ravel()])

    c = np.zeros(n_coeffs + 1)
    c[0] = 1.0
    r = residual(c)
    err = float(r @ r)
    initial = err
    converged, iterations = False, 0
    for _ in range(max_iterations):                                     # train.py:151-184
        jac = np.empty((r.size, c.size))
        for i in range(c.size):
            cp = c.copy()
            cp[i] += fd_step
            jac[:, i] = (residual(cp) - r) / fd_step
        step, *_ = np.linalg.lstsq(jac, -r, rcond=None)
        scale, accepted = 1.0, False
        while scale >= 1e-8:
            cand = c + scale * step
            rc = residual(cand)
            ec = float(rc @ rc)
            if ec < err:
                improvement = (err - ec) / err
                c, r, err = cand, rc, ec
                iterations += 1
                accepted = True
                if improvement < tolerance:
                    converged = True
                break
            scale *= 0.5
        if not accepted:
            converged = True
            break
        if converged:
            break
    return c, err, initial, converged, iterations
