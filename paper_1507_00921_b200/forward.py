"""Whole-waveform forward link simulator on the GPU.

Mirrors ``fiberdbp.channel`` (pkg/src/fiberdbp/channel.py): ``SsfmStepConfig``,
``propagate_span``, ``amplify_with_ase``, ``haar_random_unitary``,
``apply_jones_matrix``, ``random_polarization_rotation``,
``propagate_link`` -- same arguments, validation and random streams.  The
split-step work (per step: FFT of the whole circular waveform, dispersion,
inverse FFT, Manakov rotation, loss) runs in the ``dbp_sim_*`` kernels
(csrc/ssfm_kernels.cuh: four-step FFT from the DBP kernel's block-FFT
halves, the waveform resident in device memory for the whole link); the
ASE noise and the Haar-random Jones matrices are drawn on the host with
numpy exactly as the reference draws them (channel.py:97-153, 174-207), so a
seeded run reproduces the reference realisation.
"""

from __future__ import annotations

import math
import os
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _native
from .params import DualPolSignal, FiberParams, LinkConfig, effective_length

PLANCK = 6.62607015e-34
SPEED_OF_LIGHT = 299792458.0


@dataclass(frozen=True)
class SsfmStepConfig:
    """Uniform split-step discretisation of a span (channel.py:33-44)."""

    steps_per_span: int = 50
    nonlinear_enabled: bool = True

    def __post_init__(self):
        if self.steps_per_span < 1:
            raise ValueError("steps_per_span must be >= 1")


def linear_substep(spectrum, beta2: float, dz: float, freqs) -> np.ndarray:
    """Dispersion operator exp(-j 2 pi^2 beta2 1e-24 f^2 dz) on a spectrum (channel.py:47-58).

    The closed form the GPU tables are built from (float64, on the host, once
    per configuration); the per-step multiply itself runs inside the kernels.
    """
    spectrum = np.asarray(spectrum)
    freqs = np.asarray(freqs)
    if spectrum.shape[-1] != freqs.shape[-1]:
        raise ValueError("spectrum and frequency grid lengths differ")
    phase = -2.0 * np.pi ** 2 * (beta2 * 1e-24) * freqs ** 2 * dz
    return spectrum * np.exp(1j * phase)


def _as_generator(rng) -> np.random.Generator:
    return rng if isinstance(rng, np.random.Generator) else np.random.default_rng(rng)


def _log2_length(n: int) -> int:
    if n < 1 or n & (n - 1):
        raise ValueError(f"block length must be a power of two, got {n}")
    lg = n.bit_length() - 1
    if lg < 8:
        raise ValueError(f"the GPU simulator needs at least 256 samples, got {n}")
    return lg


class _SimCache:
    """One simulator per (device, length), grown to the largest batch seen.  A
    replaced simulator is dropped, not closed: a thread still holding it
    finishes its sequence and the handle is freed with the last reference."""

    sims: dict = {}
    lock = threading.Lock()

    @classmethod
    def get(cls, device: int, log2_n: int, batch: int) -> _native.NativeSim:
        key = (device, log2_n)
        with cls.lock:
            sim = cls.sims.get(key)
            if sim is None or sim.max_batch < batch:
                sim = _native.NativeSim(device, log2_n, max(batch, 1))
                cls.sims[key] = sim
            return sim


def _span_args(fiber: FiberParams, cfg: SsfmStepConfig):
    dz = fiber.length / cfg.steps_per_span
    dz_eff = effective_length(fiber.alpha, dz) if fiber.alpha > 0.0 else dz
    loss = math.exp(-fiber.alpha * dz / 2.0)
    return dz, dz_eff, loss


def propagate_span(sig: DualPolSignal, fiber: FiberParams, cfg: SsfmStepConfig, *,
                   device: int = 0) -> DualPolSignal:
    """One span of circular split-step propagation (channel.py:74-94)."""
    n = len(sig)
    lg = _log2_length(n)
    sim = _SimCache.get(device, lg, 1)
    x = np.empty((1, 2, n), dtype=np.complex64)
    x[0, 0], x[0, 1] = sig.x, sig.y
    dz, dz_eff, loss = _span_args(fiber, cfg)
    with sim.lock:
        sim.upload(x)
        sim.span(1, sig.sample_rate, fiber.beta2, fiber.gamma, dz, dz_eff, loss, cfg.steps_per_span,
                 cfg.nonlinear_enabled)
        out = sim.download(1)[0]
    return DualPolSignal(out[0], out[1], sig.sample_rate)


def _ase_noise(n: int, sample_rate: float, gain_db: float, noise_figure_db: float,
               center_wavelength_nm: float, rng) -> np.ndarray:
    """(2, n) complex ASE realisation drawn exactly as channel.py:112-125."""
    g_lin = 10.0 ** (gain_db / 10.0)
    f_lin = 10.0 ** (noise_figure_db / 10.0)
    nu = SPEED_OF_LIGHT / (center_wavelength_nm * 1e-9)
    s_ase = (g_lin - 1.0) * f_lin * PLANCK * nu / 2.0
    var = s_ase * sample_rate
    noise = _as_generator(rng).normal(scale=np.sqrt(var / 2.0), size=(2, 2, n))
    return noise[:, 0] + 1j * noise[:, 1]


def haar_random_unitary(rng=None) -> np.ndarray:
    """Haar 2x2 unitary, QR with the diagonal phase fixed (channel.py:131-138)."""
    gen = _as_generator(rng)
    z = gen.normal(size=(2, 2)) + 1j * gen.normal(size=(2, 2))
    q, r = np.linalg.qr(z)
    d = np.diagonal(r)
    return q * (d / np.abs(d))


def _apply(sig: DualPolSignal, g_amp: float, noise, jones, device: int) -> DualPolSignal:
    n = len(sig)
    lg = _log2_length(n)
    sim = _SimCache.get(device, lg, 1)
    x = np.empty((1, 2, n), dtype=np.complex64)
    x[0, 0], x[0, 1] = sig.x, sig.y
    with sim.lock:
        sim.upload(x)
        sim.amplify(1, g_amp, None if noise is None else noise[None], None if jones is None else jones[None])
        out = sim.download(1)[0]
    return DualPolSignal(out[0], out[1], sig.sample_rate)


def amplify_with_ase(sig: DualPolSignal, gain_db: float, noise_figure_db: float | None,
                     center_wavelength_nm: float = 1550.0, rng=None, *, device: int = 0) -> DualPolSignal:
    """Flat gain plus circular Gaussian ASE (channel.py:97-128)."""
    if gain_db < 0.0:
        raise ValueError("gain_db must be non-negative")
    noise = None
    if noise_figure_db is not None:
        noise = _ase_noise(len(sig), sig.sample_rate, gain_db, noise_figure_db, center_wavelength_nm, rng)
    return _apply(sig, 10.0 ** (gain_db / 20.0), noise, None, device)


def apply_jones_matrix(sig: DualPolSignal, jones, *, device: int = 0) -> DualPolSignal:
    """One 2x2 Jones matrix on every sample (channel.py:141-147)."""
    jones = np.asarray(jones, dtype=np.complex128)
    if jones.shape != (2, 2):
        raise ValueError("jones must be a 2x2 matrix")
    return _apply(sig, 1.0, None, jones, device)


def random_polarization_rotation(sig: DualPolSignal, rng=None, *, device: int = 0) -> DualPolSignal:
    """Haar-random polarisation rotation of the whole block (channel.py:150-153)."""
    return apply_jones_matrix(sig, haar_random_unitary(rng), device=device)


def apply_laser_phase_noise(sig: DualPolSignal, linewidth_hz: float, rng=None, *, device: int = 0) -> DualPolSignal:
    """Common Wiener phase noise on both polarisations (channel.py:156-171): the
    increments are the reference's seeded draws (host numpy), the running phase
    and the rotation are computed on the GPU."""
    if linewidth_hz < 0.0:
        raise ValueError("linewidth must be non-negative")
    if linewidth_hz == 0.0:
        return sig
    gen = _as_generator(rng)
    sigma = np.sqrt(2.0 * np.pi * linewidth_hz / sig.sample_rate)
    inc = gen.normal(scale=sigma, size=len(sig))
    out = _native.phase_noise(np.stack([np.asarray(sig.x), np.asarray(sig.y)]), inc, device)
    return DualPolSignal(out[0], out[1], sig.sample_rate)


def propagate_link_batch(samples: np.ndarray, sample_rate: float, link: LinkConfig, cfg: SsfmStepConfig,
                         rngs, *, device: int = 0, devices=None) -> np.ndarray:
    """(B, 2, n) complex waveforms through every span; ``rngs[i]`` seeds item i like
    ``propagate_link``'s ``rng`` (int or SeedSequence).  Returns (B, 2, n) complex64.
    ``devices``: split the batch into contiguous waveform groups, one per GPU
    (independent waveforms, no exchange); each item's result does not depend on
    the split."""
    x = np.ascontiguousarray(samples, dtype=np.complex64)
    if x.ndim == 2:
        x = x[None]
    b, _, n = x.shape
    lg = _log2_length(n)
    if len(rngs) != b:
        raise ValueError("need one rng seed per waveform")
    if devices is not None:
        devs = list(dict.fromkeys(int(d) for d in devices))
        if not devs:
            raise ValueError("devices must not be empty")
        if len(devs) > 1 and b > 1:
            bounds = [round(i * b / len(devs)) for i in range(len(devs) + 1)]
            parts = [(d, bounds[i], bounds[i + 1]) for i, d in enumerate(devs) if bounds[i + 1] > bounds[i]]
            with ThreadPoolExecutor(max_workers=len(parts)) as pool:
                futs = [pool.submit(propagate_link_batch, x[lo:hi], sample_rate, link, cfg, list(rngs[lo:hi]),
                                    device=d) for d, lo, hi in parts]
                return np.concatenate([f.result() for f in futs])
        device = devs[0]
    children = []
    for r in rngs:
        if isinstance(r, np.random.Generator):
            raise ValueError("pass an integer seed or SeedSequence, not a Generator")
        ss = r if isinstance(r, np.random.SeedSequence) else np.random.SeedSequence(r)
        children.append(ss.spawn(2 * link.num_spans))
    sim = _SimCache.get(device, lg, b)
    dz, dz_eff, loss = _span_args(link.span, cfg)
    g_amp = 10.0 ** (link.gain_db / 20.0)

    def draw_noise(s, i, out):
        out[i] = _ase_noise(n, sample_rate, link.gain_db, link.amp_noise_figure_db, link.center_wavelength_nm,
                            children[i][2 * s])

    def draws(s, rng_pool):
        # host draws of span s (ASE, Haar), made while the GPU propagates span s;
        # the waveforms' independent streams are drawn in parallel (numpy's
        # generators release the GIL), each item's values unchanged
        noise = None
        if link.amp_noise_figure_db is not None:
            noise = np.empty((b, 2, n), dtype=np.complex64)
            list(rng_pool.map(lambda i: draw_noise(s, i, noise), range(b)))
        jones = np.stack([haar_random_unitary(ch[2 * s + 1]) for ch in children]) if link.pol_rotation else None
        return noise, jones

    workers = max(1, min(b, os.cpu_count() or 1))
    with sim.lock, ThreadPoolExecutor(max_workers=1) as pool, ThreadPoolExecutor(max_workers=workers) as rng_pool:
        sim.upload(x)
        pending = pool.submit(draws, 0, rng_pool)
        for s in range(link.num_spans):
            sim.span(b, sample_rate, link.span.beta2, link.span.gamma, dz, dz_eff, loss, cfg.steps_per_span,
                     cfg.nonlinear_enabled)
            noise, jones = pending.result()
            if s + 1 < link.num_spans:
                pending = pool.submit(draws, s + 1, rng_pool)
            sim.amplify(b, g_amp, noise, jones)
        return sim.download(b)


def propagate_link(sig: DualPolSignal, link: LinkConfig, cfg: SsfmStepConfig, rng=None, *,
                   device: int = 0) -> DualPolSignal:
    """Every span: split-step fibre, amplifier (ASE unless disabled), optional Haar
    rotation, with the reference's independent child random streams (channel.py:174-207)."""
    if isinstance(rng, np.random.Generator):
        raise ValueError("pass an integer seed or SeedSequence, not a Generator")
    x = np.empty((1, 2, len(sig)), dtype=np.complex64)
    x[0, 0], x[0, 1] = sig.x, sig.y
    out = propagate_link_batch(x, sig.sample_rate, link, cfg, [rng], device=device)[0]
    return DualPolSignal(out[0], out[1], sig.sample_rate)
