"""Drop-in ``backpropagate`` for the reference's DBP API, executed on B200.

Same public names, argument meaning, validation errors and warnings as
``fiberdbp.dbp`` (pkg/src/fiberdbp/dbp.py): ``ALGORITHMS``,
``ARRANGEMENTS``, ``channel_memory_samples``, ``estimate_channel_memory``,
``DbpConfig``, ``backpropagate(sig, cfg, jobs=1)``.  The host side keeps
everything that is float64 scalar work in the reference -- validation, the
short-overlap warning (dbp.py:175-181), the reverse step schedule
(dbp.py:112-157) and the dispersion filters (dbp.py:186, 196-197) -- and
hands the per-sample work to the fused CUDA kernel through the C ABI
(include/dbp_b200.h).  Samples cross the boundary as complex64; the result
is returned as the reference's complex128 ``DualPolSignal``.
"""

from __future__ import annotations

import math
import os
import sys
import threading
import warnings
from collections import OrderedDict
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _native
from .framing import OverlapPlan, fft_frequencies, next_power_of_two, shard_blocks
from .params import DualPolSignal, EssfmCoefficients, LinkConfig

ALGORITHMS = ("ffe", "ssfm", "essfm")
ARRANGEMENTS = ("symmetric", "linear-first", "nonlinear-first")


def channel_memory_samples(beta2: float, length_km: float, bandwidth_hz: float) -> float:
    """Dispersive memory 2 pi |beta2| L B^2 in samples (dbp.py:35-41)."""
    if length_km <= 0.0:
        raise ValueError("length must be positive")
    if bandwidth_hz <= 0.0:
        raise ValueError("bandwidth must be positive")
    return 2.0 * math.pi * abs(beta2) * 1e-24 * length_km * bandwidth_hz ** 2


def estimate_channel_memory(beta2: float, length_km: float, bandwidth_hz: float) -> int:
    """Channel memory rounded up to a power of two (dbp.py:44-46)."""
    return next_power_of_two(channel_memory_samples(beta2, length_km, bandwidth_hz))


@dataclass(frozen=True)
class DbpConfig:
    """Block-wise channel-inverter configuration (dbp.py:78-109)."""

    algorithm: str
    plan: OverlapPlan
    link: LinkConfig
    num_steps: int = 1
    coeffs: EssfmCoefficients | None = None
    arrangement: str = "symmetric"

    def __post_init__(self):
        if self.algorithm not in ALGORITHMS:
            raise ValueError(f"algorithm must be one of {ALGORITHMS}, got {self.algorithm!r}")
        if self.arrangement not in ARRANGEMENTS:
            raise ValueError(f"arrangement must be one of {ARRANGEMENTS}, got {self.arrangement!r}")
        if self.num_steps < 1:
            raise ValueError("num_steps must be >= 1")
        if self.algorithm == "essfm":
            if self.coeffs is None:
                raise ValueError("essfm requires a coefficient set")
            if self.plan.block_len <= 2 * self.coeffs.n_coeffs:
                raise ValueError("block length too short for the coefficient memory")


def _reverse_step_schedule(link, num_steps: int) -> list[tuple[float, float, float]]:
    """(dz_km, weight_km, gain) per reverse step, last physical segment first.

    Restates dbp.py:112-157 exactly (exact rational step boundaries in span
    units; forward power profile 1 at amplifier outputs, exp(-alpha z)
    inside a span; weight = profile integral over the segment / profile at
    its far end; gain = sqrt(profile(a) / profile(b))).
    """
    alpha = link.span.alpha
    span_len = link.span.length
    n_spans = link.num_spans
    dz = link.total_length / num_steps

    def level(z: Fraction) -> float:
        if z.denominator == 1:
            return 1.0
        local = float(z - math.floor(z)) * span_len
        return math.exp(-alpha * local)

    def area(a: Fraction, b: Fraction) -> float:
        s, acc = math.floor(a), 0.0
        while s < b:
            t0 = float(max(a, Fraction(s)) - s) * span_len
            t1 = float(min(b, Fraction(s + 1)) - s) * span_len
            acc += (math.exp(-alpha * t0) - math.exp(-alpha * t1)) / alpha if alpha > 0.0 else t1 - t0
            s += 1
        return acc

    out = []
    for j in range(num_steps, 0, -1):
        a = Fraction((j - 1) * n_spans, num_steps)
        b = Fraction(j * n_spans, num_steps)
        lb = level(b)
        out.append((dz, area(a, b) / lb, math.sqrt(level(a) / lb)))
    return out


def _dispersion(freqs: np.ndarray, beta2: float, length: float) -> np.ndarray:
    # same float64 expression as dbp.py:186 / 196-197
    return np.exp(1j * 2.0 * np.pi ** 2 * (beta2 * 1e-24) * freqs ** 2 * length)


def _own_plan(plan) -> OverlapPlan:
    """This package's OverlapPlan for any object with the reference's fields
    (the reference's own OverlapPlan has no block-range helpers)."""
    return plan if isinstance(plan, OverlapPlan) else OverlapPlan(int(plan.block_len), int(plan.overlap))


class DbpEngine:
    """One DBP configuration compiled onto one device (tables resident in HBM)."""

    def __init__(self, cfg: DbpConfig, sample_rate: float, device: int = 0):
        self.cfg = cfg
        self.sample_rate = float(sample_rate)
        self.device = int(device)
        plan = self.plan = _own_plan(cfg.plan)
        n = plan.block_len
        if not (_native.MIN_BLOCK_LEN <= n <= _native.MAX_BLOCK_LEN):
            raise ValueError(f"block_len {n} outside the GPU-supported range "
                             f"[{_native.MIN_BLOCK_LEN}, {_native.MAX_BLOCK_LEN}]")
        self.native = _native.NativePlan(self.device, n, plan.overlap)
        link = cfg.link
        freqs = fft_frequencies(n, self.sample_rate)
        beta2 = link.span.beta2
        if cfg.algorithm == "ffe":
            self.native.set_linear(_dispersion(freqs, beta2, link.total_length), None)
            self.native.set_steps("ffe", cfg.arrangement, [0.0], [1.0], 0.0)
            self.schedule = []
        else:
            sched = _reverse_step_schedule(link, cfg.num_steps)
            dz = sched[0][0]
            self.native.set_linear(_dispersion(freqs, beta2, dz), _dispersion(freqs, beta2, 0.5 * dz))
            if cfg.algorithm == "ssfm" and cfg.coeffs is None:
                coeffs = None
            else:
                coeffs = cfg.coeffs.c if cfg.coeffs is not None else None
            self.native.set_steps(cfg.algorithm, cfg.arrangement, [w for _, w, _ in sched],
                                  [g for _, _, g in sched], -link.span.gamma,
                                  None if cfg.algorithm == "ssfm" else coeffs)
            self.schedule = sched

    def num_blocks(self, n_total: int) -> int:
        return self.plan.num_blocks(n_total)

    def run_host(self, samples: np.ndarray, out: np.ndarray | None = None,
                 block_range: tuple[int, int] | None = None) -> np.ndarray:
        """(B, 2, n) complex -> (B, 2, n) complex64 through host buffers."""
        x = np.ascontiguousarray(samples, dtype=np.complex64)
        if x.ndim == 2:
            x = x[None]
        if x.ndim != 3 or x.shape[1] != 2:
            raise ValueError("expected (batch, 2, n) or (2, n) samples")
        b, _, n = x.shape
        if out is None:
            out = np.zeros_like(x)
        b0, b1 = block_range if block_range is not None else (0, self.num_blocks(n))
        with self.native.lock:
            self.native.run_host(x, out, n, b, b0, b1)
        return out

    def close(self):
        self.native.close()


_ENGINES: "OrderedDict[tuple, DbpEngine]" = OrderedDict()
_ENGINES_LOCK = threading.Lock()
_MAX_ENGINES = 16


def _cfg_key(cfg: DbpConfig, sample_rate: float, device: int) -> tuple:
    sp = cfg.link.span
    c = None if cfg.coeffs is None else cfg.coeffs.c.tobytes()
    return (device, cfg.algorithm, cfg.plan.block_len, cfg.plan.overlap, cfg.num_steps,
            cfg.arrangement, float(sample_rate), sp.beta2, sp.gamma, sp.alpha_db_per_km, sp.length,
            cfg.link.num_spans, c)


def get_engine(cfg: DbpConfig, sample_rate: float, device: int = 0) -> DbpEngine:
    """Cached engine for (config, sample rate, device)."""
    key = _cfg_key(cfg, sample_rate, device)
    with _ENGINES_LOCK:
        eng = _ENGINES.get(key)
        if eng is not None:
            _ENGINES.move_to_end(key)
            return eng
    eng = DbpEngine(cfg, sample_rate, device)
    with _ENGINES_LOCK:
        _ENGINES[key] = eng
        while len(_ENGINES) > _MAX_ENGINES:
            # dropped, not closed: a thread may still hold the evicted engine;
            # its plan is freed with the last reference (NativePlan.__del__)
            _ENGINES.popitem(last=False)
    return eng


class _RowArena:
    """Recycled result arrays for ``backpropagate`` (complex128 rows) and
    ``backpropagate_batch`` (the complex64 batch).

    The reference returns freshly allocated rows (sigkit.py:56-68); a fresh
    numpy row of this size is an anonymous mapping whose first write faults
    in every 4 KiB page -- at the configs[0] length that costs more than the
    whole GPU round trip (`profiles/r2/final/session5/dropin_latency_*.txt`).
    The arena keeps the rows it handed out and gives one out again only once
    nothing outside the arena refers to it any more (every view, slice or
    ``DualPolSignal`` of a row holds a reference to it through ``.base``), so
    callers still own distinct, non-aliased results.  ``DBP_HOST_ARENA_MB``
    bounds the bytes the arena tracks (default 2048, 0 disables it).
    """

    _MIN_BYTES = 1 << 16      # smaller rows come from the heap and never fault

    def __init__(self, cap_bytes: int):
        self._cap = int(cap_bytes)
        self._lock = threading.Lock()
        self._rows: list[np.ndarray] = []    # least recently handed out first

    def _idle(self, i: int) -> bool:
        # the list's reference plus getrefcount's argument
        return sys.getrefcount(self._rows[i]) == 2

    def take(self, n: int) -> np.ndarray:
        """A complex128 row of n samples (the rows of a ``DualPolSignal`` result)."""
        return self.take_array((n,), np.complex128)

    def take_array(self, shape, dtype) -> np.ndarray:
        """An uninitialised C-contiguous array; every caller overwrites all of it."""
        dt = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dt.itemsize
        if nbytes < self._MIN_BYTES or 2 * nbytes > self._cap:
            return np.empty(shape, dtype=dt)
        with self._lock:
            rows = self._rows                 # owners: 1-D byte arrays
            for i in range(len(rows)):
                if rows[i].nbytes == nbytes and self._idle(i):
                    row = rows.pop(i)
                    rows.append(row)
                    return row.view(dt).reshape(shape)
            total = sum(r.nbytes for r in rows)
            i = 0
            while total + nbytes > self._cap and i < len(rows):
                if self._idle(i):
                    total -= rows[i].nbytes
                    del rows[i]
                else:
                    i += 1
            row = np.empty(nbytes, dtype=np.uint8)
            if total + nbytes <= self._cap:
                rows.append(row)
            return row.view(dt).reshape(shape)

    def tracked_bytes(self) -> int:
        with self._lock:
            return sum(r.nbytes for r in self._rows)

    def clear(self) -> None:
        with self._lock:
            self._rows.clear()


def _arena_cap_bytes() -> int:
    try:
        mb = int(os.environ.get("DBP_HOST_ARENA_MB", "2048"))
    except ValueError:
        mb = 2048
    return max(0, mb) << 20


_OUT_ROWS = _RowArena(_arena_cap_bytes())


def _warn_short_overlap(cfg: DbpConfig, sample_rate: float, stacklevel: int):
    span = cfg.link.span
    memory = (channel_memory_samples(span.beta2, cfg.link.total_length, sample_rate)
              if span.beta2 != 0.0 else 0.0)
    if cfg.plan.overlap < memory:
        warnings.warn(
            f"overlap {cfg.plan.overlap} below estimated channel memory "
            f"{memory:.0f} samples; block edges may leak interblock interference",
            stacklevel=stacklevel + 1,
        )


def _resolve_devices(device, devices) -> list[int]:
    if devices is not None:
        devs = [int(d) for d in devices]
        if not devs:
            raise ValueError("devices must not be empty")
        return devs
    return [0 if device is None else int(device)]


def backpropagate_batch(samples: np.ndarray, sample_rate: float, cfg: DbpConfig, *,
                        device: int | None = None, devices=None) -> np.ndarray:
    """Batched DBP: (B, 2, n) complex waveforms -> (B, 2, n) complex64.

    With several ``devices`` the work is split across them -- by whole
    waveforms when B >= #devices, else by contiguous overlap-save block
    ranges -- with no exchange; results are bitwise equal to one device.
    """
    x = np.ascontiguousarray(samples, dtype=np.complex64)
    if x.ndim == 2:
        x = x[None]
    if x.ndim != 3 or x.shape[1] != 2 or x.shape[2] < 1:
        raise ValueError("expected (batch, 2, n) samples with n >= 1")
    _warn_short_overlap(cfg, sample_rate, stacklevel=2)
    devs = _resolve_devices(device, devices)
    out = _OUT_ROWS.take_array(x.shape, np.complex64)   # every sample is overwritten below
    if len(devs) == 1:
        return get_engine(cfg, sample_rate, devs[0]).run_host(x, out)
    b, _, n = x.shape
    engines = [get_engine(cfg, sample_rate, d) for d in devs]
    jobs = []
    if b >= len(devs):
        for (i0, i1), eng in zip(shard_blocks(b, len(devs)), engines):
            if i1 > i0:
                jobs.append((eng, x[i0:i1], out[i0:i1], None))
    else:
        for (b0, b1), eng in zip(shard_blocks(_own_plan(cfg.plan).num_blocks(n), len(devs)), engines):
            if b1 > b0:
                jobs.append((eng, x, None, (b0, b1)))
    results = []
    with ThreadPoolExecutor(max_workers=len(jobs)) as pool:
        futs = [pool.submit(lambda j: j[0].run_host(j[1], j[2], j[3]), j) for j in jobs]
        results = [f.result() for f in futs]
    for (eng, _, dst, rng), res in zip(jobs, results):
        if rng is not None:
            lo, hi = _own_plan(cfg.plan).output_span(rng[0], rng[1], n)
            out[..., lo:hi] = res[..., lo:hi]
    return out


def backpropagate(sig: DualPolSignal, cfg: DbpConfig, jobs: int = 1, *,
                  device: int | None = None, devices=None) -> DualPolSignal:
    """Invert the configured link on a received waveform (dbp.py:160-235).

    ``jobs`` is validated like the reference (spectral.py:119-120) and
    otherwise ignored: the GPU result does not depend on it.  ``device`` /
    ``devices`` select the GPU(s).
    """
    _warn_short_overlap(cfg, sig.sample_rate, stacklevel=2)
    if jobs < 1:
        raise ValueError("jobs must be >= 1")
    devs = _resolve_devices(device, devices)
    if len(devs) == 1:
        # complex128 rows straight through the C ABI: casts on host threads,
        # pinned staging, chunked H2D / kernel / D2H pipeline
        eng = get_engine(cfg, sig.sample_rate, devs[0])
        x, y = np.ascontiguousarray(sig.x, dtype=np.complex128), np.ascontiguousarray(sig.y, dtype=np.complex128)
        out_x, out_y = _OUT_ROWS.take(x.size), _OUT_ROWS.take(y.size)
        with eng.native.lock:
            eng.native.backpropagate_c128(x, y, out_x, out_y)
        return DualPolSignal(out_x, out_y, sig.sample_rate)
    x = np.empty((1, 2, len(sig)), dtype=np.complex64)
    x[0, 0] = sig.x
    x[0, 1] = sig.y
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        out = backpropagate_batch(x, sig.sample_rate, cfg, device=device, devices=devices)
    return DualPolSignal(out[0, 0], out[0, 1], sig.sample_rate)


# ---------------------------------------------------------------------------
# sub-step mirrors (dbp.py:49-75, channel.py:61-71) on the GPU
# ---------------------------------------------------------------------------

def _rotate_block(block, gamma: float, dz_eff: float, c: np.ndarray, device: int = 0) -> np.ndarray:
    blk = np.asarray(block)
    if blk.ndim != 2 or blk.shape[0] != 2:
        raise ValueError("expected a (2, n) dual-polarization block")
    n = blk.shape[1]
    if n <= 2 * (c.size - 1):
        raise ValueError(f"block length {n} too short for {c.size - 1} side coefficients")
    return _native.nonlinear_substep(blk, gamma, dz_eff, c, device)


def nonlinear_substep_essfm(block, gamma: float, dz_eff: float, coeffs: EssfmCoefficients,
                            *, device: int = 0) -> np.ndarray:
    """GPU ESSFM rotation of one (2, n) block of any length n > 2 N_c, cyclic FIR inside
    the block, float64 (dbp.py:49-75; dbp_nonlinear_substep_c128)."""
    return _rotate_block(block, gamma, dz_eff, np.asarray(coeffs.c, dtype=np.float64), device)


def nonlinear_substep_ssfm(block, gamma: float, dz_eff: float, *, device: int = 0) -> np.ndarray:
    """GPU plain rotation exp(-j gamma dz_eff (|x|^2 + |y|^2)) (channel.py:61-71), any length."""
    return _rotate_block(block, gamma, dz_eff, np.array([1.0]), device)


class ProgramEngine:
    """A block operator that is not a DBP configuration: the identity (framing
    only, ``DBP_ALG_IDENTITY``) or a caller-supplied frequency-domain filter
    ``ifft(fft(b) * H)`` (an FFE program with table H), on one device."""

    def __init__(self, plan: OverlapPlan, sample_rate: float, device: int = 0, kernel=None):
        plan = self.plan = _own_plan(plan)
        self.sample_rate = float(sample_rate)
        self.device = int(device)
        n = plan.block_len
        if not (_native.MIN_BLOCK_LEN <= n <= _native.MAX_BLOCK_LEN):
            raise ValueError(f"block_len {n} outside the GPU-supported range "
                             f"[{_native.MIN_BLOCK_LEN}, {_native.MAX_BLOCK_LEN}]")
        self.native = _native.NativePlan(self.device, n, plan.overlap)
        if kernel is None:
            self.native.set_steps("identity", "symmetric", [0.0], [1.0], 0.0)
        else:
            h = np.asarray(kernel, dtype=np.complex128)
            if h.shape != (n,):
                raise ValueError(f"filter must have shape ({n},), got {h.shape}")
            self.native.set_linear(h, None)
            self.native.set_steps("ffe", "symmetric", [0.0], [1.0], 0.0)

    def num_blocks(self, n_total: int) -> int:
        return self.plan.num_blocks(n_total)

    run_host = DbpEngine.run_host

    def close(self):
        self.native.close()


class GpuBlockProcessor:
    """The per-block operator of ``backpropagate`` (the closure ``process`` of
    dbp.py:212-233) -- or the identity / a linear filter (``identity_processor``,
    ``filter_processor``) -- as a GPU object: callable on one (2, N) block or an
    (nb, 2, N) stack (``dbp_process_blocks``), and recognised by
    ``overlap_save_run``, which then frames and processes the whole signal in
    the fused kernel."""

    def __init__(self, cfg: DbpConfig | None, sample_rate: float, device: int = 0, *, engine=None):
        self.cfg = cfg
        self.sample_rate = float(sample_rate)
        self.device = int(device)
        self.engine = engine if engine is not None else get_engine(cfg, sample_rate, device)

    @property
    def plan(self):
        return self.cfg.plan if self.cfg is not None else self.engine.plan

    def __call__(self, block):
        import torch

        b = np.asarray(block)
        single = b.ndim == 2
        blocks = np.ascontiguousarray((b[None] if single else b).astype(np.complex64))
        n = self.plan.block_len
        if blocks.ndim != 3 or blocks.shape[1:] != (2, n):
            raise ValueError(f"expected (2, {n}) blocks")
        dev = torch.device("cuda", self.device)
        d_in = torch.from_numpy(blocks.view(np.float32)).to(dev)
        d_out = torch.empty_like(d_in)
        stream = torch.cuda.current_stream(dev)
        with self.engine.native.lock:
            self.engine.native.process_blocks(d_in.data_ptr(), d_out.data_ptr(), blocks.shape[0], stream.cuda_stream)
        stream.synchronize()
        out = d_out.cpu().numpy().view(np.complex64).astype(np.complex128)
        return out[0] if single else out


BlockProcessor = GpuBlockProcessor   # spectral.py:84: the operator type overlap_save_run accepts


def block_processor(cfg: DbpConfig, sample_rate: float, *, device: int = 0) -> GpuBlockProcessor:
    """The GPU block operator of ``cfg`` (dbp.py:193-233) for ``overlap_save_run``."""
    return GpuBlockProcessor(cfg, sample_rate, device)


def identity_processor(plan: OverlapPlan, sample_rate: float, *, device: int = 0) -> GpuBlockProcessor:
    """The identity block operator (the reference tests' ``lambda b: b``,
    test_spectral.py:72-76, 119-125): ``overlap_save_run`` then exercises the
    framing alone -- cyclic extension, keep the centre, trim -- bit-exactly."""
    return GpuBlockProcessor(None, sample_rate, device, engine=ProgramEngine(plan, sample_rate, device))


def filter_processor(plan: OverlapPlan, kernel, sample_rate: float, *, device: int = 0) -> GpuBlockProcessor:
    """The linear block operator ``ifft(fft(b) * kernel)`` for a caller-supplied
    length-N frequency response in numpy FFT bin order (test_spectral.py:78-97)."""
    return GpuBlockProcessor(None, sample_rate, device, engine=ProgramEngine(plan, sample_rate, device, kernel))


class DeviceBlockProcessor:
    """A caller-written block operator that runs on the device: ``fn`` maps an
    (nb, 2, N) complex torch tensor on ``cuda:device`` (every block of the
    signal at once -- the batched form of spectral.py:84's ``(2, N) -> (2, N)``
    callable) to a tensor of the same shape.  ``overlap_save_run`` frames the
    signal into that stack on the GPU (``dbp_frame_blocks``), calls ``fn`` once
    and assembles the kept centres on the GPU (``dbp_unframe_blocks``).
    ``dtype``: ``"complex128"`` (the reference's own, default) or
    ``"complex64"``."""

    def __init__(self, fn, *, device: int = 0, dtype: str = "complex128"):
        if dtype not in ("complex64", "complex128"):
            raise ValueError("dtype must be 'complex64' or 'complex128'")
        self.fn = fn
        self.device = int(device)
        self.dtype = dtype

    def __call__(self, blocks):
        return self.fn(blocks)


def _framed_run(sig: DualPolSignal, plan, apply, device: int, dtype: str) -> DualPolSignal:
    """Overlap-save around ``apply`` (a function of the (nb, 2, N) device block
    stack): cyclic extension + block cut and keep-centre assembly by the
    framing kernels -- pure copies, so bit-exact to spectral.py:122-145."""
    import torch

    from . import _native

    n_total = len(sig)
    n_blk, m = plan.block_len, plan.overlap
    nb = -(-n_total // (n_blk - m))   # spectral.py:126 (foreign OverlapPlan objects welcome)
    wide = dtype == "complex128"
    np_dt, t_dt, elem = ((np.complex128, torch.complex128, 16) if wide else (np.complex64, torch.complex64, 8))
    dev = torch.device("cuda", device)
    x = torch.from_numpy(np.ascontiguousarray(np.stack([np.asarray(sig.x), np.asarray(sig.y)]).astype(np_dt))).to(dev)
    blocks = torch.empty((nb, 2, n_blk), dtype=t_dt, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _native.frame_blocks(x.data_ptr(), blocks.data_ptr(), n_total, 1, n_blk, m, 0, nb, elem, stream)
    proc = apply(blocks)
    if not isinstance(proc, torch.Tensor) or tuple(proc.shape) != (nb, 2, n_blk):
        shape = tuple(proc.shape) if hasattr(proc, "shape") else type(proc).__name__
        raise ValueError(f"block processor returned shape {shape}, expected ({nb}, 2, {n_blk})")
    proc = proc.to(device=dev, dtype=t_dt).contiguous()
    out = torch.empty((2, n_total), dtype=t_dt, device=dev)
    _native.unframe_blocks(proc.data_ptr(), out.data_ptr(), n_total, 1, n_blk, m, 0, nb, elem, stream)
    o = out.cpu().numpy()
    return DualPolSignal(o[0].astype(np.complex128), o[1].astype(np.complex128), sig.sample_rate)


def overlap_save_run(sig: DualPolSignal, plan, block_processor, jobs: int = 1, *, device: int = 0) -> DualPolSignal:
    """spectral.py:87-145 on the GPU, for three kinds of block processor:

    * a ``GpuBlockProcessor`` (``block_processor(cfg, fs)``, the identity or a
      filter): framing, the per-block operator and the keep-centre assembly
      all inside the fused kernel;
    * a ``DeviceBlockProcessor``: GPU framing into one (nb, 2, N) device stack,
      the caller's torch operator on it, GPU assembly;
    * any other callable on (2, N) numpy blocks (the reference's
      ``BlockProcessor``): GPU framing in complex128, the caller's function on
      each block on the host (the caller's own code -- ``jobs`` threads, as in
      spectral.py:132-136), GPU assembly; bit-identical to the reference for a
      deterministic callable.  A result of the wrong shape raises the
      reference's ``ValueError`` (spectral.py:141-142)."""
    if jobs < 1:
        raise ValueError("jobs must be >= 1")
    if isinstance(block_processor, GpuBlockProcessor):
        if (plan.block_len, plan.overlap) != (block_processor.plan.block_len, block_processor.plan.overlap):
            raise ValueError("plan does not match the block processor's plan")
        if float(sig.sample_rate) != block_processor.sample_rate:
            raise ValueError("signal sample rate does not match the block processor's")
        out = block_processor.engine.run_host(np.stack([np.asarray(sig.x), np.asarray(sig.y)]))[0]
        return DualPolSignal(out[0].astype(np.complex128), out[1].astype(np.complex128), sig.sample_rate)
    if isinstance(block_processor, DeviceBlockProcessor):
        return _framed_run(sig, plan, block_processor.fn, block_processor.device, block_processor.dtype)
    if not callable(block_processor):
        raise TypeError("block_processor must be callable")
    n_blk = plan.block_len

    def on_host(blocks):
        import torch

        host = blocks.cpu().numpy()
        views = [host[b] for b in range(host.shape[0])]
        if jobs == 1:
            processed = [block_processor(b) for b in views]
        else:
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(max_workers=jobs) as pool:
                processed = list(pool.map(block_processor, views))
        res = np.empty_like(host)
        for b, blk in enumerate(processed):
            blk = np.asarray(blk)
            if blk.shape != (2, n_blk):
                raise ValueError(f"block processor returned shape {blk.shape}, expected (2, {n_blk})")
            res[b] = blk
        return torch.from_numpy(res).to(blocks.device)

    return _framed_run(sig, plan, on_host, device, "complex128")
