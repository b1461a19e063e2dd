"""ctypes binding of libdbp_b200.so (the C ABI in include/dbp_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA
device is visible, every entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("DBP_LIB") or Path(__file__).resolve().parent / "libdbp_b200.so")

DBP_OK, DBP_EINVAL, DBP_ECUDA, DBP_ENOMEM, DBP_ESTATE = 0, -1, -2, -3, -4
ALG_CODES = {"ffe": 0, "ssfm": 1, "essfm": 2, "rotate": 3, "identity": 4}
ARR_CODES = {"symmetric": 0, "linear-first": 1, "nonlinear-first": 2}
# any power-of-two block length in [MIN_BLOCK_LEN, MAX_BLOCK_LEN]; the fused
# block kernel covers [FUSED_MIN_BLOCK_LEN, FUSED_MAX_BLOCK_LEN], the rest runs
# the float64 multi-kernel path (csrc/dbp_general.cuh)
MIN_BLOCK_LEN, MAX_BLOCK_LEN, MAX_SIDE_COEFFS = 1, 1 << 22, 64
FUSED_MIN_BLOCK_LEN, FUSED_MAX_BLOCK_LEN = 16, 8192

# every symbol include/dbp_b200.h declares, with (restype, argtypes)
_c_int, _c_void_p, _c_int64, _c_double_p = ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_double)
SIGNATURES = {
    "dbp_last_error": (ctypes.c_char_p, []),
    "dbp_version": (_c_int, []),
    "dbp_device_count": (_c_int, [ctypes.POINTER(_c_int)]),
    "dbp_plan_create": (_c_int, [ctypes.POINTER(_c_void_p), _c_int, _c_int, _c_int]),
    "dbp_plan_destroy": (_c_int, [_c_void_p]),
    "dbp_plan_set_linear": (_c_int, [_c_void_p, _c_double_p, _c_double_p]),
    "dbp_plan_set_steps": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_double_p, _c_double_p,
                                    ctypes.c_double, _c_double_p, _c_int]),
    "dbp_num_blocks": (_c_int, [_c_void_p, _c_int64, ctypes.POINTER(_c_int64)]),
    "dbp_run": (_c_int, [_c_void_p, _c_void_p, _c_void_p, _c_int64, _c_int, _c_int64, _c_int64, _c_void_p]),
    "dbp_run_chunk": (_c_int, [_c_void_p, _c_void_p, _c_void_p, _c_int64, _c_int, _c_int64, _c_int64,
                               _c_int64, _c_int64, _c_void_p]),
    "dbp_run_host": (_c_int, [_c_void_p, _c_void_p, _c_void_p, _c_int64, _c_int, _c_int64, _c_int64]),
    "dbp_plan_set_staging": (_c_int, [_c_void_p, ctypes.c_size_t]),
    "dbp_backpropagate_c128": (_c_int, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_int64]),
    "dbp_nonlinear_substep_c128": (_c_int, [_c_int, _c_void_p, _c_void_p, _c_int64, ctypes.c_double,
                                            ctypes.c_double, _c_double_p, _c_int]),
    "dbp_process_blocks": (_c_int, [_c_void_p, _c_void_p, _c_void_p, _c_int64, _c_void_p]),
    "dbp_frame_blocks": (_c_int, [_c_void_p, _c_void_p, _c_int64, _c_int, _c_int, _c_int, _c_int64, _c_int64,
                                  _c_int, _c_void_p]),
    "dbp_unframe_blocks": (_c_int, [_c_void_p, _c_void_p, _c_int64, _c_int, _c_int, _c_int, _c_int64, _c_int64,
                                    _c_int, _c_void_p]),
    "dbp_plan_synchronize": (_c_int, [_c_void_p]),
    "dbp_host_alloc": (_c_int, [ctypes.POINTER(_c_void_p), ctypes.c_size_t]),
    "dbp_host_free": (_c_int, [_c_void_p]),
    "dbp_launch_count": (_c_int64, []),
    "dbp_probe_fp32_peak": (_c_int, [_c_int, _c_int, ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(ctypes.c_double)]),
    "dbp_probe_fp32x2_peak": (_c_int, [_c_int, _c_int, ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_double)]),
    "dbp_probe_fp32_mixed_peak": (_c_int, [_c_int, _c_int, _c_int, ctypes.POINTER(ctypes.c_double),
                                           ctypes.POINTER(ctypes.c_double)]),
    "dbp_plan_set_coeff_batch": (_c_int, [_c_void_p, _c_double_p, _c_int, _c_int]),
    "dbp_run_coeff_batch": (_c_int, [_c_void_p, _c_void_p, _c_void_p, _c_int64, _c_int64, _c_int64,
                                     _c_void_p]),
    "dbp_run_host_coeff_batch": (_c_int, [_c_void_p, _c_void_p, _c_void_p, _c_int64]),
    "dbp_sim_create": (_c_int, [ctypes.POINTER(_c_void_p), _c_int, _c_int, _c_int]),
    "dbp_sim_destroy": (_c_int, [_c_void_p]),
    "dbp_sim_length": (_c_int, [_c_void_p, ctypes.POINTER(_c_int64)]),
    "dbp_sim_upload": (_c_int, [_c_void_p, _c_void_p, _c_int]),
    "dbp_sim_download": (_c_int, [_c_void_p, _c_void_p, _c_int]),
    "dbp_sim_span": (_c_int, [_c_void_p, _c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                              ctypes.c_double, ctypes.c_double, ctypes.c_double, _c_int, _c_int]),
    "dbp_sim_amplify": (_c_int, [_c_void_p, _c_int, ctypes.c_double, _c_void_p, _c_double_p]),
    "dbp_fit_sumsq": (_c_int, [_c_void_p, _c_int, _c_int64, _c_void_p, _c_int64, _c_int64, ctypes.c_double,
                               _c_double_p, _c_void_p]),
    "dbp_fit_normal": (_c_int, [_c_void_p, _c_int, _c_int64, _c_void_p, _c_void_p, _c_int64, _c_int64,
                                ctypes.c_double, ctypes.c_double, _c_double_p, _c_double_p, _c_void_p]),
    "dbp_fft_c2c": (_c_int, [_c_int, _c_void_p, _c_void_p, _c_int64, _c_int64, _c_int]),
    "dbp_phase_noise": (_c_int, [_c_int, _c_void_p, _c_double_p, _c_void_p, _c_int64]),
    "dbp_rx_create": (_c_int, [ctypes.POINTER(_c_void_p), _c_int, _c_int64, _c_int]),
    "dbp_rx_destroy": (_c_int, [_c_void_p]),
    "dbp_rx_equalize": (_c_int, [_c_void_p, _c_void_p, _c_int, _c_int, ctypes.c_double, _c_int, _c_void_p,
                                 ctypes.POINTER(_c_int), _c_void_p]),
    "dbp_rx_carrier_recover": (_c_int, [_c_void_p, _c_void_p, _c_int, ctypes.c_double, _c_void_p, _c_int,
                                        _c_void_p, _c_double_p, ctypes.POINTER(_c_int)]),
    "dbp_rx_decide": (_c_int, [_c_void_p, _c_void_p, _c_int, _c_void_p]),
    "dbp_rx_count_errors": (_c_int, [_c_void_p, _c_void_p, _c_int, _c_void_p, _c_int64,
                                     ctypes.POINTER(_c_int64), ctypes.POINTER(_c_int64)]),
    "dbp_rx_chain": (_c_int, [_c_void_p, _c_void_p, _c_int, _c_int, _c_int, ctypes.c_double, _c_int,
                              ctypes.c_double, _c_void_p, _c_int, _c_int64, _c_double_p, ctypes.POINTER(_c_int)]),
}

_lib = None
_lock = threading.Lock()


def load_library(path: str | os.PathLike | None = None):
    """Load (once) and type the C ABI.  Raises RuntimeError when absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"{p} is missing: build the CUDA library first "
                "(python -m paper_1507_00921_b200.build); there is no CPU fallback")
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            if name in OPTIONAL and not hasattr(lib, name):
                continue   # measurement probes absent from older A/B variant builds
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def _check(rc: int, what: str):
    if rc == DBP_OK:
        return
    msg = load_library().dbp_last_error().decode(errors="replace")
    if rc == DBP_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed ({rc}): {msg}")


def device_count() -> int:
    n = ctypes.c_int(0)
    _check(load_library().dbp_device_count(ctypes.byref(n)), "dbp_device_count")
    return n.value


def launch_count() -> int:
    return int(load_library().dbp_launch_count())


def probe_fp32_peak(device: int = 0, iters: int = 4096) -> tuple[float, float]:
    """(TFLOP/s, ms) of the FFMA throughput probe on ``device``."""
    tf, ms = ctypes.c_double(), ctypes.c_double()
    _check(load_library().dbp_probe_fp32_peak(int(device), int(iters), ctypes.byref(tf), ctypes.byref(ms)),
           "dbp_probe_fp32_peak")
    return tf.value, ms.value


def probe_fp32x2_peak(device: int = 0, iters: int = 4096) -> tuple[float, float]:
    """(TFLOP/s, ms) of the packed FFMA2 throughput probe on ``device``."""
    tf, ms = ctypes.c_double(), ctypes.c_double()
    _check(load_library().dbp_probe_fp32x2_peak(int(device), int(iters), ctypes.byref(tf), ctypes.byref(ms)),
           "dbp_probe_fp32x2_peak")
    return tf.value, ms.value


def probe_fp32_mixed_peak(device: int = 0, iters: int = 4096, scalar_chains: int = 8) -> tuple[float, float]:
    """(TFLOP/s, ms) of 8 FFMA2 + ``scalar_chains`` FFMA chains interleaved on ``device``."""
    tf, ms = ctypes.c_double(), ctypes.c_double()
    _check(load_library().dbp_probe_fp32_mixed_peak(int(device), int(iters), int(scalar_chains), ctypes.byref(tf),
                                                     ctypes.byref(ms)), "dbp_probe_fp32_mixed_peak")
    return tf.value, ms.value


OPTIONAL = {"dbp_probe_fp32_mixed_peak"}


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class NativePlan:
    """Owner of one ``dbp_plan`` (device tables + staging) on one device."""

    def __init__(self, device: int, block_len: int, overlap: int):
        lib = load_library()
        if device_count() == 0:
            raise RuntimeError("no CUDA device visible: the B200 DBP path has no CPU fallback")
        h = ctypes.c_void_p()
        _check(lib.dbp_plan_create(ctypes.byref(h), int(device), int(block_len), int(overlap)),
               "dbp_plan_create")
        self._h = h
        self._lib = lib
        self.device = int(device)
        self.block_len = int(block_len)
        self.overlap = int(overlap)
        self.lock = threading.RLock()

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            with self.lock:   # never under a running call
                self._lib.dbp_plan_destroy(self._h)
                self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def set_linear(self, kernel: np.ndarray, half_kernel: np.ndarray | None):
        k = np.ascontiguousarray(np.asarray(kernel, dtype=np.complex128)).view(np.float64)
        hk = None if half_kernel is None else np.ascontiguousarray(
            np.asarray(half_kernel, dtype=np.complex128)).view(np.float64)
        _check(self._lib.dbp_plan_set_linear(self._h, _dptr(k), None if hk is None else _dptr(hk)),
               "dbp_plan_set_linear")

    def set_steps(self, algorithm: str, arrangement: str, weights, gains, gamma: float, coeffs=None):
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
        g = np.ascontiguousarray(np.asarray(gains, dtype=np.float64))
        c = np.ascontiguousarray(np.asarray([1.0] if coeffs is None else coeffs, dtype=np.float64))
        _check(self._lib.dbp_plan_set_steps(self._h, ALG_CODES[algorithm], ARR_CODES[arrangement],
                                            int(w.size), _dptr(w), _dptr(g), float(gamma), _dptr(c),
                                            int(c.size - 1)), "dbp_plan_set_steps")

    def set_staging(self, nbytes: int):
        _check(self._lib.dbp_plan_set_staging(self._h, int(nbytes)), "dbp_plan_set_staging")

    def num_blocks(self, n_total: int) -> int:
        out = ctypes.c_int64()
        _check(self._lib.dbp_num_blocks(self._h, int(n_total), ctypes.byref(out)), "dbp_num_blocks")
        return out.value

    def run_host(self, h_in: np.ndarray, h_out: np.ndarray, n_total: int, batch: int,
                 block_begin: int, block_end: int):
        """h_in / h_out: C-contiguous complex64 arrays of shape (batch, 2, n_total)."""
        for a in (h_in, h_out):
            if a.dtype != np.complex64 or not a.flags.c_contiguous or a.size != batch * 2 * n_total:
                raise ValueError("host buffers must be C-contiguous complex64 (batch, 2, n)")
        _check(self._lib.dbp_run_host(self._h, h_in.ctypes.data, h_out.ctypes.data, int(n_total),
                                      int(batch), int(block_begin), int(block_end)), "dbp_run_host")

    def backpropagate_c128(self, x: np.ndarray, y: np.ndarray, out_x: np.ndarray, out_y: np.ndarray):
        """The drop-in call on complex128 rows (dbp_backpropagate_c128): x, y -> out_x, out_y."""
        n = x.size
        for a in (x, y, out_x, out_y):
            if a.dtype != np.complex128 or not a.flags.c_contiguous or a.ndim != 1 or a.size != n:
                raise ValueError("rows must be C-contiguous 1-D complex128 arrays of equal length")
        _check(self._lib.dbp_backpropagate_c128(self._h, x.ctypes.data, y.ctypes.data, out_x.ctypes.data,
                                                out_y.ctypes.data, int(n)), "dbp_backpropagate_c128")

    def run_host_ptr(self, p_in: int, p_out: int, n_total: int, batch: int, block_begin: int,
                     block_end: int):
        _check(self._lib.dbp_run_host(self._h, p_in, p_out, int(n_total), int(batch),
                                      int(block_begin), int(block_end)), "dbp_run_host")

    def run_device(self, d_in: int, d_out: int, n_total: int, batch: int, block_begin: int,
                   block_end: int, stream: int = 0):
        _check(self._lib.dbp_run(self._h, d_in, d_out, int(n_total), int(batch), int(block_begin),
                                 int(block_end), stream or None), "dbp_run")

    def run_chunk(self, d_in: int, d_out: int, n_total: int, batch: int, block_begin: int,
                  block_end: int, in_len: int, out_len: int, stream: int = 0):
        _check(self._lib.dbp_run_chunk(self._h, d_in, d_out, int(n_total), int(batch),
                                       int(block_begin), int(block_end), int(in_len), int(out_len),
                                       stream or None), "dbp_run_chunk")

    def process_blocks(self, d_in: int, d_out: int, n_blocks: int, stream: int = 0):
        _check(self._lib.dbp_process_blocks(self._h, d_in, d_out, int(n_blocks), stream or None),
               "dbp_process_blocks")

    def set_coeff_batch(self, coeff_sets: np.ndarray):
        """coeff_sets: (n_sets, n_coeffs + 1) float64."""
        c = np.ascontiguousarray(np.asarray(coeff_sets, dtype=np.float64))
        if c.ndim != 2:
            raise ValueError("coefficient sets must be a (n_sets, n_coeffs + 1) array")
        _check(self._lib.dbp_plan_set_coeff_batch(self._h, _dptr(c), int(c.shape[0]), int(c.shape[1] - 1)),
               "dbp_plan_set_coeff_batch")
        self.n_sets = int(c.shape[0])

    def run_host_coeff_batch(self, h_in: np.ndarray, h_out: np.ndarray, n_total: int):
        """h_in (2, n) complex64, h_out (n_sets, 2, n) complex64, both C-contiguous."""
        if h_in.dtype != np.complex64 or h_out.dtype != np.complex64:
            raise ValueError("host buffers must be complex64")
        if not (h_in.flags.c_contiguous and h_out.flags.c_contiguous):
            raise ValueError("host buffers must be C-contiguous")
        if h_in.size != 2 * n_total or h_out.size != self.n_sets * 2 * n_total:
            raise ValueError("host buffer sizes do not match (2, n) / (n_sets, 2, n)")
        _check(self._lib.dbp_run_host_coeff_batch(self._h, h_in.ctypes.data, h_out.ctypes.data, int(n_total)),
               "dbp_run_host_coeff_batch")

    def run_coeff_batch(self, d_in: int, d_out: int, n_total: int, stream: int = 0):
        """Device buffers: d_in [2][n] complex64, d_out [n_sets][2][n] complex64 (async on ``stream``)."""
        nb = self.num_blocks(n_total)
        _check(self._lib.dbp_run_coeff_batch(self._h, d_in, d_out, int(n_total), 0, int(nb), stream or None),
               "dbp_run_coeff_batch")

    def synchronize(self):
        _check(self._lib.dbp_plan_synchronize(self._h), "dbp_plan_synchronize")


class PinnedBuffer:
    """Page-locked host buffer viewed as a numpy array (cudaHostAlloc)."""

    def __init__(self, shape, dtype=np.complex64):
        lib = load_library()
        dt = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dt.itemsize
        p = ctypes.c_void_p()
        _check(lib.dbp_host_alloc(ctypes.byref(p), max(nbytes, 1)), "dbp_host_alloc")
        self._p = p
        self._lib = lib
        buf = (ctypes.c_byte * max(nbytes, 1)).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape)

    def free(self):
        if self._p is not None and self._p.value:
            self.array = None
            self._lib.dbp_host_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class NativeSim:
    """Owner of one ``dbp_sim`` (whole-waveform SSFM simulator) on one device."""

    def __init__(self, device: int, log2_n: int, max_batch: int):
        lib = load_library()
        if device_count() == 0:
            raise RuntimeError("no CUDA device visible: the B200 simulator has no CPU fallback")
        h = ctypes.c_void_p()
        _check(lib.dbp_sim_create(ctypes.byref(h), int(device), int(log2_n), int(max_batch)), "dbp_sim_create")
        self._h, self._lib = h, lib
        self.device, self.n, self.max_batch = int(device), 1 << int(log2_n), int(max_batch)
        # the simulator's device state (the resident waveform) belongs to one
        # upload .. download sequence at a time: callers hold this lock
        self.lock = threading.RLock()

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            with self.lock:
                self._lib.dbp_sim_destroy(self._h)
                self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, x: np.ndarray):
        x = np.ascontiguousarray(x, dtype=np.complex64)
        _check(self._lib.dbp_sim_upload(self._h, x.ctypes.data, int(x.shape[0])), "dbp_sim_upload")

    def download(self, batch: int) -> np.ndarray:
        out = np.empty((batch, 2, self.n), dtype=np.complex64)
        _check(self._lib.dbp_sim_download(self._h, out.ctypes.data, int(batch)), "dbp_sim_download")
        return out

    def span(self, batch, sample_rate, beta2, gamma, dz, dz_eff, loss, steps, nonlinear):
        _check(self._lib.dbp_sim_span(self._h, int(batch), float(sample_rate), float(beta2), float(gamma),
                                      float(dz), float(dz_eff), float(loss), int(steps), int(bool(nonlinear))),
               "dbp_sim_span")

    def amplify(self, batch, g_amp, noise=None, jones=None):
        nz = None if noise is None else np.ascontiguousarray(noise, dtype=np.complex64)
        if noise is not None and np.shape(noise) != (batch, 2, self.n):
            raise ValueError(f"noise must have shape ({batch}, 2, {self.n})")
        if jones is not None and np.shape(jones) != (batch, 2, 2):
            raise ValueError(f"jones must have shape ({batch}, 2, 2)")
        jj = None if jones is None else np.ascontiguousarray(np.asarray(jones, dtype=np.complex128)).view(np.float64)
        _check(self._lib.dbp_sim_amplify(self._h, int(batch), float(g_amp),
                                         None if nz is None else nz.ctypes.data,
                                         None if jj is None else _dptr(jj)), "dbp_sim_amplify")


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


class NativeRx:
    """Owner of one ``dbp_rx`` (float64 receiver DSP) for waveforms of 2 n_symbols samples."""

    def __init__(self, device: int, n_symbols: int, max_batch: int):
        lib = load_library()
        if device_count() == 0:
            raise RuntimeError("no CUDA device visible: the B200 receiver has no CPU fallback")
        h = ctypes.c_void_p()
        _check(lib.dbp_rx_create(ctypes.byref(h), int(device), int(n_symbols), int(max_batch)), "dbp_rx_create")
        self._h, self._lib = h, lib
        self.device, self.n_symbols, self.max_batch = int(device), int(n_symbols), int(max_batch)
        self.lock = threading.RLock()   # one call at a time on the device buffers

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            with self.lock:
                self._lib.dbp_rx_destroy(self._h)
                self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def equalize(self, x: np.ndarray, taps: int, step_size: float, passes: int, want_taps: bool = False):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        b = x.shape[0]
        out = np.empty((b, 2, self.n_symbols), dtype=np.complex128)
        reinits = np.zeros(b, dtype=np.int32)
        tp = np.empty((b, 4, taps), dtype=np.complex128) if want_taps else None
        with self.lock:
            _check(self._lib.dbp_rx_equalize(self._h, x.ctypes.data, b, int(taps), float(step_size), int(passes),
                                              out.ctypes.data, _iptr(reinits), None if tp is None else tp.ctypes.data),
                   "dbp_rx_equalize")
        return out, reinits, tp

    def carrier_recover(self, s: np.ndarray, symbol_rate: float, reference, window: int):
        s = np.ascontiguousarray(s, dtype=np.complex128)
        b = s.shape[0]
        ref = None if reference is None else np.ascontiguousarray(reference, dtype=np.complex128)
        out = np.empty_like(s)
        f_off = np.zeros(b)
        status = np.zeros(b, dtype=np.int32)
        with self.lock:
            _check(self._lib.dbp_rx_carrier_recover(self._h, s.ctypes.data, b, float(symbol_rate),
                                                    None if ref is None else ref.ctypes.data, int(window),
                                                    out.ctypes.data, _dptr(f_off), _iptr(status)),
                   "dbp_rx_carrier_recover")
        return out, f_off, status

    def decide(self, s: np.ndarray) -> np.ndarray:
        s = np.ascontiguousarray(s, dtype=np.complex128)
        bits = np.empty(s.shape[:-1] + (2 * s.shape[-1],), dtype=np.uint8)
        with self.lock:
            _check(self._lib.dbp_rx_decide(self._h, s.ctypes.data, s.shape[0], bits.ctypes.data), "dbp_rx_decide")
        return bits

    def count_errors(self, dec: np.ndarray, ref: np.ndarray, skip_bits: int):
        dec = np.ascontiguousarray(dec, dtype=np.uint8)
        ref = np.ascontiguousarray(ref, dtype=np.uint8)
        b = dec.shape[0]
        errors = np.zeros(b, dtype=np.int64)
        counted = ctypes.c_int64()
        with self.lock:
            _check(self._lib.dbp_rx_count_errors(self._h, dec.ctypes.data, b, ref.ctypes.data, int(skip_bits),
                                                  errors.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                                  ctypes.byref(counted)), "dbp_rx_count_errors")
        return errors, counted.value

    def chain(self, x: np.ndarray, taps, step_size, passes, symbol_rate, ref_symbols, window, skip_bits):
        c64 = np.asarray(x).dtype == np.complex64
        x = np.ascontiguousarray(x, dtype=np.complex64 if c64 else np.complex128)
        b = x.shape[0]
        ref = np.ascontiguousarray(ref_symbols, dtype=np.complex128)
        metrics = np.zeros((b, 6))
        status = np.zeros(b, dtype=np.int32)
        with self.lock:
            _check(self._lib.dbp_rx_chain(self._h, x.ctypes.data, int(c64), b, int(taps), float(step_size), int(passes),
                                          float(symbol_rate), ref.ctypes.data, int(window), int(skip_bits),
                                          _dptr(metrics), _iptr(status)), "dbp_rx_chain")
        return metrics, status


def fit_sumsq(d_out: int, n_sets: int, n_total: int, d_target: int, w0: int, w1: int, scale: float,
              stream: int = 0) -> np.ndarray:
    out = np.zeros(n_sets)
    _check(load_library().dbp_fit_sumsq(d_out, int(n_sets), int(n_total), d_target, int(w0), int(w1), float(scale),
                                        _dptr(out), stream or None), "dbp_fit_sumsq")
    return out


def fit_normal(d_out: int, n_params: int, n_total: int, d_target: int, d_base: int, w0: int, w1: int,
               scale: float, fd_step: float, stream: int = 0) -> tuple[np.ndarray, np.ndarray]:
    ata = np.zeros((n_params, n_params))
    atr = np.zeros(n_params)
    _check(load_library().dbp_fit_normal(d_out, int(n_params), int(n_total), d_target, d_base, int(w0), int(w1),
                                         float(scale), float(fd_step), _dptr(ata), _dptr(atr), stream or None),
           "dbp_fit_normal")
    return ata, atr


def frame_blocks(d_sig: int, d_blocks: int, n_total: int, batch: int, block_len: int, overlap: int,
                 block_begin: int, block_end: int, elem_bytes: int, stream: int = 0):
    """[batch][2][n] -> [batch][nblk][2][N] cyclic overlap-save blocks (device pointers, async)."""
    _check(load_library().dbp_frame_blocks(d_sig, d_blocks, int(n_total), int(batch), int(block_len), int(overlap),
                                           int(block_begin), int(block_end), int(elem_bytes), stream or None),
           "dbp_frame_blocks")


def unframe_blocks(d_blocks: int, d_out: int, n_total: int, batch: int, block_len: int, overlap: int,
                   block_begin: int, block_end: int, elem_bytes: int, stream: int = 0):
    """Kept block centres -> output samples [begin step, min(n, end step)) (device pointers, async)."""
    _check(load_library().dbp_unframe_blocks(d_blocks, d_out, int(n_total), int(batch), int(block_len),
                                             int(overlap), int(block_begin), int(block_end), int(elem_bytes),
                                             stream or None), "dbp_unframe_blocks")


def fft_c2c(x: np.ndarray, inverse: bool, device: int = 0) -> np.ndarray:
    """Float64 DFT along the last axis on the GPU (own Stockham FFT, fft64.cuh); inverse scaled by 1/n."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    n = a.shape[-1]
    out = np.empty_like(a)
    batch = a.size // n if n else 0
    if batch == 0:
        return out
    if device_count() == 0:
        raise RuntimeError("no CUDA device visible: the GPU FFT has no CPU fallback")
    _check(load_library().dbp_fft_c2c(int(device), a.ctypes.data, out.ctypes.data, int(n), int(batch),
                                      int(bool(inverse))), "dbp_fft_c2c")
    return out


def phase_noise(x: np.ndarray, increments: np.ndarray, device: int = 0) -> np.ndarray:
    """(2, n) complex128 * exp(j cumsum(increments)) on the GPU."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    inc = np.ascontiguousarray(np.asarray(increments, dtype=np.float64))
    if a.ndim != 2 or a.shape[0] != 2 or inc.shape != (a.shape[1],):
        raise ValueError("expected a (2, n) waveform and n increments")
    if device_count() == 0:
        raise RuntimeError("no CUDA device visible: the GPU phase-noise path has no CPU fallback")
    out = np.empty_like(a)
    _check(load_library().dbp_phase_noise(int(device), a.ctypes.data, _dptr(inc), out.ctypes.data,
                                          int(a.shape[1])), "dbp_phase_noise")
    return out


def nonlinear_substep(block: np.ndarray, gamma: float, dz_eff: float, coeffs, device: int = 0) -> np.ndarray:
    """(2, n) complex128 block * exp(-j gamma dz_eff F) on the GPU, any n > 2 N_c (float64)."""
    a = np.ascontiguousarray(np.asarray(block, dtype=np.complex128))
    c = np.ascontiguousarray(np.asarray(coeffs, dtype=np.float64))
    if device_count() == 0:
        raise RuntimeError("no CUDA device visible: the GPU sub-step has no CPU fallback")
    out = np.empty_like(a)
    _check(load_library().dbp_nonlinear_substep_c128(int(device), a.ctypes.data, out.ctypes.data, int(a.shape[1]),
                                                     float(gamma), float(dz_eff), _dptr(c), int(c.size - 1)),
           "dbp_nonlinear_substep_c128")
    return out
