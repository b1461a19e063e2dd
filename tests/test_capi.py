"""The C-ABI library loads and exports every symbol include/dbp_b200.h declares (no GPU needed)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_1507_00921_b200 import _native

HEADER = Path(__file__).resolve().parent.parent / "include" / "dbp_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(dbp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_abi():
    names = declared_functions()
    assert "dbp_run" in names and "dbp_plan_create" in names and len(names) >= 15


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, f"{name} not bound in _native.SIGNATURES"


def test_error_paths_without_gpu():
    lib = _native.load_library()
    assert lib.dbp_version() >= 100
    if _native.device_count() > 0:
        pytest.skip("a GPU is visible; the no-device path is not exercised")
    h = ctypes.c_void_p()
    rc = lib.dbp_plan_create(ctypes.byref(h), 0, 2048, 700)
    assert rc == _native.DBP_ECUDA
    assert b"no CUDA device" in lib.dbp_last_error()
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _native.NativePlan(0, 2048, 700)


def test_invalid_geometry_rejected_before_device_lookup():
    lib = _native.load_library()
    h = ctypes.c_void_p()
    assert lib.dbp_plan_create(ctypes.byref(h), 0, 1000, 100) == _native.DBP_EINVAL
    assert b"power of two" in lib.dbp_last_error()
    assert lib.dbp_plan_create(ctypes.byref(h), 0, 1024, 1024) == _native.DBP_EINVAL
    # any power of two up to 2^22 (the general path beyond the fused kernel's 8192)
    assert lib.dbp_plan_create(ctypes.byref(h), 0, 1 << 23, 0) == _native.DBP_EINVAL
    assert b"above the supported" in lib.dbp_last_error()
    assert lib.dbp_version() >= 102


def test_framing_validates_before_touching_the_device():
    lib = _native.load_library()
    f, u = lib.dbp_frame_blocks, lib.dbp_unframe_blocks
    assert f(None, None, 100, 1, 1000, 100, 0, 1, 8, None) == _native.DBP_EINVAL
    assert b"power of two" in lib.dbp_last_error()
    assert f(None, None, 100, 1, 1024, 1024, 0, 1, 8, None) == _native.DBP_EINVAL
    assert u(None, None, 100, 1, 1024, 100, 0, 1, 12, None) == _native.DBP_EINVAL
    assert b"elem_bytes" in lib.dbp_last_error()
    assert u(None, None, 100, 1, 1024, 100, 0, 2, 8, None) == _native.DBP_EINVAL   # one block only
    assert b"block range" in lib.dbp_last_error()
    assert f(None, None, 0, 1, 1024, 100, 0, 0, 8, None) == _native.DBP_EINVAL
    # nothing to do: no device needed
    assert f(None, None, 100, 0, 1024, 100, 0, 1, 16, None) == _native.DBP_OK
    assert f(None, None, 100, 1, 1024, 100, 0, 1, 8, None) == _native.DBP_EINVAL   # null buffers
    assert b"null" in lib.dbp_last_error()


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _native.load_library(tmp_path / "nope.so")


def test_product_library_links_no_fft_or_blas_library():
    # SURVEY 8(a) / north_star: cuFFT only as a cross-check, never in the product path;
    # the library links static cudart and the C/C++ runtime only
    import subprocess
    out = subprocess.run(["ldd", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    for lib in ("cufft", "cublas", "cudnn", "libcudart.so"):
        assert lib not in out, out
    syms = subprocess.run(["nm", "-D", "--undefined-only", str(_native.LIB_PATH)], capture_output=True,
                          text=True).stdout
    assert "cufft" not in syms.lower()
