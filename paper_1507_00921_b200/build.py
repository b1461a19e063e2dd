"""Build libdbp_b200.so in-tree with nvcc for sm_100a.

    python -m paper_1507_00921_b200.build          # incremental
    python -m paper_1507_00921_b200.build --force

One object per kernel instantiation (N = 2^4 .. 2^13) compiled in parallel,
then linked with static cudart into ``paper_1507_00921_b200/libdbp_b200.so``.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
BUILD = PKG.parent / "build" / "obj"
LIB = PKG / "libdbp_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "-diag-suppress", "177"]


# per-unit flags: the N = 2048 FFE polarisation-split kernel gains 1.9% at ptxas register-usage
# level 8, every other kernel is fastest at the default (profiles/r2/ab_regusage.txt, ab_ffe_unit.txt)
UNIT_FLAGS = {"dbp_kernel_ffe_ps": ["-Xptxas", "--register-usage-level=8"]}


def nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(exe).exists():
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libdbp_b200.so")
    return exe


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _headers():
    return sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + sorted(INCLUDE.glob("*.h"))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra_flags=None, lib: Path | None = None,
          obj_dir: Path | None = None) -> Path:
    """Compile and link; ``lib`` / ``obj_dir`` redirect a variant build (A/B experiments)."""
    obj_root = Path(obj_dir) if obj_dir else BUILD
    lib_path = Path(lib) if lib else LIB
    obj_root.mkdir(parents=True, exist_ok=True)
    extra = list(extra_flags or [])
    env_flags = os.environ.get("DBP_NVCC_FLAGS", "").split()
    headers = _headers()
    jobs = []
    for src in _sources():
        obj = obj_root / (src.stem + ".o")
        if force or _stale(obj, [src, *headers, Path(__file__)]):
            cmd = [nvcc(), *ARCH, *FLAGS, *UNIT_FLAGS.get(src.stem, []), *extra, *env_flags,
                   "-I", str(CSRC), "-I", str(INCLUDE),
                   "-c", str(src), "-o", str(obj)]
            jobs.append((src, obj, cmd))

    def run(job):
        src, obj, cmd = job
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stdout}\n{res.stderr}")
        return obj

    if jobs:
        with ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as pool:
            list(pool.map(run, jobs))
    objs = [obj_root / (s.stem + ".o") for s in _sources()]
    if force or jobs or _stale(lib_path, objs):
        # static cudart and nothing else: no cuFFT / cuBLAS in the product library
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(lib_path), *map(str, objs)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    return lib_path


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    args = ap.parse_args(argv)
    lib = build(force=args.force, verbose=args.verbose)
    print(lib)


if __name__ == "__main__":
    sys.exit(main())
