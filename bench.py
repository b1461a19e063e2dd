#!/usr/bin/env python
"""B200 benchmark of the ESSFM single-step DBP hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE configs[3] batch with the configs[0] DBP): per GPU 512
independent seeded dual-pol waveforms x 2^18 samples (complex64, 2 GiB in +
2 GiB out, larger than the 126 MB L2 so no flush is needed), ESSFM N_s=1,
N_c=17, overlap-save N=2048 / M=700, symmetric arrangement (the reference
API default), 40 x 80 km SMF link, fs = 56 GHz.  One step = one launch of
the fused block kernel over the whole per-GPU batch.  Multi-GPU: one process
per GPU (torchrun), each its own 512 waveforms (weak scaling, no data-path
collective), timed with CUDA events, max over ranks.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the reference's
own CPU implementation, ``fiberdbp.dbp.backpropagate`` installed unmodified
in oracle/_ref (oracle/install_ref.sh), on this host's cores instead (rank 0
only; the oracle port only if oracle/_ref is absent).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

METRIC = "ESSFM 1-step DBP Gsamples/s (dual-pol)"
UNIT = "Gsamples/s"
SAMPLE_RATE = 56e9
POWER_DBM = 0.0


def parse_args(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--waveforms", type=int, default=512, help="waveforms per GPU")
    ap.add_argument("--log2-samples", type=int, default=18)
    ap.add_argument("--algorithm", default="essfm", choices=("ffe", "ssfm", "essfm"))
    ap.add_argument("--arrangement", default="symmetric",
                    choices=("symmetric", "linear-first", "nonlinear-first"))
    ap.add_argument("--num-steps", type=int, default=1)
    ap.add_argument("--nc", type=int, default=17)
    ap.add_argument("--block-len", type=int, default=2048)
    ap.add_argument("--overlap", type=int, default=700)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------
# configuration and algorithmic work per output sample
# ---------------------------------------------------------------------------

def link_kwargs():
    from oracle.waveforms import d_to_beta2
    return dict(beta2=d_to_beta2(17.0), gamma=1.3, alpha_db_per_km=0.2, span_km=80.0, num_spans=40)


def port_kwargs(a) -> dict:
    from oracle.waveforms import gaussian_coeffs
    lk = link_kwargs()
    return dict(algorithm=a.algorithm, block_len=a.block_len, overlap=a.overlap, beta2=lk["beta2"],
                gamma=lk["gamma"], alpha_db_per_km=lk["alpha_db_per_km"], span_km=lk["span_km"],
                num_spans=lk["num_spans"], num_steps=a.num_steps,
                coeffs=gaussian_coeffs(a.nc) if a.algorithm == "essfm" else None,
                arrangement=a.arrangement)


def make_cfg(a):
    import paper_1507_00921_b200 as pb
    from oracle.waveforms import gaussian_coeffs
    lk = link_kwargs()
    span = pb.FiberParams(lk["beta2"], lk["gamma"], lk["alpha_db_per_km"], lk["span_km"])
    link = pb.LinkConfig(span, lk["num_spans"], amp_noise_figure_db=None, pol_rotation=False)
    coeffs = pb.EssfmCoefficients(gaussian_coeffs(a.nc)) if a.algorithm == "essfm" else None
    return pb.DbpConfig(a.algorithm, pb.OverlapPlan(a.block_len, a.overlap), link,
                        num_steps=a.num_steps, coeffs=coeffs, arrangement=a.arrangement)


def work_per_sample(a, gains_not_one: bool = False) -> tuple[float, float]:
    """(FP32 flops, HBM bytes) per output sample, FFTW 5 N log2 N convention
    (paper_1507_00921_b200.costmodel.work_per_sample)."""
    from paper_1507_00921_b200.costmodel import work_per_sample as wps

    return wps(a.algorithm, a.block_len, a.overlap, a.nc, a.num_steps, a.arrangement, gains_not_one)


def kernel_twp(a) -> int:
    """The FFT flavour the launcher picks (csrc/launch.h): 4 = fused-twiddle
    decimation in time (FFE and programs of <= 2 steps, N <= 4096), 3 = the
    exact-adjoint FFT."""
    import math as _m
    steps = 0 if a.algorithm == "ffe" else a.num_steps
    logn = int(_m.log2(a.block_len))
    dit = a.algorithm == "ffe" or steps <= 2
    # the R2 kernel's 4096-point transforms follow the N = 4096 rule
    return 4 if dit and (logn <= 12 or (logn == 13 and a.algorithm != "ffe")) else 3


def kernel_name(a) -> str:
    """The instantiation the launcher picks (csrc/launch.h): the FFE program
    from N = 2048 runs as polarisation-split pairs (template argument PS = 1,
    one CTA per polarisation)."""
    logn = int(math.log2(a.block_len))
    if logn < 4 or logn > 13:
        # outside the fused kernel's range: the float64 multi-kernel path (csrc/dbp_general.cuh)
        return "dbp_general::stockham_pass16 + frame/mul/rotate/store (float64 multi-kernel path)"
    if logn == 13 and a.algorithm != "ffe":
        # N = 8192 split-step programs: the radix-2-around-4096 kernel (csrc/dbp_r2_kernel.cuh)
        return f"dbp::dbp_r2_kernel<{kernel_prog(a)}, {kernel_twp(a)}>"
    ps = a.algorithm == "ffe" and logn >= 11
    return f"dbp::dbp_block_kernel<{logn}, {kernel_prog(a)}, {kernel_twp(a)}{', 1' if ps else ', 0'}>"


def kernel_prog(a) -> int:
    """Which instantiation of the block kernel the launcher picks (csrc/launch.h
    launch_block_kernel_impl): 0 generic (fixed-tap FIR), 1 FFE-only, 2 no-FIR
    split-step, 3 generic FIR (runtime N_c outside {1, 9, 17, 32, 33})."""
    nc = a.nc if a.algorithm == "essfm" else 0
    prog = 0
    if a.block_len >= 2048 and a.algorithm == "ffe":
        prog = 1
    if a.block_len >= 2048 and a.algorithm != "ffe" and nc == 0:
        prog = 2
    if a.algorithm != "ffe" and nc > 0 and nc not in (1, 9, 17, 32, 33):
        prog = 3
    return prog


def cpu_model() -> str:
    """The host CPU model (state the cores and the model beside the CPU figure)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload_config(a, world: int) -> dict:
    return {
        "workload": (f"configs[3] batch with configs[0] DBP: {a.waveforms} x 2^{a.log2_samples} dual-pol "
                     f"waveforms per GPU, {a.algorithm.upper()} Ns={a.num_steps} Nc={a.nc if a.algorithm == 'essfm' else 0} "
                     f"N={a.block_len} M={a.overlap} {a.arrangement}, 40x80 km SMF, 56 GS/s"),
        "algorithm": a.algorithm, "arrangement": a.arrangement, "num_steps": a.num_steps,
        "n_coeffs": a.nc if a.algorithm == "essfm" else 0, "block_len": a.block_len, "overlap": a.overlap,
        "waveforms_per_gpu": a.waveforms, "samples_per_waveform": 1 << a.log2_samples,
        "global_waveforms": a.waveforms * world, "sharding": f"waveforms split over {world} GPU(s), no collective",
        "l2": (f"inputs ({a.waveforms * (16 << a.log2_samples) / 2**30:.3g} GiB/GPU) "
               + ("larger than the 126 MB L2; no flush" if a.waveforms * (16 << a.log2_samples) > 126e6
                  else "NOT larger than L2 (tuning run, not a bench line)")),
    }


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def time_dropin(a, cfg, dev) -> dict:
    """The reference-facing call itself: ``backpropagate(sig, cfg)`` (dbp.py:160)
    on a complex128 ``DualPolSignal`` in host memory, complex128 result back --
    at the configs[0] length (2^17 samples/pol) and at 2^24 samples/pol.  Each
    call includes the casts, the H2D / D2H copies and the synchronisation."""
    import warnings

    import numpy as np

    import paper_1507_00921_b200 as pb
    out = {}
    for log2n, reps in ((17, 50), (24, 5)):
        n = 1 << log2n
        rng = np.random.default_rng(log2n)
        amp = math.sqrt(10 ** ((POWER_DBM - 30) / 10) / 4.0)
        xs = amp * (rng.standard_normal((2, n)) + 1j * rng.standard_normal((2, n)))
        sig = pb.DualPolSignal(xs[0], xs[1], SAMPLE_RATE)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            pb.backpropagate(sig, cfg, device=dev)          # warm: engine, staging, host threads
            t0 = time.perf_counter()
            for _ in range(reps):
                res = pb.backpropagate(sig, cfg, device=dev)
            sec = (time.perf_counter() - t0) / reps
        assert res.x.dtype == np.complex128 and len(res) == n
        out[f"2^{log2n}"] = {"value": n / sec / 1e9, "unit": UNIT, "seconds_per_call": sec, "calls": reps,
                             "h2d_bytes_per_step": 2 * n * 8, "d2h_bytes_per_step": 2 * n * 8,
                             "host_bytes_in": 2 * n * 16, "host_bytes_out": 2 * n * 16}
    out["path"] = ("paper_1507_00921_b200.backpropagate(DualPolSignal complex128, DbpConfig) -> "
                   "dbp_backpropagate_c128 (host-thread casts into pinned staging, chunked H2D / kernel / D2H)")
    return out


def pcie_roof(dev, nbytes: int = 1 << 30, reps: int = 3) -> dict:
    """The host link's ceiling for the e2e leg, measured on this box: pinned
    H2D alone, D2H alone and both at once on two streams (the e2e pipeline
    overlaps the two directions), best of ``reps``, CUDA-event timed."""
    import torch
    h_a = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h_b = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{dev}")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{dev}")
    s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

    def timed(h2d: bool, d2h: bool) -> float:
        best = float("inf")
        for _ in range(reps + 1):
            torch.cuda.synchronize(dev)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            cur = torch.cuda.current_stream(dev)
            e0.record(cur)
            s1.wait_event(e0)
            s2.wait_event(e0)
            if h2d:
                with torch.cuda.stream(s1):
                    d_a.copy_(h_a, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    h_b.copy_(d_b, non_blocking=True)
            e1.record(s1)
            e2.record(s2)
            cur.wait_event(e1)
            cur.wait_event(e2)
            e3 = torch.cuda.Event(enable_timing=True)
            e3.record(cur)
            torch.cuda.synchronize(dev)
            best = min(best, e0.elapsed_time(e3) * 1e-3)
        return best

    timed(True, True)  # warm
    h2d = nbytes / timed(True, False) / 1e9
    d2h = nbytes / timed(False, True) / 1e9
    both = nbytes / timed(True, True) / 1e9   # per direction, both directions at once
    del h_a, h_b, d_a, d_b
    return {"h2d_gbs": h2d, "d2h_gbs": d2h, "bidir_gbs_per_direction": both, "bytes_per_copy": nbytes}


def run_ours(a) -> int:
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1507_00921_b200 as pb
    from paper_1507_00921_b200 import _native

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; BENCH_DIST_BACKEND=gloo (CPU reductions) lets the
    # multi-rank path be exercised with several ranks on one device
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    red_dev = f"cuda:{dev}" if backend == "nccl" else "cpu"
    n = 1 << a.log2_samples
    B = a.waveforms
    cfg = make_cfg(a)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        eng = pb.get_engine(cfg, SAMPLE_RATE, dev)
    nb = eng.num_blocks(n)

    # seeded synthetic input at the launch power, generated on the device
    gen = torch.Generator(device=f"cuda:{dev}")
    gen.manual_seed(1000 + rank)
    amp = math.sqrt(10 ** ((POWER_DBM - 30) / 10) / 4.0)
    d_in = torch.randn((B, 2, n, 2), generator=gen, device=f"cuda:{dev}", dtype=torch.float32) * amp
    d_out = torch.empty_like(d_in)
    stream = torch.cuda.Stream(device=dev)
    sh = stream.cuda_stream

    def step():
        eng.native.run_device(d_in.data_ptr(), d_out.data_ptr(), n, B, 0, nb, sh)

    # FP32 roofline denominator: the better of the scalar FFMA and packed FFMA2 probes
    peak_ffma, _ = _native.probe_fp32_peak(dev, 8192)
    peak_ffma2, _ = _native.probe_fp32x2_peak(dev, 8192)
    peak_tf = max(peak_ffma, peak_ffma2)
    for _ in range(max(3, a.warmup)):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(dev)
    clocks.start()
    time.sleep(0.3)
    l0 = _native.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    launches = _native.launch_count() - l0
    ms = e0.elapsed_time(e1)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())

    samples_all = float(world * B * n * a.steps)
    value = samples_all / (ms_max * 1e-3) / 1e9
    f_s, b_s = work_per_sample(a, gains_not_one=any(g != 1.0 for _, _, g in eng.schedule))
    per_launch_samples = B * n
    launch_s = ms * 1e-3 / a.steps
    achieved_tf = f_s * per_launch_samples / launch_s / 1e12
    achieved_gbs = b_s * per_launch_samples / launch_s / 1e9
    peaks = json.loads((REPO / "MEASURED_PEAKS.json").read_text()) if (REPO / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)

    # DRAM traffic of the same kernel from the committed ncu capture of this command
    traffic, traffic_src = None, None
    prof = REPO / "profiles" / "latest_ncu.json"
    default = (a.algorithm, a.arrangement, a.num_steps, a.nc, a.block_len, a.overlap) == \
        ("essfm", "symmetric", 1, 17, 2048, 700)
    if prof.exists() and default:
        pj = json.loads(prof.read_text())
        if f"dbp_block_kernel<{int(math.log2(a.block_len))}" in str(pj.get("kernel", "")):
            traffic = pj["dram_bytes_per_sample"] * per_launch_samples
            traffic_src = ("profiles/latest_ncu.json: dram__bytes_read.sum + dram__bytes_write.sum of one "
                           "ncu --set full launch of this command, scaled per launch")

    # ---- end to end through the public API with pinned host buffers ----
    e2e = None
    if not a.no_e2e:
        hin = _native.PinnedBuffer((B, 2, n), np.complex64)
        hout = _native.PinnedBuffer((B, 2, n), np.complex64)
        hin.array.view(np.float32).reshape(-1)[:] = d_in.reshape(-1).cpu().numpy()
        eng.run_host(hin.array, hout.array)  # warm (staging allocation)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(a.e2e_steps):
            eng.run_host(hin.array, hout.array)
        e2e_s = time.perf_counter() - t0
        te = torch.tensor([e2e_s], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item())
        e2e = {"value": world * B * n * a.e2e_steps / e2e_s / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": B * 2 * n * 8, "d2h_bytes_per_step": B * 2 * n * 8,
               "path": "DbpEngine.run_host -> dbp_run_host (C ABI), pinned host buffers, 2-stream H2D/kernel/D2H pipeline"}
        # spot parity of the e2e output against the device path
        ok = np.array_equal(hout.array[0].view(np.float32).reshape(-1), d_out[0].reshape(-1).cpu().numpy())
        e2e["matches_device_path"] = bool(ok)
        hin.free()
        hout.free()
        # the e2e leg's own roofline: every step moves Bi host->device and Bo
        # device->host over the host link, overlapped by the 2-stream pipeline
        link = pcie_roof(dev)
        moved = max(e2e["h2d_bytes_per_step"], e2e["d2h_bytes_per_step"])
        per_dir = moved * a.e2e_steps / e2e_s / 1e9
        e2e["roofline"] = {"bound": "pcie", "achieved": per_dir, "peak": link["bidir_gbs_per_direction"],
                           "unit": "GB/s per direction", "frac": per_dir / link["bidir_gbs_per_direction"],
                           "link": link,
                           "note": "achieved = bytes copied each way per step / e2e step time; peak = pinned "
                                   "H2D and D2H copies running at once on this box (measured in this run)"}
        e2e["dropin"] = time_dropin(a, cfg, dev)

    # ---- CPU baseline (rank 0, single-GPU runs only) ----
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        from oracle.cpu_bench import CpuBaseline
        cores = os.cpu_count() or 1
        cb = CpuBaseline(port_kwargs(a), SAMPLE_RATE, n, POWER_DBM, cores)
        # calibrate on two waveforms per core, then time a sample of ~10-30 s of
        # CPU work: the whole per-GPU workload when it fits, else a slice of it
        waves = max(16, 2 * cores)
        secs, _ = cb.step(waves, seed0=100_000)
        per_wave = secs / waves
        waves = a.waveforms if per_wave * a.waveforms <= 30.0 else \
            max(waves, int(15.0 / per_wave) // cores * cores)
        secs, samples = cb.step(waves)
        one_core = cb.one_core_rate()
        cb.close()
        cpu = {"value": samples / secs / 1e9, "unit": UNIT, "cores": cores, "kind": cb.kind,
               "sample": f"{waves} waveforms x 2^{a.log2_samples} samples of the same workload through "
                         + cb.describe(),
               "seconds": secs, "cpu_model": cpu_model(), "one_core_value": one_core / 1e9}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": max(3, a.warmup), "ms_per_step": ms_max / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32 (complex64)",
            "data": "synthetic: seeded complex Gaussian dual-pol waveforms at 0 dBm (dispersed-QPSK stand-in)",
            "config": workload_config(a, world),
            "roofline": {"bound": "fp32", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved_tf / peak_tf,
                         "peak_source": "measured in this run: max of the FFMA probe (dbp_probe_fp32_peak, "
                                        f"{peak_ffma:.1f}) and the packed FFMA2 probe (dbp_probe_fp32x2_peak, "
                                        f"{peak_ffma2:.1f}); MEASURED_PEAKS.json has no FP32 entry",
                         "flops_per_sample": f_s, "traffic": traffic, "traffic_unit": "bytes per launch",
                         "traffic_source": traffic_src,
                         "algorithmic_bytes_per_launch": b_s * per_launch_samples,
                         "kernel": kernel_name(a)},
            "roofline_hbm": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                             "frac": achieved_gbs / hbm_peak, "bytes_per_sample": b_s,
                             "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)"},
            "clocks": clk, "gpu_launches": int(launches), "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU DBP (oracle/_ref) on the host cores
# ---------------------------------------------------------------------------

def run_reference(a) -> int:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    from oracle.cpu_bench import CpuBaseline
    cores = os.cpu_count() or 1
    n = 1 << a.log2_samples
    cb = CpuBaseline(port_kwargs(a), SAMPLE_RATE, n, POWER_DBM, cores)
    for w in range(a.warmup):
        cb.step(cores, seed0=10_000 + w * cores)
    tot_s, tot_n = 0.0, 0.0
    for k in range(a.steps):
        s, m = cb.step(cores, seed0=k * cores)
        tot_s += s
        tot_n += m
    one_core = cb.one_core_rate()
    kind, desc = cb.kind, cb.describe()
    cb.close()
    value = tot_n / tot_s / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": tot_s / a.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp64 (complex128)",
        "data": "synthetic: seeded complex Gaussian dual-pol waveforms at 0 dBm",
        "config": workload_config(a, world), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"each step: {cores} waveforms x 2^{a.log2_samples} samples "
                                   f"(one per core) through {desc}", "cpu_model": cpu_model(),
                         "one_core_value": one_core / 1e9},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main(argv=None) -> int:
    a = parse_args(argv)
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
