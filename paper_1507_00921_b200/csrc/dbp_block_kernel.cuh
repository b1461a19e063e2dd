// Fused overlap-save DBP block kernel for sm_100a (one polarisation per thread).
//
// One overlap-save block of N dual-polarisation samples per block slice of
// 2T threads, T = N/16: lanes 0-15 of a warp carry polarisation x and lanes
// 16-31 polarisation y of the same 16 sample positions, 16 samples per
// thread (positions t + T m, m = 0..15).  The whole multi-step program --
// dispersion filter (FFT -> x table -> IFFT), the SSFM / ESSFM nonlinear
// rotation with the in-block cyclic intensity FIR, gains -- runs on-chip
// between ONE coalesced load of the block (with its halo, cyclic wrap of the
// whole signal) and ONE store of its centre.
//
// Reference behaviour reproduced (pkg/src/fiberdbp/...):
//   framing  spectral.py:122-145  block b = samples [b*step - M/2, +N) mod n,
//                                 keep [M/2, M/2 + step), trim to n
//   FFE      dbp.py:185-191       ifft(fft(b) * H)
//   SSFM     dbp.py:193-235       symmetric / linear-first / nonlinear-first
//   rotate   dbp.py:49-75, channel.py:61-71
//            b * exp(-j g w (c0 I_k + sum_i c_i (I_{k-i} + I_{k+i}))), cyclic in-block
//
// FFT: N = R0 * 16^(NP-1), passes radix R0 (2..16, G0 = 16/R0 groups per
// thread) then radix 16.  Forward passes are decimation-in-frequency, so the
// spectrum ends digit-reversed across threads; the dispersion table is
// permuted on the host to each register's bin and the inverse is the exact
// adjoint walk back (no reorder pass).  Exchanges go through per-
// polarisation shared-memory planes with padded layouts (pad16 / pad256,
// conflict-free 8-byte accesses); the exchange into the last pass is a
// 16 x 16 transpose inside each half-warp's own 288-element tile (only a
// __syncwarp), and at N = 2048 the first exchange pairs positions i, i + T
// into 16-byte accesses (Geo::X01_PAIRED).  Twiddles are built by powers of
// one table load per group (DBP_TW_POWERS), and all complex arithmetic runs
// on the packed FP32 pipe (FADD2 / FMUL2 / FFMA2, dft_small.cuh).  The
// operator program arrives decoded (KernelParams::n_ops, conv_parity, ...).
// Measured-and-off compile-time options: double-buffered exchange regions
// (DBP_DOUBLE_BUFFER), TMA bulk input (DBP_TMA_LOAD), packed FIR
// (DBP_FIR_PACKED) -- DESIGN.md section 4.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <vector>

#include "dbp_common.cuh"
#include "dft_small.cuh"

namespace dbp {

// Resident threads per SM targeted by __launch_bounds__ (sets the register
// budget 65536 / target) and block positions per CTA (DBP_CTA_POSITIONS:
// CTAs hold max(1, 32 / T) blocks, so every block of N >= 512 has its own
// CTA and its own barrier domain).  Tuned on B200 with the packed-FP32
// kernel (tools/ab_small_n.sh, profiles/r1/ab_small_n.txt): N <= 256: 512
// threads/SM; N = 512: 896 (7 CTAs, 72 regs; profiles/r1/ab_896.txt);
// N >= 1024: 1024 (64 regs) since the direct-form FIR (DBP_FIR_DIRECT) and
// the separate generic-FIR instantiation (kProgGenericFir) left the fixed-tap
// kernel without spills at 64 registers: ESSFM 2048 +3.9%, 1024 +0.4%
// (profiles/r1/ab_fir_direct.txt; before: 896 / 768 / 1024 at N = 1024 /
// 2048 / 4096, still used by kProgGenericFir).  -DDBP_THREADS_PER_SM overrides.
__host__ __device__ constexpr int threads_per_sm(int logn) {
#ifdef DBP_THREADS_PER_SM
  return DBP_THREADS_PER_SM + 0 * logn;
#else
  return logn <= 8 ? 512 : (logn == 9 ? 896 : 1024);
#endif
}
// ... of the generic-FIR instantiation (runtime N_c / per-item coefficient
// sets: fir8_generic's 24-float tap windows need the pre-v8 register budgets)
__host__ __device__ constexpr int genfir_threads_per_sm(int logn) {
  return logn <= 8 ? 512 : (logn <= 10 ? 896 : (logn == 11 ? 768 : 1024));
}
// Resident threads per SM of the FFE-only kernel (launch.h selects it for
// N >= 2^DBP_FFE_KERNEL_MIN_LOGN).  Without the rotation it fits 64 registers,
// so N = 2048 runs four 256-thread CTAs per SM instead of the ESSFM kernel's
// three: FFE 87.0 -> 91.9 GS/s; 768 / 512 threads -0.1% / -9%
// (profiles/r1/ab_ffe_tps.txt).  -DDBP_FFE_THREADS_PER_SM overrides.
__host__ __device__ constexpr int ffe_threads_per_sm(int logn) {
#ifdef DBP_FFE_THREADS_PER_SM
  return DBP_FFE_THREADS_PER_SM + 0 * logn;
#else
  return logn == 11 ? 1024 : threads_per_sm(logn);
#endif
}
// Resident threads per SM of the no-FIR split-step kernel (SSFM, ESSFM N_c = 0;
// launch.h selects it for N >= 2^DBP_NOFIR_KERNEL_MIN_LOGN).  Without the FIR
// window (48 floats beside the 16 samples) it fits 64 registers without
// spills: N = 2048 runs 1024 threads per SM (SSFM-20 +2.0 / +2.6%, ESSFM
// N_c = 0 +4.3%), N = 4096 / 8192 lose the generic kernel's stack spill (+1% /
// +4.2%) (profiles/r1/ab_nofir.txt).  -DDBP_NOFIR_THREADS_PER_SM overrides.
__host__ __device__ constexpr int nofir_threads_per_sm(int logn) {
#ifdef DBP_NOFIR_THREADS_PER_SM
  return DBP_NOFIR_THREADS_PER_SM + 0 * logn;
#else
  return logn == 11 ? 1024 : threads_per_sm(logn);
#endif
}
enum KernelProg : int { kProgGeneric = 0, kProgFFE = 1, kProgNoFir = 2, kProgGenericFir = 3, kProgSym1 = 4 };
// kProgSym1: the configs[0] program -- symmetric, one nonlinear step, fixed-tap
// FIR -- compiled as a straight line (L(K^1/2) R_0 L(K^1/2), dbp.py:214-223)
// instead of the runtime operator loop: no program decode, the SFU sincos
// N_c with a compiled fixed-tap FIR (fir8_fixed); anything else, and per-item
// coefficient sets, run fir8_generic in the kProgGenericFir instantiation
__host__ __device__ constexpr bool fixed_fir_nc(int nc) {
  return nc == 1 || nc == 9 || nc == 17 || nc == 32 || nc == 33;
}
// Block input through the TMA bulk-copy engine into the exchange planes
// (Geo::TMA_LOAD): the loads bypass the L1 data path, so the kernel no
// longer depends on the L1 share of the unified array (carve-out 86%: LDG
// path -11%, TMA path -0.1%).  Off by default: at the default carve-out the
// extra barrier and shared reads cost 1.9% (ESSFM) / +0.1% (FFE); with
// double-buffered exchanges on top it is +2.9% (FFE) / -0.8% (ESSFM)
// (tools/ab.sh, variants tma / tma_db / notma).
// Block lengths compiled with the persistent group loop (the launcher uses it
// for N = 8192; smaller N only as the DBP_PERSISTENT experiment).
#ifndef DBP_PERSIST_MIN_LOGN
#define DBP_PERSIST_MIN_LOGN 13
#endif
// Split write-after-read exchange barriers (Shm kShmSplitWar, see Geo).
#ifndef DBP_SPLIT_WAR
#define DBP_SPLIT_WAR 1
#endif
#ifndef DBP_TMA_LOAD
#define DBP_TMA_LOAD 0
#endif
#ifndef DBP_FFE_TMA_LOAD
#define DBP_FFE_TMA_LOAD 1
#endif
// Output through the TMA bulk-copy engine (Geo::TMA_STORE): the kept centre is
// staged in shared memory and written by two cp.async.bulk stores, so the
// CTA retires as soon as the engine has read shared memory instead of
// draining 16 predicated STG per thread (measured cost of the STG path:
// ESSFM 4.3%, FFE 11%, profiles/r2/ab_pre.txt)
#ifndef DBP_TMA_STORE
#define DBP_TMA_STORE 1
#endif
// N = 1024 measured -1.1% with it (profiles/r2/ab_tmastore.txt): N >= 2048
#ifndef DBP_TMA_STORE_MIN_LOGN
#define DBP_TMA_STORE_MIN_LOGN 11
#endif
#ifndef DBP_EXPERIMENT_NOBAR
#define DBP_EXPERIMENT_NOBAR 0
#endif
#ifndef DBP_EXPERIMENT_NOWAR
#define DBP_EXPERIMENT_NOWAR 0
#endif
// timing experiments only (WRONG results): no global block loads (registers
// synthesised from the thread index) / no output stores / no nonlinear step
#ifndef DBP_EXPERIMENT_NOLOAD
#define DBP_EXPERIMENT_NOLOAD 0
#endif
#ifndef DBP_EXPERIMENT_NOSTORE
#define DBP_EXPERIMENT_NOSTORE 0
#endif
// timing experiment only: the nonlinear step's two CTA-wide __syncthreads
// removed (its write-after-read barrier kept: the split mbarrier protocol) -- WRONG results
#ifndef DBP_EXPERIMENT_NONLBAR
#define DBP_EXPERIMENT_NONLBAR 0
#endif
#ifndef DBP_EXPERIMENT_NONL
#define DBP_EXPERIMENT_NONL 0
#endif
#ifndef DBP_CTA_POSITIONS
#define DBP_CTA_POSITIONS 32
#endif
// Bounds checks for debug builds (compute-sanitizer is closed on the pool):
// -DDBP_DEBUG_BOUNDS=1 asserts every shared-memory and global index against
// its region; tools/build_variants.py "bounds" + tests -m gpu exercise it.
#ifndef DBP_DEBUG_BOUNDS
#define DBP_DEBUG_BOUNDS 0
#endif
#if DBP_DEBUG_BOUNDS
#include <cassert>
#define DBP_CHECK(...) assert((__VA_ARGS__))
#else
#define DBP_CHECK(...) ((void)0)
#endif

// Double-buffered exchange regions (Geo::DB, see Shm).  Off: at N = 2048 the
// 70 KB slices leave 28 KB of L1 and lose 10% (ESSFM) / 18% (FFE); at an equal
// forced carve-out they gain only 0.8% (tools/ab_carveout.sh).
#ifndef DBP_DOUBLE_BUFFER
#define DBP_DOUBLE_BUFFER 0
#endif

// half-warp tile: 16 rows of kTilePitch; 18 keeps the rows 16-byte aligned
// (8 LDS.128 / STS.128 on the row side), 17 is the minimal conflict-free pad
#ifndef DBP_TILE_PITCH
#define DBP_TILE_PITCH 18
#endif
constexpr int kTilePitch = DBP_TILE_PITCH;
constexpr int kTileLen = 16 * kTilePitch;    // = 256 + the pad256 pad of its half-warp
constexpr int kTilePad = kTileLen - 256;     // pad256: elements of pad per 256
__host__ __device__ constexpr int pad256(int i) { return i + (i >> 8) * kTilePad; }
// padded exchange plane (float2): pad256 for N >= 512, pad16 below
__host__ __device__ constexpr int plane_elems(int n) { return n + (n >= 256 ? (n >> 8) * kTilePad : n / 16); }

// DIT base tables: one float2 (the base b) per entry, or with
// DBP_DIT_TABLED four (b, b^2, b^4, b^8, each rounded from float64), so the
// butterflies use independently rounded powers instead of a squaring chain
#ifndef DBP_DIT_TABLED
#define DBP_DIT_TABLED 0
#endif
constexpr int kDitEntry = DBP_DIT_TABLED ? 4 : 1;

template <int LOGN>
struct Geo {
  static constexpr int N = 1 << LOGN;
  static constexpr int T = N / 16;                       // position-threads per block
  static constexpr int NP = (LOGN + 3) / 4;              // FFT passes
  static constexpr int LOGR0 = LOGN - 4 * (NP - 1);
  static constexpr int R0 = 1 << LOGR0;                  // first-pass radix
  static constexpr int G0 = 16 / R0;                     // first-pass groups per thread
  static constexpr int BPC = T >= DBP_CTA_POSITIONS ? 1 : DBP_CTA_POSITIONS / T;
  static constexpr int THREADS = 2 * T * BPC;
  static constexpr int MIN_CTAS = threads_per_sm(LOGN) / THREADS > 0 ? threads_per_sm(LOGN) / THREADS : 1;
  // the FFE-only instantiation (no rotation, fewer live registers)
  static constexpr int FFE_MIN_CTAS =
      ffe_threads_per_sm(LOGN) / THREADS > 0 ? ffe_threads_per_sm(LOGN) / THREADS : 1;
  static constexpr int NOFIR_MIN_CTAS =
      nofir_threads_per_sm(LOGN) / THREADS > 0 ? nofir_threads_per_sm(LOGN) / THREADS : 1;
  static constexpr int GENFIR_MIN_CTAS =
      genfir_threads_per_sm(LOGN) / THREADS > 0 ? genfir_threads_per_sm(LOGN) / THREADS : 1;
  // two exchange regions per slice while MIN_CTAS CTAs still fit the SM's
  // 228 KB (N = 128, 512 .. 2048): one CTA barrier per exchange instead of two
  static constexpr bool DB =
      DBP_DOUBLE_BUFFER && MIN_CTAS * (2 * 16 * plane_elems(N) * BPC + 1024) <= 228 * 1024;
  // split write-after-read barriers (Shm kShmSplitWar, needs every warp in one
  // slice): measured per block length against __syncthreads
  // (profiles/r1/ab_split_war.txt): N = 256 +1.7%, 4096 +3 to +5%; N = 512
  // -1.5%, 1024 -0.8%, 8192 -17% (32 warps polling one mbarrier, one CTA per
  // SM); N = 2048 -0.3% with the v7 kernel's 3 CTAs per SM but +1.3% (ESSFM) /
  // +1.7% (FFE) with v8's 4 (profiles/r1/ab_v8_opts.txt) -- on for N = 256,
  // 2048 and 4096 (DBP_SPLIT_WAR=2: every N >= 256, 0: none)
  static constexpr bool SPLIT_WAR =
      !DB && T >= 16 &&
      (DBP_SPLIT_WAR == 2 || (DBP_SPLIT_WAR == 1 && (LOGN == 8 || LOGN == 11 || LOGN == 12)));
  // one block per CTA and one group per CTA (no persistent loop): input by TMA
  // TMA block input: measured per program (profiles/r2/ab_tmaload.txt): the FFE-only
  // instantiation +1.6% (N = 2048) / +7.8% (4096); the split-step programs -0.4..-0.5%
  static constexpr bool TMA_LOAD_OK = BPC == 1 && LOGN >= 9 && LOGN <= 12;
  static constexpr bool TMA_LOAD = DBP_TMA_LOAD && TMA_LOAD_OK;
  // kept centre through shared memory and one TMA bulk store per polarisation
  // (one block per CTA, non-persistent grid): see process_group
  static constexpr bool TMA_STORE = DBP_TMA_STORE && BPC == 1 && LOGN >= DBP_TMA_STORE_MIN_LOGN && LOGN < DBP_PERSIST_MIN_LOGN;
  // first exchange with 16-byte paired accesses (see fft_fwd)
  static constexpr bool X01_PAIRED = (NP == 3 && R0 == 8);
  // log2 of the pass stride S_p = N / (L_p r_p)
  __host__ __device__ static constexpr int log_s(int p) { return LOGN - LOGR0 - 4 * p; }
  // offset (float2 units) of pass p's twiddle table.  Tables are k-paired:
  // row r holds (W^{(2r+1) c}, W^{(2r+2) c}) for every column c as one
  // 16-byte entry, so a thread fetches two twiddles per load.  Pass 0: R0/2
  // rows x N/R0 columns; pass q >= 1: 8 rows x S_q columns.
  __host__ __device__ static constexpr int tw_offset(int p) {
    int off = 0;
    for (int q = 0; q < p; ++q) off += q == 0 ? (R0 / 2) * (N / R0) * 2 : 8 * (1 << log_s(q)) * 2;
    return off;
  }
  // Decimation-in-time base tables (one float2 per entry) behind the k-paired
  // tables (make_twiddles):
  //  forward pass p >= 1: W_{R0 16^p}^{K}, R0 16^(p-1) entries, indexed by the
  //    thread's sub-problem K = t >> log_s(p) -- except the last pass (NP >= 2),
  //    indexed by t (K = (t >> 4) + (N / 256)(t & 15) after the tile transpose
  //    for NP >= 3, K = t for NP == 2);
  //  inverse pass 0: W_N^{-g}, g = t + T q < N / R0; inverse middle pass p:
  //    W_{16 S_p}^{-ns}, ns = t mod S_p < S_p.
  __host__ __device__ static constexpr int tw_legacy_size() { return NP > 1 ? tw_offset(NP - 1) : 1; }
  __host__ __device__ static constexpr int dit_fwd_size(int p) {
    int s = R0;
    for (int q = 1; q < p; ++q) s *= 16;
    return s;
  }
  __host__ __device__ static constexpr int dit_fwd_offset(int p) {
    int off = tw_legacy_size();
    for (int q = 1; q < p; ++q) off += kDitEntry * dit_fwd_size(q);
    return off;
  }
  __host__ __device__ static constexpr int dit_inv_size(int p) { return p == 0 ? N / R0 : (1 << log_s(p)); }
  __host__ __device__ static constexpr int dit_inv_offset(int p) {
    int off = dit_fwd_offset(NP);
    for (int q = 0; q < p; ++q) off += kDitEntry * dit_inv_size(q);
    return off;
  }
};

// Twiddle tables, float64 -> float32, k-paired (see Geo::tw_offset):
// pass 0 W_N^{g k} (g < N/R0, k < R0), pass p >= 1 W_{16 S_p}^{ns k}
// (ns < S_p, k < 16); entry [r][c] = (W^{(2r+1) c}, W^{(2r+2) c}), the
// second half zero when 2r+2 reaches the radix.
//
// Unit complex numbers are rounded to the float pair (within +-1 ulp per
// component of the nearest) whose squared magnitude is closest to 1, the
// phase error held to <= 1.5 ulp: a forward twiddle and its conjugate in the
// inverse transform compose to |w|^2, so the magnitude rounding -- not the
// phase -- is what a long chain of transform pairs (the 10^3 - 10^4 split
// steps of a link simulation) accumulates systematically.
inline float2 unit_float2(double ang) {
  const double c = std::cos(ang), s = std::sin(ang);
  const float c0 = (float)c, s0 = (float)s;
  float2 best = make_float2(c0, s0);
  double best_mag = std::fabs((double)c0 * c0 + (double)s0 * s0 - 1.0);
  const double phase_tol = 1.5 * 5.9604644775390625e-8;
  for (int dc = -1; dc <= 1; ++dc)
    for (int ds = -1; ds <= 1; ++ds) {
      float cc = c0, ss = s0;
      if (dc) cc = std::nextafter(cc, dc > 0 ? 2.f : -2.f);
      if (ds) ss = std::nextafter(ss, ds > 0 ? 2.f : -2.f);
      const double mag = std::fabs((double)cc * cc + (double)ss * ss - 1.0);
      const double dphi = std::fabs(std::atan2(ss * c - cc * s, cc * c + ss * s));
      if (dphi <= phase_tol && mag < best_mag) {
        best_mag = mag;
        best = make_float2(cc, ss);
      }
    }
  return best;
}

inline std::vector<float2> make_twiddles(int logn) {
  const int np = (logn + 3) / 4;
  const int logr0 = logn - 4 * (np - 1);
  const long long n = 1LL << logn, r0 = 1LL << logr0;
  std::vector<float2> tw;
  auto w = [](long long m, long long period) {
    return unit_float2(-2.0 * M_PI * (double)(m % period) / (double)period);
  };
  auto table = [&](long long radix, long long cols, long long period) {
    for (long long r = 0; r < radix / 2; ++r)
      for (long long c = 0; c < cols; ++c) {
        const long long k0 = 2 * r + 1, k1 = 2 * r + 2;
        tw.push_back(w(c * k0, period));
        tw.push_back(k1 < radix ? w(c * k1, period) : make_float2(0.f, 0.f));
      }
  };
  if (np > 1) {
    table(r0, n / r0, n);
    for (int p = 1; p < np - 1; ++p) {
      const long long s = n >> (logr0 + 4 * p);
      table(16, s, 16 * s);
    }
  }
  if (tw.empty()) tw.push_back(make_float2(1.f, 0.f));
  // decimation-in-time bases (Geo::dit_fwd_offset / dit_inv_offset): per
  // index b = W^k (kDitEntry == 1) or (b, b^2, b^4, b^8) (kDitEntry == 4)
  auto entry = [&](long long k, long long period, double sign) {
    for (int e = 0; e < kDitEntry; ++e) {
      const long long kk = (k << e) % period;   // b^(2^e)
      tw.push_back(unit_float2(sign * 2.0 * M_PI * (double)kk / (double)period));
    }
  };
  if (np > 1) {
    const long long tt = n / 16;
    for (int p = 1; p < np; ++p) {
      const long long period = r0 << (4 * p), size = period / 16;
      if (p == np - 1) {
        for (long long t = 0; t < tt; ++t) {
          const long long k = np >= 3 ? (t >> 4) + (n / 256) * (t & 15) : t;
          entry(k, period, -1.0);
        }
      } else {
        for (long long k = 0; k < size; ++k) entry(k, period, -1.0);
      }
    }
    for (int p = 0; p < np - 1; ++p) {
      const long long period = p == 0 ? n : n >> (logr0 + 4 * p - 4), size = p == 0 ? n / r0 : period / 16;
      for (long long k = 0; k < size; ++k) entry(k, period, +1.0);
    }
  }
  return tw;
}

// Dispersion-table entry index of (thread t, register e): tables are
// e-paired like the twiddles, [e/2][t] -> (H_e, H_{e+1}) per 16 bytes.
__host__ __device__ constexpr int tab_index(int logn, int t, int e) {
  return (e >> 1) * 2 * ((1 << logn) / 16) + 2 * t + (e & 1);
}

__host__ __device__ inline int fir_phys(int u) { return u + ((u >> 4) << 2); }  // pad 4 per 16 floats
__host__ __device__ inline int cs_phys(int j) { return j + ((j >> 4) << 1); }   // pad 2 per 16 float2

// shared floats per block slice.  Single region: max(exchange planes,
// FIR intensity + (cos, sin) buffers).  Double-buffered: two regions, each
// max(planes, intensity, (cos, sin)); the kernel's region 1 starts at
// slice_floats / 2.

inline int fir_floats(int n, int pw) { return fir_phys(n + 2 * pw) + 4 + 2 * (cs_phys(n) + 2); }

// polarisation-split pair (PS): one polarisation's planes, the intensity
// exchange buffer behind them (N floats), or the FIR buffers publishing F
inline int ps_smem_floats(int n, int pw, bool fir, bool xchg) {
  int total = 2 * plane_elems(n) + (xchg ? n : 0);
  const int f = fir ? fir_phys(n + 2 * pw) + 4 + fir_phys(n) + 4 : 0;
  if (f > total) total = f;
  return (total + 3) & ~3;
}

inline int slice_floats(int n, int pw, bool double_buffer) {
  const int planes = 4 * plane_elems(n);
  if (double_buffer) {
    int r = planes;
    if (fir_phys(n + 2 * pw) + 4 > r) r = fir_phys(n + 2 * pw) + 4;
    if (2 * (cs_phys(n) + 2) > r) r = 2 * (cs_phys(n) + 2);
    return 2 * ((r + 3) & ~3);
  }
  const int fir = fir_floats(n, pw);
  const int v = planes > fir ? planes : fir;
  return (v + 3) & ~3;
}

// Exchange layouts.
//  * NP == 2 (N <= 256): the one exchange feeds the last pass, whose lanes
//    gather 16 consecutive elements (128-byte lane stride): one pad element
//    per 16 ("pad16") makes it conflict free.
//  * NP >= 3: the exchange INTO pass NP-2 uses one pad of 32 elements per
//    256 ("pad256"), so half-warp h gathers exactly [288 h, 288 h + 256); the
//    exchange into the last pass then stays inside half-warp h's own
//    288-element tile (16 rows of pitch 18, see fft_fwd) and needs only
//    __syncwarp.
//  * all other exchanges: plain.
// Every form is linear in the register index, so accesses are base + immediates.
__host__ __device__ constexpr int pad16(int i) { return i + (i >> 4); }

template <int LOGN, int P>
__device__ __forceinline__ int xchg_index(int i) {
  constexpr int NP = Geo<LOGN>::NP;
  if constexpr (NP == 2 && P == 0) return pad16(i);
  else if constexpr (NP >= 3 && P + 1 == NP - 2) return pad256(i);
  else return i;
}

// plane index of position t + T m (the strided side of exchange P)
template <int LOGN, int P>
__device__ __forceinline__ int side_index(int t, int m) {
  constexpr int T = Geo<LOGN>::T, NP = Geo<LOGN>::NP;
  if constexpr (NP == 2 && P == 0) {
    if constexpr (T % 16 == 0) return pad16(t) + m * (T + T / 16);
    else return pad16(t + T * m);
  } else if constexpr (NP >= 3 && P + 1 == NP - 2) {
    // t < T: for T <= 256, (t + T m) >> 8 == (T m) >> 8 (no carry); else linear
    if constexpr (T <= 256) return t + T * m + ((T * m) >> 8) * kTilePad;
    else return pad256(t) + m * (T + (T >> 8) * kTilePad);
  } else {
    return t + T * m;
  }
}

// Bin index held by register e of thread t after the last forward pass
// (host-side permutation of the dispersion tables, read as tab[t + T e]).
__host__ __device__ constexpr int last_pass_bin(int logn, int t, int e) {
  const int n = 1 << logn, tt = n / 16, np = (logn + 3) / 4;
  return np >= 3 ? (t >> 4) + (n / 256) * (t & 15) + (n / 16) * e : t + tt * e;
}

__device__ __forceinline__ void st_pair(float2* p, float2 a, float2 b) {
  *reinterpret_cast<float4*>(p) = make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void ld_pair(const float2* p, float2& a, float2& b) {
  const float4 q = *reinterpret_cast<const float4*>(p);
  a = make_float2(q.x, q.y);
  b = make_float2(q.z, q.w);
}

// TMA bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)), "r"(parity)
      : "memory");
}
// shared -> global bulk copy (bulk_group completion) and its read-side wait
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_store_commit_and_wait_read() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
// Polarisation-split pairs (PS, N = 8192): the two CTAs of a 2-CTA cluster
// each hold one polarisation of the block, so two independent half-size CTAs
// share each SM where one 1024-thread CTA did.  The only coupling is the
// nonlinear step's total intensity |x|^2 + |y|^2: each CTA writes its 16 T
// values of |v|^2 into the partner's shared memory with st.async (completion
// counted on the partner's ``full`` mbarrier) and, once it no longer needs
// the values it received, arrives on the partner's ``free`` mbarrier.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t peer_smem_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_async_v4(uint32_t raddr, float4 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   raddr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rbar)
               : "memory");
}
// The write-after-read handshake is relaxed: the release / acquire forms
// cost a GPU-scope MEMBAR and an L1 invalidation per step.  Ordering instead
// comes from data: every lane makes the arrive depend on the last value it
// read from the buffer (so its loads have completed), the warp converges, and
// the partner issues its st.async only after observing the phase.
__device__ __forceinline__ uint32_t zero_after(float x) {
  uint32_t z;
  asm volatile("and.b32 %0, %1, 0;" : "=r"(z) : "r"(__float_as_uint(x)));
  return z;
}
__device__ __forceinline__ void mbar_arrive_peer_relaxed(uint32_t rbar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_wait_relaxed_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(smem_addr(bar)), "r"(parity)
      : "memory");
}

struct PolXchg {
  float* xbuf;          // local: the partner's |v|^2 at this CTA's positions, [t][16] swizzled
  uint32_t peer_xbuf;   // the partner's xbuf (shared::cluster address)
  uint64_t* full;       // local: completes when the partner's 16 T values have landed
  uint32_t peer_full;
  uint64_t* free_;      // local: the partner has consumed what this CTA wrote into its xbuf
  uint32_t peer_free;
  uint32_t step;        // nonlinear steps exchanged so far
};
// float offset of chunk c (4 floats) of thread t's 16 in the exchange buffer:
// 16-byte accesses of a quarter warp land in eight distinct bank groups
__device__ __forceinline__ int xbuf_slot(int t, int c) { return 16 * t + 4 * (c ^ ((t >> 1) & 3)); }

// Shared memory of one block slice: exchange planes (x, y) and the FIR
// buffers, aliased.  Single region: every exchange is "barrier; write;
// barrier; read".  Double-buffered (DB): two regions used alternately and
// the choice is compile time -- an FFT's forward exchange P writes region
// (P + 1) & 1, its inverse exchange P region P & 1, the half-warp tile
// exchanges stay in region (NP - 2) & 1 (the one their half-warp just read),
// and the rotation writes intensities to region 1 and (cos, sin) factors to
// region 0 -- so every op starts and ends on the same parity and each write
// phase goes to the region NOT read in the phase before: "write; barrier;
// read" (the barrier of the previous phase already ordered the last reads of
// this region).  ESSFM block at N = 2048: 6 CTA barriers instead of 11.
//
// Split write-after-read barriers (MODE kShmSplitWar, single region): the
// barrier before an exchange's writes only has to know that every warp of
// the slice finished its reads of the previous exchange.  Each warp arrives
// on the slice's mbarrier right after its last read of a phase
// (``reads_done``) and the next write phase waits on it (``before_write``),
// so the wait overlaps the pass computed in between instead of a
// __syncthreads.  Arrive / wait alternate strictly: one initial arrive at
// kernel start, then per CTA-wide write phase one wait and, after the last
// read before the next such phase, one arrive.
enum ShmMode : int { kShmSync = 0, kShmDouble = 1, kShmSplitWar = 2 };

template <int LOGN, int MODE = kShmSync>
struct Shm {
  static constexpr bool DB = MODE == kShmDouble;
  static constexpr bool SPLIT = MODE == kShmSplitWar;
  float* base;    // region 0
  float* base1;   // region 1 (== base without double buffering)
  int pol;
  uint64_t* war;  // SPLIT: the slice's write-after-read mbarrier
  uint32_t war_phase;
  __device__ __forceinline__ void init(float* slice_base, int slice_floats, int polarisation) {
    base = slice_base;
    base1 = DB ? slice_base + slice_floats / 2 : slice_base;
    pol = polarisation;
    war = nullptr;
    war_phase = 0;
  }
  __device__ __forceinline__ static int plane_len() { return plane_elems(Geo<LOGN>::N); }
  template <int R>
  __device__ __forceinline__ float* region() const {
    return (R & 1) ? base1 : base;
  }
  template <int R>
  __device__ __forceinline__ float2* plane() const {
    return reinterpret_cast<float2*>(region<R>()) + pol * plane_len();
  }
#if DBP_EXPERIMENT_NOBAR   // timing experiment only: exchange barriers removed (WRONG results)
  __device__ __forceinline__ void before_write() const { __syncwarp(); }
  __device__ __forceinline__ void after_write() const { __syncwarp(); }
  __device__ __forceinline__ void reads_done() const {}
#elif DBP_EXPERIMENT_NOWAR   // timing experiment only: write-after-read barriers removed (racy)
  __device__ __forceinline__ void before_write() const {}
  __device__ __forceinline__ void after_write() const { __syncthreads(); }
  __device__ __forceinline__ void reads_done() const {}
#else
  __device__ __forceinline__ void before_write() {
    if constexpr (SPLIT) {
      mbar_wait(war, war_phase);
      war_phase ^= 1u;
    } else if constexpr (!DB) {
      __syncthreads();
    }
  }
  __device__ __forceinline__ void after_write() const { __syncthreads(); }
  __device__ __forceinline__ void reads_done() const {
    if constexpr (SPLIT) {
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(war);
    }
  }
#endif
};

// u[k] *= W (or conj W) for k = 1 .. R-1 from a k-paired table column
// (``col`` points at row 0 of this thread's column, rows ``row_stride``
// float2 apart): two twiddles per 16-byte load.
template <int R, bool CONJ>
__device__ __forceinline__ void twiddle_paired(float2* u, const float2* col, int row_stride) {
#pragma unroll
  for (int k = 1; k < R; k += 2) {
    float2 w0, w1;
    ldg_table_pair(col + ((k - 1) >> 1) * row_stride, w0, w1);
    u[k] = CONJ ? c_mulc(u[k], w0) : c_mul(u[k], w0);
    if (k + 1 < R) u[k + 1] = CONJ ? c_mulc(u[k + 1], w1) : c_mul(u[k + 1], w1);
  }
}

// Same twiddles from ONE 8-byte load of W (row 0 first half) and complex
// products of depth <= 4 (W^2, W^4, W^8 by squaring): trades L1 table
// traffic for FP32 work.  Selected per pass by DBP_TW_POWERS (bit 0: first
// pass, bit 1: later passes).  Default 3 since the packed-FP32 complex
// arithmetic (dft_small.cuh) made the L1 data pipe the co-limiter: +1.3%
// (ESSFM) / +2.8% (FFE) over 1 at N = 2048, worst golden-case per-block
// error 1.2e-6 -> 2.2e-6 (tolerance 1e-5).  The link simulator uses table
// loads only (TWP = 0).
__device__ __forceinline__ float2 c_sqr(float2 a) { return c_mul(a, a); }

template <int R, bool CONJ>
__device__ __forceinline__ void twiddle_powers(float2* u, const float2* col) {
  float2 p[16];
  p[1] = ldg_table(col);
  if constexpr (R > 2) p[2] = c_sqr(p[1]);
  if constexpr (R > 3) p[3] = c_mul(p[2], p[1]);
  if constexpr (R > 4) {
    p[4] = c_sqr(p[2]);
    p[5] = c_mul(p[4], p[1]);
    p[6] = c_sqr(p[3]);
    p[7] = c_mul(p[4], p[3]);
  }
  if constexpr (R > 8) {
    p[8] = c_sqr(p[4]);
#pragma unroll
    for (int k = 9; k < 16; ++k) p[k] = c_mul(p[8], p[k - 8]);
  }
#pragma unroll
  for (int k = 1; k < R; ++k) u[k] = CONJ ? c_mulc(u[k], p[k]) : c_mul(u[k], p[k]);
}

#ifndef DBP_TW_POWERS
#define DBP_TW_POWERS 3
#endif
// TWP value of the decimation-in-time fused-twiddle FFT (see dit_base)
constexpr int kTwDit = 4;
// Programs with at most this many nonlinear steps run the fused-twiddle FFT;
// longer programs keep the exact-adjoint FFT (DBP_TW_POWERS), whose forward
// and inverse twiddles are conjugates of the same rounded values, so phase
// errors cancel within each transform pair instead of accumulating coherently
// over the steps (SSFM-20 at +5.6 dBm: 1.3e-5 per-block rel-L2 with the fused
// FFT, tolerance 1e-5).  -DDBP_DIT_MAX_STEPS=0 disables the fused FFT.
#ifndef DBP_DIT_MAX_STEPS
#define DBP_DIT_MAX_STEPS 2
#endif

template <int R, bool CONJ, bool FIRST, int TWP>
__device__ __forceinline__ void twiddle(float2* u, const float2* col, int row_stride) {
  if constexpr ((TWP & (FIRST ? 1 : 2)) != 0) twiddle_powers<R, CONJ>(u, col);
  else twiddle_paired<R, CONJ>(u, col, row_stride);
}

// v[e] *= table entry of (t, e), e-paired dispersion table
template <int LOGN>
__device__ __forceinline__ void apply_table(float2 (&v)[16], const float2* __restrict__ tab, int t) {
#pragma unroll
  for (int e = 0; e < 16; e += 2) {
    float2 h0, h1;
    ldg_table_pair(tab + tab_index(LOGN, t, e), h0, h1);
    v[e] = c_mul(v[e], h0);
    v[e + 1] = c_mul(v[e + 1], h1);
  }
}

// v[e] *= (hi + lo) of a double-float table pair (same layout as apply_table):
// the table's own rounding drops to ~2^-48, for operators applied 10^3+ times
template <int LOGN>
__device__ __forceinline__ void apply_table_df(float2 (&v)[16], const float2* __restrict__ hi,
                                               const float2* __restrict__ lo, int t) {
#pragma unroll
  for (int e = 0; e < 16; e += 2) {
    float2 h0, h1, l0, l1;
    ldg_table_pair(hi + tab_index(LOGN, t, e), h0, h1);
    ldg_table_pair(lo + tab_index(LOGN, t, e), l0, l1);
    const float2 a0 = c_mul(v[e], l0), a1 = c_mul(v[e + 1], l1);
    v[e] = make_float2(fmaf(v[e].x, h0.x, fmaf(-v[e].y, h0.y, a0.x)), fmaf(v[e].x, h0.y, fmaf(v[e].y, h0.x, a0.y)));
    v[e + 1] = make_float2(fmaf(v[e + 1].x, h1.x, fmaf(-v[e + 1].y, h1.y, a1.x)),
                           fmaf(v[e + 1].x, h1.y, fmaf(v[e + 1].y, h1.x, a1.y)));
  }
}

// Decimation-in-time twiddles (TWP != 0, the DBP kernel): the forward passes
// p >= 1 take their twiddles at the input as powers of one base per thread
// (W_{R0 16^p}^{K}, K the thread's accumulated sub-problem index) and the
// inverse passes keep theirs at the input too, so every twiddle multiply
// fuses into a DFT butterfly (dft_tw, dft_small.cuh): 74 + 30 + 28 -> 112
// instructions per twiddled radix-16 pass, and the radix-R0 forward pass
// carries none (v9).  TWP == 0 (the link simulator) keeps the table-twiddle
// decimation-in-frequency forward, whose magnitude error does not compound.
#if DBP_DIT_TABLED
using DitBase = TwPow;
__device__ __forceinline__ DitBase dit_base(const float2* __restrict__ tw, int off, int idx) {
  DitBase r;
  ldg_table_pair(tw + off + 4 * idx, r.b, r.b2);
  ldg_table_pair(tw + off + 4 * idx + 2, r.b4, r.b8);
  return r;
}
__device__ __forceinline__ DitBase dit_zero() { return DitBase{}; }
#else
using DitBase = float2;
__device__ __forceinline__ DitBase dit_base(const float2* __restrict__ tw, int off, int idx) {
  return ldg_table(tw + off + idx);
}
__device__ __forceinline__ DitBase dit_zero() { return make_float2(0.f, 0.f); }
#endif

// ---------------------------------------------------------------------------
// Block FFT on one polarisation: fft_fwd walks the decimation-in-frequency
// passes 0 .. NP-1 (register m of thread t holds block position t + T m on
// entry; on exit register e holds bin last_pass_bin(t, e)); fft_inv is the
// exact adjoint walk back (bins in that distribution -> positions t + T m,
// unscaled).  conv_block = fft_fwd, x table, fft_inv.
// ---------------------------------------------------------------------------
// TWP: which passes build twiddles by powers (DBP_TW_POWERS bits); the link
// simulator passes 0 (table loads only: powers compound the magnitude error)
// pb (TWP == kTwDit, P >= 1): this pass's input-twiddle base, loaded by the
// caller before the exchange in front of the pass, so the load latency hides
// behind the exchange's barrier instead of stalling the pass
template <int LOGN, int P, int TWP = kTwDit, int MODE = kShmSync, bool CALLER_WAR = false>
__device__ __forceinline__ void fft_fwd(float2 (&v)[16], Shm<LOGN, MODE>& sh, const float2* __restrict__ tw,
                                        int t, DitBase pb = dit_zero()) {
  using G = Geo<LOGN>;
  constexpr int N = G::N, T = G::T, NP = G::NP;
  if constexpr (NP == 1) {
    dft<16, false>(v);  // N == 16: a single radix-16 pass, bins k = e
  } else if constexpr (P == 0) {
    // radix R0 over G0 groups: group q = registers q + G0 e, g = t + T q
    constexpr int R0 = G::R0, G0 = G::G0, S0 = N / R0;
#pragma unroll
    for (int q = 0; q < G0; ++q) {
      float2 u[R0];
#pragma unroll
      for (int e = 0; e < R0; ++e) u[e] = v[q + G0 * e];
      dft<R0, false>(u);
      if constexpr (TWP != kTwDit) twiddle<R0, false, true, TWP>(u, tw + 2 * (t + T * q), 2 * S0);
#pragma unroll
      for (int e = 0; e < R0; ++e) v[q + G0 * e] = u[e];
    }
    // exchange into the pass-1 layout
    constexpr int LS1 = G::log_s(1);
    DitBase nb = dit_zero();
    if constexpr (TWP == kTwDit) nb = dit_base(tw, G::dit_fwd_offset(1), t >> LS1);
    // CALLER_WAR: the caller omits this exchange's write-after-read barrier
    // (the FFE kernel's single convolution in a CTA that has not read shared
    // memory yet)
    if constexpr (!CALLER_WAR) sh.before_write();
    if constexpr (G::X01_PAIRED) {
      // R0 = 8, N = 2048: positions i and i + T pair up on both sides of this
      // exchange (registers (m, m+1) when writing, gathers (e, e+8) when
      // reading), so the plane stores them adjacently -- layout
      // pad256(256 (i >> 8) + 2 (i & 127) + ((i >> 7) & 1)) -- and every
      // access is a conflict-free 16-byte vector: half the LDS/STS.
      float2* plane = sh.template plane<1>() + 2 * t;
      DBP_CHECK(2 * t + kTileLen * 7 + 1 < sh.plane_len());
#pragma unroll
      for (int m = 0; m < 16; m += 2) st_pair(plane + kTileLen * (m >> 1), v[m], v[m + 1]);
    } else {
      float2* plane = sh.template plane<1>();
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        DBP_CHECK(side_index<LOGN, 0>(t, m) < sh.plane_len());
        plane[side_index<LOGN, 0>(t, m)] = v[m];
      }
    }
    sh.after_write();
    if constexpr (G::X01_PAIRED) {
      const float2* plane = sh.template plane<1>() + kTileLen * (t >> 4) + 2 * (t & 15);
#pragma unroll
      for (int e = 0; e < 8; ++e) ld_pair(plane + 32 * e, v[e], v[e + 8]);
    } else {
      const float2* plane = sh.template plane<1>();
      const int base = ((t >> LS1) << (LS1 + 4)) + (t & ((1 << LS1) - 1));
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        DBP_CHECK(xchg_index<LOGN, 0>(base + (e << LS1)) < sh.plane_len());
        v[e] = plane[xchg_index<LOGN, 0>(base + (e << LS1))];
      }
    }
    if constexpr (NP != 3) sh.reads_done();   // NP == 3: the half-warp tile follows
    fft_fwd<LOGN, 1, TWP>(v, sh, tw, t, nb);
  } else if constexpr (NP >= 3 && P == NP - 2) {
    // second-to-last pass (S = 16) + last pass, joined by a half-warp-local
    // 16 x 16 transpose: half-warp h = t >> 4 owns sub-problem h, lane
    // ns = t & 15 holds its register k; the last pass's group (h, k) goes to
    // lane k of the same half-warp.  The tile [288 h, 288 h + 288) is the
    // region this half-warp alone read in the previous (pad256) exchange;
    // rows of pitch 18 keep the row side 16-byte aligned (8 LDS.128) and
    // both sides conflict free.
    if constexpr (TWP != kTwDit) {
      dft<16, false>(v);
      twiddle<16, false, false, TWP>(v, tw + G::tw_offset(P) + 2 * (t & 15), 2 * 16);
    } else {
      dft_tw<16, false>(v, pb);
    }
    DitBase nb = dit_zero();
    if constexpr (TWP == kTwDit) nb = dit_base(tw, G::dit_fwd_offset(NP - 1), t);
    float2* tile = sh.template plane<(NP - 2) & 1>() + kTileLen * (t >> 4);
    const int l = t & 15;
    DBP_CHECK(kTileLen * (t >> 4) + kTileLen <= sh.plane_len());
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[l + kTilePitch * k] = v[k];
    __syncwarp();
    if constexpr (kTilePitch % 2 == 0) {
#pragma unroll
      for (int e = 0; e < 16; e += 2) ld_pair(tile + kTilePitch * l + e, v[e], v[e + 1]);
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = tile[kTilePitch * l + e];
    }
    if constexpr (TWP != kTwDit) dft<16, false>(v);  // last pass: group (h, l)
    else dft_tw<16, false>(v, nb);
  } else if constexpr (P < NP - 1) {
    // middle radix-16 pass: group g = t, ns = t mod S_P
    constexpr int LS = G::log_s(P), S = 1 << LS, LS1 = G::log_s(P + 1);
    if constexpr (TWP != kTwDit) {
      dft<16, false>(v);
      twiddle<16, false, false, TWP>(v, tw + G::tw_offset(P) + 2 * (t & (S - 1)), 2 * S);
    } else {
      dft_tw<16, false>(v, pb);
    }
    DitBase nb = dit_zero();
    if constexpr (TWP == kTwDit) nb = dit_base(tw, G::dit_fwd_offset(P + 1), t >> LS1);
    sh.before_write();
    {
      float2* plane = sh.template plane<(P + 1) & 1>();
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        DBP_CHECK(side_index<LOGN, P>(t, m) < sh.plane_len());
        plane[side_index<LOGN, P>(t, m)] = v[m];
      }
    }
    sh.after_write();
    {
      const float2* plane = sh.template plane<(P + 1) & 1>();
      const int base = ((t >> LS1) << (LS1 + 4)) + (t & ((1 << LS1) - 1));
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        DBP_CHECK(xchg_index<LOGN, P>(base + (e << LS1)) < sh.plane_len());
        v[e] = plane[xchg_index<LOGN, P>(base + (e << LS1))];
      }
    }
    if constexpr (P + 1 != NP - 2) sh.reads_done();
    fft_fwd<LOGN, P + 1, TWP>(v, sh, tw, t, nb);
  } else {
    // last pass (NP == 2): S = 1, group g = t, bins t + T e
    if constexpr (TWP != kTwDit) dft<16, false>(v);
    else dft_tw<16, false>(v, pb);
  }
}

template <int LOGN, int P, int TWP = kTwDit, int MODE = kShmSync>
__device__ __forceinline__ void fft_inv(float2 (&v)[16], Shm<LOGN, MODE>& sh, const float2* __restrict__ tw,
                                        int t) {
  using G = Geo<LOGN>;
  constexpr int N = G::N, T = G::T, NP = G::NP;
  if constexpr (NP == 1) {
    dft<16, true>(v);
  } else if constexpr (P == 0) {
    constexpr int R0 = G::R0, G0 = G::G0, S0 = N / R0;
    constexpr int LS1 = G::log_s(1);
    fft_inv<LOGN, 1, TWP>(v, sh, tw, t);
    // this pass's input-twiddle bases, loaded ahead of the exchange (G0 <= 2)
    constexpr bool kPre = TWP == kTwDit && G0 <= 2;
    DitBase pre[kPre ? G0 : 1];
    if constexpr (kPre) {
#pragma unroll
      for (int q = 0; q < G0; ++q) pre[q] = dit_base(tw, G::dit_inv_offset(0), t + T * q);
    }
    sh.before_write();
    if constexpr (G::X01_PAIRED) {
      float2* plane = sh.template plane<0>() + kTileLen * (t >> 4) + 2 * (t & 15);
#pragma unroll
      for (int e = 0; e < 8; ++e) st_pair(plane + 32 * e, v[e], v[e + 8]);
    } else {
      float2* plane = sh.template plane<0>();
      const int base = ((t >> LS1) << (LS1 + 4)) + (t & ((1 << LS1) - 1));
#pragma unroll
      for (int e = 0; e < 16; ++e) plane[xchg_index<LOGN, 0>(base + (e << LS1))] = v[e];
    }
    sh.after_write();
    if constexpr (G::X01_PAIRED) {
      const float2* plane = sh.template plane<0>() + 2 * t;
#pragma unroll
      for (int m = 0; m < 16; m += 2) ld_pair(plane + kTileLen * (m >> 1), v[m], v[m + 1]);
    } else {
      const float2* plane = sh.template plane<0>();
#pragma unroll
      for (int m = 0; m < 16; ++m) v[m] = plane[side_index<LOGN, 0>(t, m)];
    }
    sh.reads_done();
#pragma unroll
    for (int q = 0; q < G0; ++q) {
      float2 u[R0];
#pragma unroll
      for (int e = 0; e < R0; ++e) u[e] = v[q + G0 * e];
      if constexpr (TWP != kTwDit) {
        twiddle<R0, true, true, TWP>(u, tw + 2 * (t + T * q), 2 * S0);
        dft<R0, true>(u);
      } else if constexpr (kPre) {
        dft_tw<R0, true>(u, pre[q]);
      } else {
        dft_tw<R0, true>(u, dit_base(tw, G::dit_inv_offset(0), t + T * q));
      }
#pragma unroll
      for (int e = 0; e < R0; ++e) v[q + G0 * e] = u[e];
    }
  } else if constexpr (NP >= 3 && P == NP - 2) {
    dft<16, true>(v);  // last pass
    DitBase pb = dit_zero();
    if constexpr (TWP == kTwDit) pb = dit_base(tw, G::dit_inv_offset(P), t & 15);
    float2* tile = sh.template plane<(NP - 2) & 1>() + kTileLen * (t >> 4);
    const int l = t & 15;
    __syncwarp();
    if constexpr (kTilePitch % 2 == 0) {
#pragma unroll
      for (int e = 0; e < 16; e += 2) st_pair(tile + kTilePitch * l + e, v[e], v[e + 1]);
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) tile[kTilePitch * l + e] = v[e];
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = tile[l + kTilePitch * k];
    sh.reads_done();
    if constexpr (TWP != kTwDit) {
      twiddle<16, true, false, TWP>(v, tw + G::tw_offset(P) + 2 * (t & 15), 2 * 16);
      dft<16, true>(v);
    } else {
      dft_tw<16, true>(v, pb);
    }
  } else if constexpr (P < NP - 1) {
    constexpr int LS = G::log_s(P), S = 1 << LS, LS1 = G::log_s(P + 1);
    fft_inv<LOGN, P + 1, TWP>(v, sh, tw, t);
    DitBase pb = dit_zero();
    if constexpr (TWP == kTwDit) pb = dit_base(tw, G::dit_inv_offset(P), t & (S - 1));
    sh.before_write();
    {
      float2* plane = sh.template plane<P & 1>();
      const int base = ((t >> LS1) << (LS1 + 4)) + (t & ((1 << LS1) - 1));
#pragma unroll
      for (int e = 0; e < 16; ++e) plane[xchg_index<LOGN, P>(base + (e << LS1))] = v[e];
    }
    sh.after_write();
    {
      const float2* plane = sh.template plane<P & 1>();
#pragma unroll
      for (int m = 0; m < 16; ++m) v[m] = plane[side_index<LOGN, P>(t, m)];
    }
    sh.reads_done();
    if constexpr (TWP != kTwDit) {
      twiddle<16, true, false, TWP>(v, tw + G::tw_offset(P) + 2 * (t & (S - 1)), 2 * S);
      dft<16, true>(v);
    } else {
      dft_tw<16, true>(v, pb);
    }
  } else {
    dft<16, true>(v);  // last pass
  }
}

// FFT -> x table (bins in register order, 1/N folded in) -> IFFT
template <int LOGN, int MODE, bool CALLER_WAR = false, int TWP = kTwDit>
__device__ __forceinline__ void conv_block(float2 (&v)[16], Shm<LOGN, MODE>& sh, const float2* __restrict__ tab,
                                           const float2* __restrict__ tw, int t) {
  fft_fwd<LOGN, 0, TWP, MODE, CALLER_WAR>(v, sh, tw, t);
  apply_table<LOGN>(v, tab, Geo<LOGN>::NP == 1 ? 0 : t);
  // value barrier: the inverse recomputes its indices instead of holding the
  // forward ones (and reloading twiddles) across the last pass
  fft_inv<LOGN, 0, TWP>(v, sh, tw, opaque(t));
}

// ---------------------------------------------------------------------------
// Nonlinear rotation with the in-block cyclic intensity FIR.
// ---------------------------------------------------------------------------

// (cos, sin) * g of theta = a * F with explicit 2 pi range reduction
// (cos, sin) * g of theta = a * F.  ``precise``: quadrant reduction
// r = th - k pi/2 (two-constant Cody-Waite) and minimax polynomials on
// [-pi/4, pi/4], about 1 ulp and unbiased; otherwise 2 pi reduction and the
// SFU's __sincosf, whose smooth argument-correlated absolute error (up to
// 2^-21.4) accumulates coherently over many SSFM steps -- the host picks the
// precise form for programs with >= 3 nonlinear steps.
template <bool PRECISE, bool GAIN = true>
__device__ __forceinline__ float2 rot_factor(float a, float g, float f) {
  const float th = a * f;
  float s, c;
  if constexpr (PRECISE) {
    const float k = rintf(th * 0.636619772367581343f);
    float r = fmaf(k, -1.57079637050628662f, th);
    r = fmaf(k, 4.37113900018624283e-8f, r);
    const float z = r * r;
    float sp = fmaf(z, -1.9515295891e-4f, 8.3321608736e-3f);
    sp = fmaf(z, sp, -1.6666654611e-1f);
    const float sn = fmaf(r * z, sp, r);
    float cp = fmaf(z, 2.443315711809948e-5f, -1.388731625493765e-3f);
    cp = fmaf(z, cp, 4.166664568298827e-2f);
    const float cs = fmaf(z * z, cp, fmaf(z, -0.5f, 1.0f));
    const int q = static_cast<int>(k) & 3;
    s = (q & 1) ? cs : sn;
    c = (q & 1) ? sn : cs;
    if (q & 2) s = -s;
    if ((q + 1) & 2) c = -c;
  } else {
    const float k = rintf(th * 0.159154943091895336f);
    float r = fmaf(k, -6.28318548202514648f, th);
    r = fmaf(k, 1.74845553e-7f, r);
    __sincosf(r, &s, &c);
  }
  if constexpr (GAIN) return make_float2(c * g, s * g);
  else return make_float2(c, s);   // g == 1: c * 1 == c, bit-identical
}

// 8 filtered intensities -> rotation factors -> (cos, sin) buffer
template <bool PRECISE>
__device__ __forceinline__ void store_factors8(float2* __restrict__ csbuf, int p0, const float (&f)[8],
                                               float a, float g) {
#pragma unroll
  for (int o = 0; o < 8; o += 2) {
    const float2 c0 = rot_factor<PRECISE>(a, g, f[o]), c1 = rot_factor<PRECISE>(a, g, f[o + 1]);
    *reinterpret_cast<float4*>(csbuf + cs_phys(p0 + o)) = make_float4(c0.x, c0.y, c1.x, c1.y);
  }
}

__device__ __forceinline__ void store_factors8(float2* __restrict__ csbuf, int p0, const float (&f)[8],
                                               float a, float g, bool precise) {
  if (precise) store_factors8<true>(csbuf, p0, f, a, g);
  else store_factors8<false>(csbuf, p0, f, a, g);
}

// What the FIR lanes publish for the rotation (DBP_NL_PUBLISH_F):
//  1 (default): programs on the SFU sincos (<= 2 steps) publish the filtered
//    intensity F itself, 4 bytes per position at fir_phys(p) -- each lane
//    then evaluates the (cos, sin) of its own 16 positions (twice the SFU
//    work, which has room) and the shared-memory traffic of the factor
//    exchange halves: 2 STS.128 + 16 LDS.32 (24 wavefronts per warp) instead
//    of 4 STS.128 + 16 LDS.64 (48).  Programs on the polynomial sincos
//    (>= 3 steps) publish the factors: doubling ~15 FMA-pipe operations per
//    factor cost N_s = 4 up to 6% (profiles/r2/final/configs_v10.jsonl);
//  0: always the rotation factors (cos, sin) g, 8 bytes per position at cs_phys(p).
#ifndef DBP_NL_PUBLISH_F
#define DBP_NL_PUBLISH_F 1
#endif
// factors: publish (cos, sin) g (the polynomial-sincos programs of the
// exact-adjoint instantiation), else F; precise: which sincos the factors use
__device__ __forceinline__ void publish8(float* __restrict__ nlbuf, int p0, const float (&f)[8], float a, float g,
                                         bool precise, bool factors) {
#if DBP_NL_PUBLISH_F
  if (!factors) {
    // p0 = 16 t + 8 pol: both float4 stay inside one 16-float pad group
    float* dst = nlbuf + fir_phys(p0);
    *reinterpret_cast<float4*>(dst) = make_float4(f[0], f[1], f[2], f[3]);
    *reinterpret_cast<float4*>(dst + 4) = make_float4(f[4], f[5], f[6], f[7]);
    return;
  }
  store_factors8(reinterpret_cast<float2*>(nlbuf), p0, f, a, g, precise);
#else
  store_factors8(reinterpret_cast<float2*>(nlbuf), p0, f, a, g, precise);
#endif
}

// v[m] *= the published (cos, sin) g factor of position m T + t
template <int LOGN, class SH>
__device__ __forceinline__ void rotate_by_factors(float2 (&v)[16], const float* __restrict__ nlbuf, SH& sh, int t) {
  constexpr int T = Geo<LOGN>::T;
  const float2* csbuf = reinterpret_cast<const float2*>(nlbuf);
  if constexpr (T >= 16) {
    const float2* cb = csbuf + cs_phys(t);  // cs_phys(m T + t) = m (9T/8) + cs_phys(t)
    float2 cs[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) cs[m] = cb[m * (9 * T / 8)];
    sh.reads_done();
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = c_mul(v[m], cs[m]);
  } else {
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = c_mul(v[m], csbuf[cs_phys(m * T + t)]);
    sh.reads_done();
  }
}

// v[m] *= (cos, sin)(a F_m) g for the 16 published F of this lane's positions
template <bool PRECISE>
__device__ __forceinline__ void rotate_by_f(float2 (&v)[16], const float (&fv)[16], float a, float g) {
  if (g == 1.0f) {
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = c_mul(v[m], rot_factor<PRECISE, false>(a, g, fv[m]));
  } else {
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = c_mul(v[m], rot_factor<PRECISE, true>(a, g, fv[m]));
  }
}

#ifndef DBP_FIR_PACKED
#define DBP_FIR_PACKED 0
#endif
// Packed FP32 pairs for the FIR (FADD2 / FMUL2 / FFMA2 on float2)
__device__ __forceinline__ float2 p_mul(float2 a, float2 b) {
  return f2_unpack(f2_mul(f2_pack(a.x, a.y), f2_pack(b.x, b.y)));
}
__device__ __forceinline__ float2 p_fma(float2 a, float2 b, float2 c) {
  return f2_unpack(f2_fma(f2_pack(a.x, a.y), f2_pack(b.x, b.y), f2_pack(c.x, c.y)));
}

// 8 consecutive FIR outputs p0 .. p0+7 from a register window of the padded
// intensity buffer, turned into rotation factors and stored to csbuf.
// Packed: the window's aligned register pairs (w[2k], w[2k+1]) feed FADD2 /
// FFMA2 directly when the pair of outputs and the tap share parity, so the
// centre and even taps accumulate into output pairs (f[2j], f[2j+1]) and the
// odd taps into (f[2j-1], f[2j]) (j = 0..4; f[-1], f[8] are discarded), the
// two halves added at the end: 166 instead of 280 FP instructions at N_c = 17.
#ifndef DBP_FIR_DIRECT
#define DBP_FIR_DIRECT 1
#endif
// packed direct form (FFMA2 on output pairs, bit-identical): measured -0.9% at
// N_c = 17 and -1.8% at 33 (profiles/r2/ab_firpacked.txt) -- the FIR is
// FMA-pipe bound, and FFMA2 needs every coefficient moved from a uniform
// register into a regular one (~100 MOV per lane) -- so off
#ifndef DBP_FIR_DIRECT_PACKED
#define DBP_FIR_DIRECT_PACKED 0
#endif
// DIRECT: the streamed direct form (N >= 1024, where it lets the fixed-tap
// kernel fit 64 registers); below, the folded symmetric form measured 0.2-1%
// faster (profiles/r1/ab_v8.txt)
template <int NC, bool DIRECT>
__device__ __forceinline__ void fir8_fixed(const float* __restrict__ ibuf, float* __restrict__ nlbuf,
                                           int p0, float a, float g, const KernelParams& kp, int n_blk,
                                           bool factors) {
  constexpr int PW = (NC + 3) & ~3;
  constexpr int W = 8 + 2 * PW;
  if constexpr (DIRECT) {
  // Direct form streamed over the window: each 4-float piece of the padded
  // intensity window is folded into the 8 accumulators with the coefficient of
  // its tap offset (a constant-bank FFMA operand), so only f[8] and one piece
  // are live -- the same 2 N_c + 1 FP instructions per output as the folded
  // symmetric form, ~40 fewer registers at N_c = 17.
  float fd[8];
#if DBP_FIR_DIRECT_PACKED
  // Packed: output pairs (f[2j], f[2j+1]) take window pairs (w[u], w[u+1])
  // with ONE tap, d = u - 2j - PW, so each FFMA2 serves two outputs -- half the
  // FIR instructions, the same FMA-pipe time, and the same per-output
  // summation order (increasing u) as the scalar form: bit-identical.  Pairs
  // at even u are a float4's (x, y) / (z, w); odd u pairs (y, z) and
  // (previous w, x) are assembled with moves.
  unsigned long long acc[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j] = f2_pack(0.f, 0.f);
  float prev_w = 0.f;
#pragma unroll
  for (int m = 0; m < W / 4; ++m) {
    DBP_CHECK(fir_phys(p0 + 4 * m) + 3 < fir_phys(n_blk + 2 * PW) + 4);
    const float4 q = *reinterpret_cast<const float4*>(ibuf + fir_phys(p0 + 4 * m));
    const unsigned long long pr[4] = {f2_pack(prev_w, q.x), f2_pack(q.x, q.y), f2_pack(q.y, q.z),
                                      f2_pack(q.z, q.w)};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int u = 4 * m - 1 + k;          // first window index of pair k
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int d = u - 2 * j - PW;
        if (u >= 0 && d >= -NC && d <= NC) {
          const float c = kp.c[d < 0 ? -d : d];
          acc[j] = f2_fma(f2_pack(c, c), pr[k], acc[j]);
        }
      }
    }
    prev_w = q.w;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f2 = f2_unpack(acc[j]);
    fd[2 * j] = f2.x;
    fd[2 * j + 1] = f2.y;
  }
#else
#pragma unroll
  for (int o = 0; o < 8; ++o) fd[o] = 0.f;
#pragma unroll
  for (int m = 0; m < W / 4; ++m) {
    DBP_CHECK(fir_phys(p0 + 4 * m) + 3 < fir_phys(n_blk + 2 * PW) + 4);
    const float4 q = *reinterpret_cast<const float4*>(ibuf + fir_phys(p0 + 4 * m));
    const float wq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        const int d = 4 * m + e - PW - o;   // tap offset of this window sample for output o
        if (d >= -NC && d <= NC) fd[o] = fmaf(kp.c[d < 0 ? -d : d], wq[e], fd[o]);
      }
    }
  }
#endif
  publish8(nlbuf, p0, fd, a, g, kp.precise_sincos, factors);
  return;
  }
  float w[W];
#pragma unroll
  for (int m = 0; m < W / 4; ++m) {
    DBP_CHECK(fir_phys(p0 + 4 * m) + 3 < fir_phys(n_blk + 2 * PW) + 4);
    const float4 q = *reinterpret_cast<const float4*>(ibuf + fir_phys(p0 + 4 * m));
    w[4 * m] = q.x; w[4 * m + 1] = q.y; w[4 * m + 2] = q.z; w[4 * m + 3] = q.w;
  }
#if DBP_FIR_PACKED
  auto wp = [&](int k) { return make_float2(w[k], w[k + 1]); };   // k even: one register pair
  float2 e[4], o[5];
  const float2 cc0 = make_float2(kp.c[0], kp.c[0]);
#pragma unroll
  for (int j = 0; j < 4; ++j) e[j] = p_mul(cc0, wp(2 * j + PW));
#pragma unroll
  for (int i = 2; i <= NC; i += 2) {
    const float2 ci = make_float2(kp.c[i], kp.c[i]);
#pragma unroll
    for (int j = 0; j < 4; ++j) e[j] = p_fma(ci, c_add(wp(2 * j + PW - i), wp(2 * j + PW + i)), e[j]);
  }
#pragma unroll
  for (int i = 1; i <= NC; i += 2) {
    const float2 ci = make_float2(kp.c[i], kp.c[i]);
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const float2 s = c_add(wp(2 * j - 1 + PW - i), wp(2 * j - 1 + PW + i));
      o[j] = i == 1 ? p_mul(ci, s) : p_fma(ci, s, o[j]);
    }
  }
  float f[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    f[2 * j] = e[j].x + o[j].y;
    f[2 * j + 1] = e[j].y + o[j + 1].x;
  }
#else
  float f[8];
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    float acc = kp.c[0] * w[o + PW];
#pragma unroll
    for (int i = 1; i <= NC; ++i) acc = fmaf(kp.c[i], w[o + PW - i] + w[o + PW + i], acc);
    f[o] = acc;
  }
#endif
  publish8(nlbuf, p0, f, a, g, kp.precise_sincos, factors);
}

// any nc (and per-item coefficient sets): taps in chunks of four, scalar
// (summation order differs from the packed fir8_fixed at the last ulp)
__device__ __forceinline__ void fir8_generic(const float* __restrict__ ibuf, float* __restrict__ nlbuf,
                                             int p0, int pw, float a, float g, const KernelParams& kp,
                                             const float* __restrict__ cptr, float c0, bool factors) {
  float f[8];
  {
    const float4 u = *reinterpret_cast<const float4*>(ibuf + fir_phys(p0 + pw));
    const float4 w = *reinterpret_cast<const float4*>(ibuf + fir_phys(p0 + pw + 4));
    f[0] = c0 * u.x; f[1] = c0 * u.y; f[2] = c0 * u.z; f[3] = c0 * u.w;
    f[4] = c0 * w.x; f[5] = c0 * w.y; f[6] = c0 * w.z; f[7] = c0 * w.w;
  }
#pragma unroll 1
  for (int i0 = 1; i0 <= kp.nc; i0 += 4) {
    // left: positions p0 - i0 - 3 .. p0 + 7 - i0; right: p0 + i0 .. p0 + 10 + i0
    float l[12], r[12];
    const int ul = p0 + pw - i0 - 3;
    const int ur = p0 + pw + i0 - 1;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const float4 x = *reinterpret_cast<const float4*>(ibuf + fir_phys(ul + 4 * m));
      const float4 y = *reinterpret_cast<const float4*>(ibuf + fir_phys(ur + 4 * m));
      l[4 * m] = x.x; l[4 * m + 1] = x.y; l[4 * m + 2] = x.z; l[4 * m + 3] = x.w;
      r[4 * m] = y.x; r[4 * m + 1] = y.y; r[4 * m + 2] = y.z; r[4 * m + 3] = y.w;
    }
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const float ci = __ldg(cptr + i0 + d);
#pragma unroll
      for (int o = 0; o < 8; ++o) f[o] = fmaf(ci, l[o + 3 - d] + r[o + 1 + d], f[o]);
    }
  }
  publish8(nlbuf, p0, f, a, g, kp.precise_sincos, factors);
}

// PROG (KernelProg): kProgNoFir compiles the F = c0 I path only; kProgGeneric
// the fixed-tap FIRs; kProgGenericFir adds the runtime-N_c fir8_generic
template <int LOGN, int MODE, int PROG = kProgGenericFir, int TWP = kTwDit, int PS = 0>
__device__ __forceinline__ void rotate(float2 (&v)[16], Shm<LOGN, MODE>& sh, const KernelParams& kp,
                                       int step_idx, int t, int pol, const float* __restrict__ cptr,
                                       PolXchg* px = nullptr) {
  // the fused-twiddle instantiation runs <= 2-step programs (SFU sincos): F is
  // published; the exact-adjoint one publishes factors for polynomial sincos
  // (N = 8192, one CTA per SM: the factors measured +1.9%, profiles/r2/ab_pubf_8192.txt);
  // polarisation-split pairs publish F (the factor buffer would not leave room
  // for two CTAs per SM)
  const bool factors = !PS && (DBP_NL_PUBLISH_F == 0 || LOGN >= 13 ||
                               (TWP != kTwDit && PROG != kProgSym1 && kp.precise_sincos));
  // per-item coefficient sets (training batches) read from global memory
  const float c0 = kp.coeff_stride ? __ldg(cptr) : kp.c[0];
  using G = Geo<LOGN>;
  constexpr int N = G::N, T = G::T;
  const float2 sg = __ldg(kp.steps + step_idx);  // (a_j, g_j)
  // total dual-pol intensity of positions t + T m, m = 8 pol .. 8 pol + 7:
  // each lane of a pair forms half of the 16 (own |v|^2 plus the partner
  // lane's, one shuffle per two positions)
  constexpr int NI = PS ? 16 : 8;
  float inten[NI];
  if constexpr (PS) {
    // this CTA's |v|^2 to the partner, the partner's to us (see PolXchg)
    float own[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) own[m] = fmaf(v[m].x, v[m].x, v[m].y * v[m].y);
    const uint32_t s = px->step;
    if (threadIdx.x == 0) mbar_expect_tx(px->full, 16u * T * sizeof(float));
    if (s > 0) mbar_wait_relaxed_cluster(px->free_, (s - 1) & 1u);
#pragma unroll
    for (int c = 0; c < 4; ++c)
      st_async_v4(px->peer_xbuf + 4u * xbuf_slot(t, c),
                  make_float4(own[4 * c], own[4 * c + 1], own[4 * c + 2], own[4 * c + 3]), px->peer_full);
    mbar_wait(px->full, s & 1u);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float4 o = *reinterpret_cast<const float4*>(px->xbuf + xbuf_slot(t, c));
      inten[4 * c] = own[4 * c] + o.x;
      inten[4 * c + 1] = own[4 * c + 1] + o.y;
      inten[4 * c + 2] = own[4 * c + 2] + o.z;
      inten[4 * c + 3] = own[4 * c + 3] + o.w;
    }
  } else {
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const float lo = fmaf(v[m].x, v[m].x, v[m].y * v[m].y);
      const float hi = fmaf(v[m + 8].x, v[m + 8].x, v[m + 8].y * v[m + 8].y);
      const float other = __shfl_xor_sync(0xffffffffu, pol ? lo : hi, 16);
      inten[m] = (pol ? hi : lo) + other;
    }
  }
  // PS: the partner may write its next values once ours are consumed (the
  // exchange buffer overlaps the tail of the F buffer, so after the F reads)
  auto release_xbuf = [&](float last_read) {
    if constexpr (PS) {
      const uint32_t dep = zero_after(last_read);
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive_peer_relaxed(px->peer_free + dep);
      ++px->step;
    }
  };
  if constexpr (PS) {
    if (PROG == kProgNoFir || kp.nc == 0) {
      release_xbuf((inten[3] + inten[7]) + (inten[11] + inten[15]));   // one value per xbuf load
      if (kp.precise_sincos) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = c_mul(v[i], rot_factor<true>(sg.x, sg.y, c0 * inten[i]));
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = c_mul(v[i], rot_factor<false>(sg.x, sg.y, c0 * inten[i]));
      }
      return;
    }
  }
  if (!PS && (PROG == kProgNoFir || kp.nc == 0)) {
    // F = c0 I: each lane of the pair evaluates half the factors, then swaps
    float2 fac[8];
    if (kp.precise_sincos) {
#pragma unroll
      for (int i = 0; i < 8; ++i) fac[i] = rot_factor<true>(sg.x, sg.y, c0 * inten[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) fac[i] = rot_factor<false>(sg.x, sg.y, c0 * inten[i]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float2 mine = fac[i];
      const float2 oth = make_float2(__shfl_xor_sync(0xffffffffu, mine.x, 16),
                                     __shfl_xor_sync(0xffffffffu, mine.y, 16));
      v[i] = c_mul(v[i], pol ? oth : mine);
      v[8 + i] = c_mul(v[8 + i], pol ? mine : oth);
    }
  } else {
    const int pw = kp.fir_pad;
    // intensity buffer (logical [-pw, N + pw)) and (cos, sin) buffer: regions
    // 1 and 0 when double-buffered, else the second behind the first
    float* ibuf = sh.template region<1>();
    float* nlbuf = Shm<LOGN, MODE>::DB ? sh.template region<0>() : ibuf + fir_phys(N + 2 * pw) + 4;
    // each lane stores its half of the intensities
    sh.before_write();
    const int m0 = 8 * pol;
    if constexpr (PS) {
      static_assert(T >= 16, "polarisation split only for large N");
      float* ib = ibuf + fir_phys(t + pw);
#pragma unroll
      for (int m = 0; m < 16; ++m) ib[m * (5 * T / 4)] = inten[m];
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const int j = m * T + t;
        if (j < pw) ibuf[fir_phys(j + N + pw)] = inten[m];
        if (j >= N - pw) ibuf[fir_phys(j - N + pw)] = inten[m];
      }
    } else if constexpr (T >= 16) {
      // fir_phys(m T + t + pw) = m (5T/4) + fir_phys(t + pw) for T >= 16
      float* ib = ibuf + fir_phys(t + pw) + m0 * (5 * T / 4);
#pragma unroll
      for (int m = 0; m < 8; ++m) ib[m * (5 * T / 4)] = inten[m];
      if (pw <= T) {
        if (!pol && t < pw) ibuf[fir_phys(t + N + pw)] = inten[0];                // j = t < pw
        if (pol && t >= T - pw) ibuf[fir_phys(15 * T + t - N + pw)] = inten[7];   // j >= N - pw
      } else {
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const int j = (m0 + m) * T + t;
          if (j < pw) ibuf[fir_phys(j + N + pw)] = inten[m];
          if (j >= N - pw) ibuf[fir_phys(j - N + pw)] = inten[m];
        }
      }
    } else {
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int j = (m0 + m) * T + t;
        ibuf[fir_phys(j + pw)] = inten[m];
        if (j < pw) ibuf[fir_phys(j + N + pw)] = inten[m];
        if (j >= N - pw) ibuf[fir_phys(j - N + pw)] = inten[m];
      }
    }
    if (DBP_EXPERIMENT_NONLBAR) __syncwarp(); else sh.after_write();
    constexpr bool kDirectFir = DBP_FIR_DIRECT && LOGN >= 10;
    // PS: each CTA filters all 16 of its positions (the partner does the same work)
#pragma unroll 1
    for (int h = 0; h < (PS ? 2 : 1); ++h) {
    const int p0 = 16 * t + 8 * (PS ? h : pol);
    switch (kp.coeff_stride ? -1 : kp.nc) {
      case 1: fir8_fixed<1, kDirectFir>(ibuf, nlbuf, p0, sg.x, sg.y, kp, N, factors); break;
      case 9: fir8_fixed<9, kDirectFir>(ibuf, nlbuf, p0, sg.x, sg.y, kp, N, factors); break;
      case 17: fir8_fixed<17, kDirectFir>(ibuf, nlbuf, p0, sg.x, sg.y, kp, N, factors); break;
      case 32: fir8_fixed<32, kDirectFir>(ibuf, nlbuf, p0, sg.x, sg.y, kp, N, factors); break;
      case 33: fir8_fixed<33, kDirectFir>(ibuf, nlbuf, p0, sg.x, sg.y, kp, N, factors); break;
      default:
        if constexpr (PROG == kProgGenericFir) fir8_generic(ibuf, nlbuf, p0, pw, sg.x, sg.y, kp, cptr, c0, factors);
        else __trap();   // the launcher routes these programs to kProgGenericFir
        break;
    }
    }
    if (DBP_EXPERIMENT_NONLBAR) __syncwarp(); else sh.after_write();
#if DBP_NL_PUBLISH_F
    if (!factors) {
      float fv[16];
      if constexpr (T >= 16) {
        const float* fb = nlbuf + fir_phys(t);  // fir_phys(m T + t) = m (5T/4) + fir_phys(t)
#pragma unroll
        for (int m = 0; m < 16; ++m) fv[m] = fb[m * (5 * T / 4)];
      } else {
#pragma unroll
        for (int m = 0; m < 16; ++m) fv[m] = nlbuf[fir_phys(m * T + t)];
      }
      sh.reads_done();
      if constexpr (PS) {
        float sum = 0.f;
#pragma unroll
        for (int m = 0; m < 16; ++m) sum += fv[m];
        release_xbuf(sum);   // every F read (the F buffer overlaps the exchange buffer)
      }
      if (PROG != kProgSym1 && kp.precise_sincos) rotate_by_f<true>(v, fv, sg.x, sg.y);
      else rotate_by_f<false>(v, fv, sg.x, sg.y);
    } else {
      rotate_by_factors<LOGN>(v, nlbuf, sh, t);
      release_xbuf(v[15].x);
    }
#else
    rotate_by_factors<LOGN>(v, nlbuf, sh, t);
    release_xbuf(v[15].x);
#endif
  }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
// Programs whose interior blocks arrive through the exchange planes (TMA bulk
// load): one block per CTA, so this never meets the persistent loop.
template <int LOGN, int PROG>
__device__ __host__ constexpr bool tma_load_program() {
  return Geo<LOGN>::TMA_LOAD || (Geo<LOGN>::TMA_LOAD_OK && PROG == kProgFFE && DBP_FFE_TMA_LOAD);
}

// One CTA-sized group of blocks (block slices) through the whole program.
template <int LOGN, int MODE, int PROG, int TWP, int PS = 0>
__device__ __forceinline__ void process_group(const KernelParams& kp, Shm<LOGN, MODE>& sh, long long grp,
                                              long long n_groups, int t, int slice, int pol,
                                              long long gstride, PolXchg* px = nullptr) {
  using G = Geo<LOGN>;
  constexpr int N = G::N, T = G::T;
  const long long blk = grp * G::BPC + slice;
  const bool active = blk < kp.total_blocks;
  long long item = 0, b = 0;
  if (active) {
    item = kp.bpi_magic ? (long long)__umul64hi(kp.bpi_magic, (unsigned long long)blk) : blk / kp.blocks_per_item;
    b = kp.block_begin + (blk - item * kp.blocks_per_item);
  }

  const float* cptr = kp.coeff + (kp.coeff_stride ? item * kp.coeff_stride : 0);
  float2 v[16];
  const long long s0 = b * kp.step - kp.lead;  // global index of block sample 0
  bool loaded = false;
  constexpr bool kTmaLoad = tma_load_program<LOGN, PROG>();
  static_assert(!kTmaLoad || LOGN < DBP_PERSIST_MIN_LOGN, "TMA block input assumes one group per CTA");
  if constexpr (kTmaLoad) {
    // Interior block, 16-byte aligned rows (uniform per CTA): one elected
    // thread copies both polarisation rows (2 x 8N bytes) into the planes
    // with the TMA bulk engine and every thread then reads its 16 samples
    // from shared memory (conflict free).  The first exchange's leading
    // barrier orders these reads before the planes are overwritten: with
    // __syncthreads (kShmSync) directly, with split write-after-read barriers
    // because each warp's initial arrival is made after its reads below and
    // not at kernel start (an arrival at kernel start let a fast warp write
    // its first exchange over rows a slow warp had not read yet).  The
    // LDG path would stage 32 KB per CTA in flight through L1, whose
    // capacity (the unified L1 / shared array) measurably limits the kernel.
    __shared__ alignas(8) uint64_t in_bar;
    const long long off = kp.cyclic ? s0 : s0 - kp.in_origin;
    const float2* src = kp.in + item * kp.in_item_stride + off;
    const bool bulk = active && (!kp.cyclic || (s0 >= 0 && s0 + N <= kp.n_total)) &&
                      ((reinterpret_cast<uintptr_t>(src) | (uintptr_t)(kp.in_pol_stride * 8)) & 15) == 0;
    if (bulk) {
      if (threadIdx.x == 0) mbar_init(&in_bar, 1);
      __syncthreads();
      float2* dst0 = reinterpret_cast<float2*>(sh.base);
      if (threadIdx.x == 0) {
        if constexpr (PS) {   // this CTA's polarisation only
          mbar_expect_tx(&in_bar, N * sizeof(float2));
          bulk_load(dst0, src + pol * kp.in_pol_stride, N * sizeof(float2), &in_bar);
        } else {
          mbar_expect_tx(&in_bar, 2 * N * sizeof(float2));
          bulk_load(dst0, src, N * sizeof(float2), &in_bar);
          bulk_load(dst0 + sh.plane_len(), src + kp.in_pol_stride, N * sizeof(float2), &in_bar);
        }
      }
      mbar_wait(&in_bar, 0);
      const float2* pl = dst0 + (PS ? 0 : pol) * sh.plane_len() + t;
#pragma unroll
      for (int m = 0; m < 16; ++m) v[m] = pl[m * T];
      loaded = true;
    }
  }
  if (loaded) {
  } else if (DBP_EXPERIMENT_NOLOAD && active) {
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = make_float2(1e-3f * (float)(t + m), 1e-3f * (float)(b & 7));
  } else if (active) {
    const float2* pin = kp.in + item * kp.in_item_stride + pol * kp.in_pol_stride;
    if (!kp.cyclic || (s0 >= 0 && s0 + N <= kp.n_total)) {
      // interior block (or pre-extended chunk): one contiguous window, immediate offsets
      const float2* src = pin + (kp.cyclic ? s0 : s0 - kp.in_origin) + t;
      DBP_CHECK((kp.cyclic ? s0 : s0 - kp.in_origin) >= 0);
      DBP_CHECK((kp.cyclic ? s0 : s0 - kp.in_origin) + N <= kp.in_pol_stride);
#pragma unroll
      for (int m = 0; m < 16; ++m) v[m] = ld_stream(src + m * T);
    } else {
      // edge block: circular extension of the whole signal (spectral.py:128)
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        long long gi = s0 + m * T + t;
        if (gi < 0 || gi >= kp.n_total) {
          gi %= kp.n_total;
          if (gi < 0) gi += kp.n_total;
        }
        DBP_CHECK(gi >= 0 && gi < kp.n_total);
        v[m] = ld_stream(pin + gi);
      }
    }
  } else {
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = make_float2(0.f, 0.f);
  }
  if constexpr (kTmaLoad && MODE == kShmSplitWar) sh.reads_done();  // the deferred initial arrival
  if (grp + gstride < n_groups) {
    // L2 prefetch of the next group's block: one 128-byte line per thread and polarisation
    const long long nblk = (grp + gstride) * G::BPC + slice;
    if (nblk < kp.total_blocks) {
      const long long nitem = kp.bpi_magic ? (long long)__umul64hi(kp.bpi_magic, (unsigned long long)nblk)
                                           : nblk / kp.blocks_per_item;
      const long long nb = kp.block_begin + (nblk - nitem * kp.blocks_per_item);
      const long long ns0 = nb * kp.step - kp.lead;
      if (!kp.cyclic || (ns0 >= 0 && ns0 + N <= kp.n_total)) {
        const float2* pn = kp.in + nitem * kp.in_item_stride + pol * kp.in_pol_stride +
                           (kp.cyclic ? ns0 : ns0 - kp.in_origin) + 16 * t;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pn));
      }
    }
  }

  // operator program (dbp.py:212-233), decoded on the host (KernelParams)
  if constexpr (PROG == kProgFFE) {
    // linear-only program (dbp.py:185-191): one convolution with H.  Its
    // exchange needs no write-after-read barrier when the CTA has not read
    // shared memory before (one group per CTA, input by LDG, plain
    // __syncthreads barriers): 3 CTA barriers instead of 4.  Used for N >= 2048
    // (launch.h): at N = 2048 with 1024 threads per SM (ffe_threads_per_sm),
    // at N = 8192 it also drops the generic kernel's stack spill.
    // In the generic kernel the same skip costs more than it saves (the
    // ESSFM / SSFM programs lose 0.1-1.8% to a moved barrier, a runtime op == 0
    // predicate that spills, or a peeled first operator:
    // profiles/r1/ab_fresh_start.txt).
    constexpr bool kFresh = MODE == kShmSync && !kTmaLoad && LOGN < DBP_PERSIST_MIN_LOGN;
    conv_block<LOGN, MODE, kFresh, TWP>(v, sh, kp.tab_full, kp.twiddle, t);
  } else if constexpr (PROG == kProgSym1) {
    conv_block<LOGN, MODE, false, TWP>(v, sh, kp.tab_half, kp.twiddle, t);
    if constexpr (!DBP_EXPERIMENT_NONL) rotate<LOGN, MODE, PROG, TWP, PS>(v, sh, kp, 0, t, pol, cptr, px);
    conv_block<LOGN, MODE, false, TWP>(v, sh, kp.tab_half, kp.twiddle, t);
  } else {
  const int n_ops = kp.n_ops;
  for (int op = 0; op < n_ops; ++op) {
    const bool is_conv = kp.conv_all || (op & 1) == kp.conv_parity;
    const float2* tab = kp.half_ends && (op == 0 || op == n_ops - 1) ? kp.tab_half : kp.tab_full;
    const int sidx = op >> kp.sidx_shift;
    if (is_conv) {
      conv_block<LOGN, MODE, false, TWP>(v, sh, tab, kp.twiddle, t);
    } else if (DBP_EXPERIMENT_NONL) {
    } else {
      rotate<LOGN, MODE, PROG, TWP, PS>(v, sh, kp, sidx, t, pol, cptr, px);
    }
  }
  }

  if (DBP_EXPERIMENT_NOSTORE && active) {
    // keep the results live without storing them (a never-taken data-dependent store)
    float acc = 0.f;
#pragma unroll
    for (int m = 0; m < 16; ++m) acc += v[m].x + v[m].y;
    if (__float_as_uint(acc) == 0x7fc00123u) kp.out[t] = make_float2(acc, acc);
  }
  if constexpr (G::TMA_STORE) {
    // One block per CTA, so every condition below is CTA-uniform.  Kept
    // samples j in [lead, hi) go to shared memory as [pol][step] (the exchange
    // planes are free once every warp has passed the write-after-read
    // barrier), then one elected thread writes each polarisation's row with a
    // bulk copy; it alone waits for the engine to have read shared memory.
    if (active && !DBP_EXPERIMENT_NOSTORE) {
      const long long rem = kp.n_total - b * kp.step;
      const int len = rem < kp.step ? (int)rem : kp.step;
      const long long o0 = b * kp.step - kp.out_origin;       // output index of kept sample `lead`
      float2* row0 = kp.out + item * kp.out_item_stride + o0;
      const bool bulk = ((kp.step | len) & 1) == 0 && (kp.out_pol_stride & 1) == 0 &&
                        (reinterpret_cast<uintptr_t>(row0) & 15) == 0;
      if (bulk) {
        sh.before_write();
        float2* stg = reinterpret_cast<float2*>(sh.base) + (PS ? 0 : pol) * kp.step - kp.lead;
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          const int j = m * T + t;
          if (j >= kp.lead && j < kp.lead + len) stg[j] = v[m];
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
          const float2* src = reinterpret_cast<const float2*>(sh.base);
          if constexpr (PS) {
            bulk_store(row0 + pol * kp.out_pol_stride, src, (uint32_t)len * 8u);
          } else {
            bulk_store(row0, src, (uint32_t)len * 8u);
            bulk_store(row0 + kp.out_pol_stride, src + kp.step, (uint32_t)len * 8u);
          }
          bulk_store_commit_and_wait_read();
        }
        return;
      }
    }
  }
  if (active && !DBP_EXPERIMENT_NOSTORE) {
    float2* pout = kp.out + item * kp.out_item_stride + pol * kp.out_pol_stride;
    const long long ob = b * kp.step - kp.lead - kp.out_origin;  // output index of block sample 0
    // kept samples j in [lead, min(lead + step, lead + n_total - b step))
    const long long rem = kp.n_total - b * kp.step;
    const int hi = kp.lead + (rem < kp.step ? (int)rem : kp.step);
    float2* dst = pout + ob + t;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int j = m * T + t;
      if (j >= kp.lead && j < hi) {
        DBP_CHECK(ob + j >= 0 && ob + j < kp.out_pol_stride);
        __stcs(dst + m * T, v[m]);
      }
    }
  }
}

// PROG: kProgGeneric (any operator program, fixed-tap FIRs), kProgFFE (the
// single-convolution FFE program), kProgNoFir (split-step programs without an
// intensity FIR), kProgGenericFir (runtime N_c and per-item coefficient sets)
// PS = 1: polarisation-split pair (N = 8192, launched as 2-CTA clusters of
// T threads, see PolXchg); every other argument as the pol-pair kernel
template <int LOGN, int PROG = kProgGeneric, int TWP = kTwDit, int PS = 0>
__global__ void __launch_bounds__(PS ? Geo<LOGN>::T : Geo<LOGN>::THREADS,
                                  PS                        ? (1024 / Geo<LOGN>::T > 0 ? 1024 / Geo<LOGN>::T : 1)
                                  : PROG == kProgFFE        ? Geo<LOGN>::FFE_MIN_CTAS
                                  : PROG == kProgNoFir      ? Geo<LOGN>::NOFIR_MIN_CTAS
                                  : PROG == kProgGenericFir ? Geo<LOGN>::GENFIR_MIN_CTAS
                                                            : Geo<LOGN>::MIN_CTAS)
dbp_block_kernel(const KernelParams kp) {
  using G = Geo<LOGN>;
  constexpr int N = G::N, T = G::T;
  extern __shared__ float4 smem_raw[];
  if constexpr (PS) {
    static_assert(G::BPC == 1 && (LOGN >= DBP_PERSIST_MIN_LOGN || (PROG == kProgFFE && LOGN >= 10)),
                  "polarisation split: N = 8192, or the FFE program from N = 1024");
    constexpr int MODE = kShmSync;
    const int t = threadIdx.x;
    Shm<LOGN, MODE> sh;
    sh.init(reinterpret_cast<float*>(smem_raw), kp.slice_floats, 0);   // this CTA's planes only
    const long long n_groups = (kp.total_blocks + G::BPC - 1) / G::BPC;
    const long long gstride = gridDim.x >> 1;
    if constexpr (PROG == kProgFFE) {
      // the linear program never couples the polarisations: independent CTAs, no cluster
      for (long long grp = blockIdx.x >> 1; grp < n_groups; grp += gstride)
        process_group<LOGN, MODE, PROG, TWP, 1>(kp, sh, grp, n_groups, t, 0, blockIdx.x & 1, gstride);
      return;
    }
    const uint32_t rank = cluster_ctarank();
    const int pol = (int)rank;
    __shared__ alignas(8) uint64_t xbars[2];   // full, free
    PolXchg px;
    px.xbuf = reinterpret_cast<float*>(smem_raw) + 2 * plane_elems(N);   // behind this CTA's planes
    px.full = &xbars[0];
    px.free_ = &xbars[1];
    if (threadIdx.x == 0) {
      mbar_init(px.full, 1);
      mbar_init(px.free_, T / 32);
    }
    px.peer_xbuf = peer_smem_addr(px.xbuf, rank ^ 1u);
    px.peer_full = peer_smem_addr(px.full, rank ^ 1u);
    px.peer_free = peer_smem_addr(px.free_, rank ^ 1u);
    px.step = 0;
    cluster_sync_all();   // both CTAs' mbarriers initialised before any remote operation
    for (long long grp = blockIdx.x >> 1; grp < n_groups; grp += gstride)
      process_group<LOGN, MODE, PROG, TWP, 1>(kp, sh, grp, n_groups, t, 0, pol, gstride, &px);
    cluster_sync_all();   // no CTA leaves while its partner may still signal it
    return;
  } else {
  const int lane = threadIdx.x & 31;
  const int pol = lane >> 4;
  const int q = ((threadIdx.x >> 5) << 4) + (lane & 15);  // position-thread index within the CTA
  const int t = q % T;
  const int slice = q / T;
  constexpr int MODE = G::DB ? kShmDouble : (G::SPLIT_WAR ? kShmSplitWar : kShmSync);
  Shm<LOGN, MODE> sh;
  sh.init(reinterpret_cast<float*>(smem_raw) + slice * kp.slice_floats, kp.slice_floats, pol);
  if constexpr (MODE == kShmSplitWar) {
    // one write-after-read mbarrier per slice, arrived on by each of its T/16 warps
    __shared__ alignas(8) uint64_t war_bars[G::BPC];
    if (threadIdx.x < G::BPC) mbar_init(&war_bars[threadIdx.x], T / 16);
    __syncthreads();
    sh.war = &war_bars[slice];
    // nothing to protect before the first write phase -- unless the block
    // input arrives through the planes (TMA load): process_group arrives then
    if constexpr (!tma_load_program<LOGN, PROG>()) sh.reads_done();
  }

  // N <= 4096: one group per CTA (full-size grid).  N = 8192: a persistent
  // grid strides over the groups, prefetching the next group's input into L2
  // meanwhile (the launcher sizes it; DBP_PERSISTENT).
  // (compile-time split: the strided loop costs ~0.5% where it is not used)
  const long long n_groups = (kp.total_blocks + G::BPC - 1) / G::BPC;
  if constexpr (LOGN >= DBP_PERSIST_MIN_LOGN) {
    for (long long grp = blockIdx.x; grp < n_groups; grp += gridDim.x)
      process_group<LOGN, MODE, PROG, TWP>(kp, sh, grp, n_groups, t, slice, pol, gridDim.x);
  } else {
    process_group<LOGN, MODE, PROG, TWP>(kp, sh, blockIdx.x, n_groups, t, slice, pol, gridDim.x);
  }
  }
}

}  // namespace dbp

namespace dbp {

// ---------------------------------------------------------------------------
// FFE program (dbp.py:185-191) as a persistent, software-pipelined stream:
// each CTA strides over the blocks, and while it transforms block i the TMA
// engine already copies block i + gridDim.x into a dedicated shared buffer
// (both polarisation rows, 2 N float2), so every SM keeps a block's input in
// flight at all times -- the one-shot CTA of dbp_block_kernel<.., kProgFFE>
// left the HBM idle while its CTAs computed (HBM fraction 0.6).  The output
// leaves through the TMA bulk store (Geo::TMA_STORE path).  Blocks that are
// not bulk-copyable (cyclic edge blocks, odd alignment) fall back to LDG / STG.
// Measured slower and off by default (DBP_FFE_STREAM=1 selects it): 87.5 vs
// 100.7 GS/s at 2048/700, 80.8 vs 97.2 at 4096/700 -- the input buffer costs
// a CTA per SM (24 instead of 32 warps at N = 2048, 16 instead of 32 at 4096)
// and the prefetch does not win it back (profiles/r2/ffe_stream.txt).
// ---------------------------------------------------------------------------
// resident CTAs per SM the stream kernel is built for: shared memory allows
// three at N = 2048 (planes 37 KB + input buffer 32 KB each), one at 4096
__host__ __device__ constexpr int ffe_stream_ctas(int logn) { return logn <= 11 ? 3 : 1; }

template <int LOGN>
__global__ void __launch_bounds__(Geo<LOGN>::THREADS, ffe_stream_ctas(LOGN)) dbp_ffe_stream_kernel(const KernelParams kp) {
  using G = Geo<LOGN>;
  static_assert(G::BPC == 1, "one block per CTA");
  constexpr int N = G::N, T = G::T;
  extern __shared__ float4 smem_raw[];
  const int lane = threadIdx.x & 31;
  const int pol = lane >> 4;
  const int t = ((threadIdx.x >> 5) << 4) + (lane & 15);
  constexpr int MODE = G::SPLIT_WAR ? kShmSplitWar : kShmSync;
  Shm<LOGN, MODE> sh;
  sh.init(reinterpret_cast<float*>(smem_raw), kp.slice_floats, pol);
  float2* inbuf = reinterpret_cast<float2*>(reinterpret_cast<float*>(smem_raw) + kp.slice_floats);  // [2][N]
  __shared__ alignas(8) uint64_t in_bar;
  __shared__ alignas(8) uint64_t war_bar;
  if (threadIdx.x == 0) {
    mbar_init(&in_bar, 1);
    if constexpr (MODE == kShmSplitWar) mbar_init(&war_bar, T / 16);
  }
  __syncthreads();
  if constexpr (MODE == kShmSplitWar) {
    sh.war = &war_bar;
    sh.reads_done();
  }
  // block blk -> (item, b, source row of polarisation x), and whether the TMA may copy it
  auto locate = [&](long long blk, long long& item, long long& b, const float2*& src) -> bool {
    item = kp.bpi_magic ? (long long)__umul64hi(kp.bpi_magic, (unsigned long long)blk) : blk / kp.blocks_per_item;
    b = kp.block_begin + (blk - item * kp.blocks_per_item);
    const long long s0 = b * kp.step - kp.lead;
    const long long off = kp.cyclic ? s0 : s0 - kp.in_origin;
    src = kp.in + item * kp.in_item_stride + off;
    const bool interior = !kp.cyclic || (s0 >= 0 && s0 + N <= kp.n_total);
    return interior && ((reinterpret_cast<uintptr_t>(src) | (uintptr_t)(kp.in_pol_stride * 8)) & 15) == 0;
  };
  auto issue = [&](const float2* src) {
    mbar_expect_tx(&in_bar, 2 * N * sizeof(float2));
    bulk_load(inbuf, src, N * sizeof(float2), &in_bar);
    bulk_load(inbuf + N, src + kp.in_pol_stride, N * sizeof(float2), &in_bar);
  };
  uint32_t in_phase = 0;
  long long blk = blockIdx.x;
  bool pending = false;
  if (blk < kp.total_blocks) {
    long long item, b;
    const float2* src;
    pending = locate(blk, item, b, src);
    if (pending && threadIdx.x == 0) issue(src);
  }
  for (; blk < kp.total_blocks; blk += gridDim.x) {
    long long item, b;
    const float2* src;
    locate(blk, item, b, src);
    float2 v[16];
    if (pending) {
      mbar_wait(&in_bar, in_phase);
      in_phase ^= 1u;
      const float2* pl = inbuf + pol * N + t;
#pragma unroll
      for (int m = 0; m < 16; ++m) v[m] = pl[m * T];
    } else {
      const float2* pin = kp.in + item * kp.in_item_stride + pol * kp.in_pol_stride;
      const long long s0 = b * kp.step - kp.lead;
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        long long gi = s0 + m * T + t;
        if (kp.cyclic && (gi < 0 || gi >= kp.n_total)) {
          gi %= kp.n_total;
          if (gi < 0) gi += kp.n_total;
        }
        v[m] = ld_stream(pin + (kp.cyclic ? gi : gi - kp.in_origin));
      }
    }
    // every thread holds its samples: the buffer may take the next block
    __syncthreads();
    pending = false;
    const long long nxt = blk + gridDim.x;
    if (nxt < kp.total_blocks) {
      long long ni, nb;
      const float2* nsrc;
      pending = locate(nxt, ni, nb, nsrc);
      if (pending && threadIdx.x == 0) issue(nsrc);
    }
    conv_block<LOGN, MODE, false, kTwDit>(v, sh, kp.tab_full, kp.twiddle, t);
    // kept centre [lead, lead + len): TMA bulk store through the planes, else STG
    const long long rem = kp.n_total - b * kp.step;
    const int len = rem < kp.step ? (int)rem : kp.step;
    const long long o0 = b * kp.step - kp.out_origin;
    float2* row0 = kp.out + item * kp.out_item_stride + o0;
    const bool bulk = ((kp.step | len) & 1) == 0 && (kp.out_pol_stride & 1) == 0 &&
                      (reinterpret_cast<uintptr_t>(row0) & 15) == 0;
    if (bulk) {
      sh.before_write();
      float2* stg = reinterpret_cast<float2*>(sh.base) + pol * kp.step - kp.lead;
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const int j = m * T + t;
        if (j >= kp.lead && j < kp.lead + len) stg[j] = v[m];
      }
      fence_proxy_async_smem();
      __syncthreads();
      if (threadIdx.x == 0) {
        const float2* s = reinterpret_cast<const float2*>(sh.base);
        bulk_store(row0, s, (uint32_t)len * 8u);
        bulk_store(row0 + kp.out_pol_stride, s + kp.step, (uint32_t)len * 8u);
        bulk_store_commit_and_wait_read();
      }
      sh.reads_done();   // warp 0 arrives once the engine has read the staging rows
    } else {
      float2* dst = kp.out + item * kp.out_item_stride + pol * kp.out_pol_stride + (o0 - kp.lead) + t;
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const int j = m * T + t;
        if (j >= kp.lead && j < kp.lead + len) __stcs(dst + m * T, v[m]);
      }
    }
  }
}

}  // namespace dbp
