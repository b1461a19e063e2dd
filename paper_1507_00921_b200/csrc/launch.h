// Per-block-length launchers of the fused kernel (one translation unit per
// log2 N so the big unrolled kernels compile in parallel).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

#include "dbp_block_kernel.cuh"
#include "dbp_warp_kernel.cuh"
#include "dbp_r2_kernel.cuh"
#include "dbp_r2t_kernel.cuh"

namespace dbp {

constexpr int kMinLogN = 4;   // N = 16
constexpr int kMaxLogN = 13;  // N = 8192

struct LaunchShape {
  int threads_x;  // threads per CTA along x
  int threads_y;  // along y
  int slices;     // block slices per CTA
  bool double_buffer;  // two exchange regions per slice (Geo::DB)
  int min_ctas;       // resident CTAs per SM the kernel is built for (Geo::MIN_CTAS)
};

template <int LOGN>
cudaError_t launch_block_kernel(const KernelParams& kp, long long n_ctas, size_t smem_bytes,
                                cudaStream_t stream);

struct SimParams;

template <int LOGN>
cudaError_t launch_ssfm_row(const SimParams& sp, long long n_ctas, size_t smem_bytes, cudaStream_t stream,
                            bool column);

// Dynamic shared memory opt-in and, for tuning experiments, the preferred
// shared-memory carve-out in percent (env DBP_CARVEOUT; default: the driver's choice).
template <class K>
cudaError_t set_smem_attrs(K* kernel, size_t smem_bytes) {
  static const int carveout = [] {
    const char* v = std::getenv("DBP_CARVEOUT");
    return v && *v ? std::atoi(v) : -1;
  }();
  if (smem_bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
  }
  if (carveout >= 0) return cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  return cudaSuccess;
}

template <int LOGN>
LaunchShape launch_shape();

// Block lengths whose linear (FFE) program runs the FFE-only instantiation
// (measured, profiles/r1/ab_ffe_kernel.txt, ab_ffe_tps.txt: N = 8192 +6.5%,
// 4096 +0.2%, 2048 +5.6% at 1024 threads per SM; N = 1024 -0.2 to -2.7% at
// any occupancy, so it keeps the generic kernel)
#ifndef DBP_FFE_KERNEL_MIN_LOGN
#define DBP_FFE_KERNEL_MIN_LOGN 11
#endif

// The fused block kernel for one block length: the FFE-only instantiation for
// the linear program (N >= 2^DBP_FFE_KERNEL_MIN_LOGN), the generic
// operator-program kernel otherwise.
// Block lengths whose split-step programs without an intensity FIR (SSFM,
// ESSFM N_c = 0) run the no-FIR instantiation (profiles/r1/ab_nofir.txt:
// N = 2048 +2 to +4%, 4096 +1%, 8192 +4.2%; N = 1024 +0.1%, kept generic)
#ifndef DBP_NOFIR_KERNEL_MIN_LOGN
#define DBP_NOFIR_KERNEL_MIN_LOGN 11
#endif

// FFT flavour per program (DBP_DIT_MAX_STEPS): the fused-twiddle FFT for the
// linear program and split-step programs of <= DBP_DIT_MAX_STEPS steps, the
// exact-adjoint FFT above.  DBP_FFT=dit|adjoint (env) forces one (A/B runs).
#ifndef DBP_DIT_MAX_LOGN
#define DBP_DIT_MAX_LOGN 12
#endif
inline bool use_dit_fft(const KernelParams& kp) {
  static const int forced = [] {
    const char* v = std::getenv("DBP_FFT");
    if (!v || !*v) return -1;
    return (v[0] == 'd') ? 1 : 0;
  }();
  if (forced >= 0) return forced == 1;
  return kp.program == kFFE || kp.n_steps <= DBP_DIT_MAX_STEPS;
}

// Block lengths whose configs[0]-shaped program (symmetric, N_s = 1, fixed-tap
// FIR) runs the straight-line kProgSym1 instantiation.  Measured slower and
// off (14 = none): the two inlined convolutions spill 80 bytes at 64
// registers, -6% at N = 2048, -9% at 4096 (profiles/r2/ab_sym1.txt)
#ifndef DBP_SYM1_KERNEL_MIN_LOGN
#define DBP_SYM1_KERNEL_MIN_LOGN 14
#endif

template <int LOGN, int TWP>
auto select_block_kernel(const KernelParams& kp) {
  auto* kernel = dbp_block_kernel<LOGN, kProgGeneric, TWP>;
  if constexpr (LOGN >= DBP_FFE_KERNEL_MIN_LOGN) {
    if (kp.program == kFFE) kernel = dbp_block_kernel<LOGN, kProgFFE, TWP>;
  }
  if constexpr (LOGN >= DBP_NOFIR_KERNEL_MIN_LOGN) {
    if ((kp.program == kSSFM || kp.program == kESSFM) && kp.nc == 0)
      kernel = dbp_block_kernel<LOGN, kProgNoFir, TWP>;
  }
  if (kp.program != kFFE && kp.nc > 0 && (kp.coeff_stride != 0 || !fixed_fir_nc(kp.nc)))
    kernel = dbp_block_kernel<LOGN, kProgGenericFir, TWP>;
  if constexpr (LOGN >= DBP_SYM1_KERNEL_MIN_LOGN) {
    if ((kp.program == kSSFM || kp.program == kESSFM) && kp.arrangement == kSymmetric && kp.n_steps == 1 &&
        kp.nc > 0 && kp.coeff_stride == 0 && fixed_fir_nc(kp.nc) && !kp.precise_sincos)
      kernel = dbp_block_kernel<LOGN, kProgSym1, TWP>;
  }
  return kernel;
}

// FFE programs at these block lengths can run the persistent TMA-prefetching
// stream kernel (dbp_ffe_stream_kernel, DBP_FFE_STREAM=1; measured slower)
#ifndef DBP_FFE_STREAM_MIN_LOGN
#define DBP_FFE_STREAM_MIN_LOGN 11
#endif
#ifndef DBP_FFE_STREAM_MAX_LOGN
#define DBP_FFE_STREAM_MAX_LOGN 12
#endif
inline bool ffe_stream_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("DBP_FFE_STREAM");
    return v && v[0] == '1';
  }();
  return on;
}

template <int LOGN>
cudaError_t launch_ffe_stream(const KernelParams& kp, size_t smem_bytes, cudaStream_t stream) {
  auto* kernel = dbp_ffe_stream_kernel<LOGN>;
  const size_t smem = smem_bytes + (size_t)2 * Geo<LOGN>::N * sizeof(float2);
  cudaError_t e = set_smem_attrs(kernel, smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, Geo<LOGN>::THREADS, smem);
  if (e != cudaSuccess) return e;
  long long grid = (long long)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > kp.total_blocks) grid = kp.total_blocks;
  kernel<<<dim3((unsigned)grid), dim3(Geo<LOGN>::THREADS), smem, stream>>>(kp);
  return cudaGetLastError();
}

// FFE programs at N = 1024 .. 4096 run the warp-resident kernel
// (dbp_warp_kernel.cuh); env DBP_WARP_FFE=0 selects the block kernel (A/B runs)
inline bool warp_ffe_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("DBP_WARP_FFE");
    if (v && *v) return v[0] != '0';
    return DBP_WARP_FFE != 0;
  }();
  return on;
}

template <int LOGL>
cudaError_t launch_warp_ffe(const KernelParams& kp, cudaStream_t stream) {
  using W = WGeo<LOGL>;
  auto* kernel = dbp_warp_ffe_kernel<LOGL>;
  cudaError_t e = set_smem_attrs(kernel, W::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const long long ctas = (kp.total_blocks + W::BPC - 1) / W::BPC;
  if (ctas > 0x7fffffffLL) return cudaErrorInvalidValue;
  kernel<<<dim3((unsigned)ctas), dim3(W::THREADS), W::SMEM_BYTES, stream>>>(kp);
  return cudaGetLastError();
}

// N = 8192: polarisation-split pairs (dbp_block_kernel<13, PROG, TWP, 1>, one
// 512-thread CTA per polarisation, two CTAs per SM; split-step programs as
// 2-CTA clusters exchanging the intensity).  Measured against the 1024-thread
// pol-pair CTA (profiles/r2/ab_ps1.txt): FFE 8192/1024 +4.4%, but the
// per-step intensity handshake locks the pair together: ESSFM 8192/1400
// -17%, SSFM-20 8192/1024 -21%.  Default: the FFE program only; env
// DBP_POLSPLIT=1 (every program) / 0 (none) overrides.
inline int polsplit_mode() {
  static const int mode = [] {
    const char* v = std::getenv("DBP_POLSPLIT");
    if (v && *v) return v[0] == '0' ? 0 : 2;
    return 1;
  }();
  return mode;
}
// FFE programs from this block length run the split (env DBP_POLSPLIT_FFE_MIN_LOGN)
inline int polsplit_ffe_min_logn() {
  static const int v = [] {
    const char* e = std::getenv("DBP_POLSPLIT_FFE_MIN_LOGN");
    return e && *e ? std::atoi(e) : 11;
  }();
  return v;
}
template <int LOGN>
inline bool polsplit_enabled(const KernelParams& kp) {
  const int m = polsplit_mode();
  if (LOGN < 13) return m != 0 && kp.program == kFFE && LOGN >= polsplit_ffe_min_logn();
  return m == 2 || (m == 1 && kp.program == kFFE);
}

template <int LOGN, int TWP>
auto select_ps_kernel(const KernelParams& kp) {
  auto* kernel = dbp_block_kernel<LOGN, kProgGeneric, TWP, 1>;
  if (kp.program == kFFE) kernel = dbp_block_kernel<LOGN, kProgFFE, TWP, 1>;
  if ((kp.program == kSSFM || kp.program == kESSFM) && kp.nc == 0) kernel = dbp_block_kernel<LOGN, kProgNoFir, TWP, 1>;
  if (kp.program != kFFE && kp.nc > 0 && (kp.coeff_stride != 0 || !fixed_fir_nc(kp.nc)))
    kernel = dbp_block_kernel<LOGN, kProgGenericFir, TWP, 1>;
  return kernel;
}

template <int LOGN>
cudaError_t launch_polsplit(const KernelParams& kp0, cudaStream_t stream) {
  using G = Geo<LOGN>;
  KernelParams kp = kp0;
  const bool fir = kp.program != kFFE && kp.nc > 0;
  kp.slice_floats = ps_smem_floats(G::N, kp.fir_pad, fir, kp.program != kFFE);
  const size_t smem = (size_t)kp.slice_floats * sizeof(float);
  auto* kernel = dbp_block_kernel<LOGN, kProgFFE, kTwDit, 1>;   // N = 1024 .. 4096: FFE only, DIT FFT
  if constexpr (LOGN >= DBP_PERSIST_MIN_LOGN) kernel = select_ps_kernel<LOGN, DBP_TW_POWERS>(kp);
  cudaError_t e = set_smem_attrs(kernel, smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long clusters = kp.total_blocks;   // one block (group) per pair
  if (LOGN >= DBP_PERSIST_MIN_LOGN && clusters > sms) clusters = sms;   // persistent: two CTAs per SM
  if (2 * clusters > 0x7fffffffLL) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * clusters));
  cfg.blockDim = dim3(G::T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = kp.program == kFFE ? 0 : 1;   // the FFE pairs never communicate
  e = cudaLaunchKernelEx(&cfg, kernel, kp);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// N = 8192 as a radix-2 step around two 4096-point transforms per thread
// (dbp_r2_kernel.cuh); env DBP_R2=0|1 overrides the default
inline bool r2_enabled(const KernelParams& kp) {
  static const int mode = [] {   // 0 off, 1 split-step programs, 2 every program
    const char* v = std::getenv("DBP_R2");
    if (v && *v) return v[0] == '0' ? 0 : 2;
    return DBP_R2 != 0 ? 1 : 0;
  }();
  return mode == 2 || (mode == 1 && kp.program != kFFE);
}

template <int TWP>
auto select_r2_kernel(const KernelParams& kp) {
  auto* kernel = dbp_r2_kernel<kProgGeneric, TWP>;
  if (kp.program == kFFE) kernel = dbp_r2_kernel<kProgFFE, TWP>;
  if ((kp.program == kSSFM || kp.program == kESSFM) && kp.nc == 0) kernel = dbp_r2_kernel<kProgNoFir, TWP>;
  if (kp.program != kFFE && kp.nc > 0 && (kp.coeff_stride != 0 || !fixed_fir_nc(kp.nc)))
    kernel = dbp_r2_kernel<kProgGenericFir, TWP>;
  return kernel;
}

template <int LOGN>
cudaError_t launch_r2(const KernelParams& kp0, cudaStream_t stream) {
  KernelParams kp = kp0;
  kp.slice_floats = r2_slice_floats(kp.fir_pad);
  const size_t smem = (size_t)kp.slice_floats * sizeof(float);
  auto* kernel = use_dit_fft(kp) ? select_r2_kernel<kTwDit>(kp) : select_r2_kernel<DBP_TW_POWERS>(kp);
  cudaError_t e = set_smem_attrs(kernel, smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long grid = kp.total_blocks < sms ? kp.total_blocks : sms;   // persistent, one CTA per SM
  kernel<<<dim3((unsigned)grid), dim3(R2Geo::THREADS), smem, stream>>>(kp);
  return cudaGetLastError();
}

// N = 8192 split-step programs with the parked subsequence in TMEM, two CTAs
// per SM (dbp_r2t_kernel.cuh); env DBP_R2T=0|1 overrides the default
inline bool r2t_enabled(const KernelParams& kp) {
  static const int mode = [] {   // 0 off, 1 split-step programs, 2 every program
    const char* v = std::getenv("DBP_R2T");
    if (v && *v) return v[0] == '0' ? 0 : (v[0] == '2' ? 2 : 1);
    return DBP_R2T != 0 ? 1 : 0;
  }();
  return mode == 2 || (mode == 1 && kp.program != kFFE);
}

template <int TWP>
auto select_r2t_kernel(const KernelParams& kp) {
  auto* kernel = dbp_r2t_kernel<kProgGeneric, TWP>;
  if (kp.program == kFFE) kernel = dbp_r2t_kernel<kProgFFE, TWP>;
  if ((kp.program == kSSFM || kp.program == kESSFM) && kp.nc == 0) kernel = dbp_r2t_kernel<kProgNoFir, TWP>;
  if (kp.program != kFFE && kp.nc > 0 && (kp.coeff_stride != 0 || !fixed_fir_nc(kp.nc)))
    kernel = dbp_r2t_kernel<kProgGenericFir, TWP>;
  return kernel;
}

// (templates on the block length so only the N = 8192 translation unit
// instantiates the R2 / R2T kernels)
template <int LOGN>
cudaError_t launch_r2t(const KernelParams& kp0, cudaStream_t stream) {
  KernelParams kp = kp0;
  kp.slice_floats = r2t_slice_floats(kp.fir_pad);
  const size_t smem = (size_t)kp.slice_floats * sizeof(float);
  auto* kernel = use_dit_fft(kp) ? select_r2t_kernel<kTwDit>(kp) : select_r2t_kernel<DBP_TW_POWERS>(kp);
  cudaError_t e = set_smem_attrs(kernel, smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // persistent, two CTAs per SM (each holds half the SM's TMEM columns)
  long long grid = kp.total_blocks < 2LL * sms ? kp.total_blocks : 2LL * sms;
  kernel<<<dim3((unsigned)grid), dim3(R2TGeo::THREADS), smem, stream>>>(kp);
  return cudaGetLastError();
}

// launch_polsplit<11> (the FFE program as polarisation-split pairs at N = 2048), dbp_kernel_ffe_ps.cu
cudaError_t launch_polsplit_ffe_2048(const KernelParams& kp, cudaStream_t stream);

template <int LOGN>
cudaError_t launch_block_kernel_impl(const KernelParams& kp, long long n_ctas, size_t smem_bytes,
                                     cudaStream_t stream) {
  if constexpr (LOGN == 13) {
    if (kp.r2_full != nullptr && kp.r2_tw != nullptr && (kp.half_ends == 0 || kp.r2_half != nullptr)) {
      if (r2t_enabled(kp)) return launch_r2t<LOGN>(kp, stream);
      if (r2_enabled(kp)) return launch_r2<LOGN>(kp, stream);
    }
  }
  if constexpr (LOGN == 13) {
    if (polsplit_enabled<LOGN>(kp)) return launch_polsplit<LOGN>(kp, stream);
  } else if constexpr (LOGN >= 10 && LOGN <= 12) {
    // the N = 2048 FFE pairs are instantiated in their own unit (dbp_kernel_ffe_ps.cu),
    // which build.py compiles with its own ptxas register-usage level
    if (polsplit_enabled<LOGN>(kp)) {
      if constexpr (LOGN == 11) return launch_polsplit_ffe_2048(kp, stream);
      else return launch_polsplit<LOGN>(kp, stream);
    }
  }
  if constexpr (LOGN >= 10 && LOGN <= 12) {
    if (kp.program == kFFE && kp.wtw != nullptr && kp.tab_nat != nullptr && warp_ffe_enabled()) return launch_warp_ffe<LOGN - 6>(kp, stream);
  }
  if constexpr (LOGN >= DBP_FFE_STREAM_MIN_LOGN && LOGN <= DBP_FFE_STREAM_MAX_LOGN) {
    if (kp.program == kFFE && ffe_stream_enabled()) return launch_ffe_stream<LOGN>(kp, smem_bytes, stream);
  }
  // N = 8192 keeps the exact-adjoint FFT: +1% there (profiles/r2/ab_dit_by_n.txt)
  const bool dit = LOGN <= DBP_DIT_MAX_LOGN && use_dit_fft(kp);
  auto* kernel = dit ? select_block_kernel<LOGN, kTwDit>(kp) : select_block_kernel<LOGN, DBP_TW_POWERS>(kp);
  cudaError_t e = set_smem_attrs(kernel, smem_bytes);
  if (e != cudaSuccess) return e;
  const LaunchShape sh = launch_shape<LOGN>();
  kernel<<<dim3((unsigned)n_ctas), dim3(sh.threads_x, sh.threads_y), smem_bytes, stream>>>(kp);
  return cudaGetLastError();
}

template <int LOGN>
LaunchShape launch_shape() {
  return LaunchShape{Geo<LOGN>::THREADS, 1, Geo<LOGN>::BPC, Geo<LOGN>::DB, Geo<LOGN>::MIN_CTAS};
}

}  // namespace dbp
