// Per-block-length launchers of the fused kernel (one translation unit per
// log2 N so the big unrolled kernels compile in parallel).
#pragma once
#include <cuda_runtime.h>

#include "dbp_block_kernel.cuh"

namespace dbp {

constexpr int kMinLogN = 4;   // N = 16
constexpr int kMaxLogN = 13;  // N = 8192

struct LaunchShape {
  int threads_x;  // threads per CTA along x
  int threads_y;  // along y
  int slices;     // block slices per CTA
  bool separate_fir;  // FIR buffers behind the exchange planes (Geo::SEP_FIR)
  int min_ctas;       // resident CTAs per SM the kernel is built for (Geo::MIN_CTAS)
};

template <int LOGN>
cudaError_t launch_block_kernel(const KernelParams& kp, long long n_ctas, size_t smem_bytes,
                                cudaStream_t stream);

struct SimParams;

template <int LOGN>
cudaError_t launch_ssfm_row(const SimParams& sp, long long n_ctas, size_t smem_bytes, cudaStream_t stream,
                            bool column);

template <int LOGN>
LaunchShape launch_shape() {
  return LaunchShape{Geo<LOGN>::THREADS, 1, Geo<LOGN>::BPC, Geo<LOGN>::SEP_FIR, Geo<LOGN>::MIN_CTAS};
}

}  // namespace dbp
