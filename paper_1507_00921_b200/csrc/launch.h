// Per-block-length launchers of the fused kernel (one translation unit per
// log2 N so the big unrolled kernels compile in parallel).
#pragma once
#include <cuda_runtime.h>

#ifdef DBP_KERNEL_V1
#include "dbp_block_kernel_v1.cuh"
#else
#include "dbp_block_kernel.cuh"
#endif

namespace dbp {

constexpr int kMinLogN = 4;   // N = 16
constexpr int kMaxLogN = 13;  // N = 8192

struct LaunchShape {
  int threads_x;  // threads per CTA along x
  int threads_y;  // along y (v1: one row per block slice)
  int slices;     // block slices per CTA
  int buffers;    // shared buffers per slice (2 = double-buffered exchanges)
};

template <int LOGN>
cudaError_t launch_block_kernel(const KernelParams& kp, long long n_ctas, size_t smem_bytes,
                                cudaStream_t stream);

template <int LOGN>
LaunchShape launch_shape() {
#ifdef DBP_KERNEL_V1
  return LaunchShape{Geo<LOGN>::T, Geo<LOGN>::BPC, Geo<LOGN>::BPC, 1};
#else
  return LaunchShape{Geo<LOGN>::THREADS, 1, Geo<LOGN>::BPC, Geo<LOGN>::DB ? 2 : 1};
#endif
}

}  // namespace dbp
