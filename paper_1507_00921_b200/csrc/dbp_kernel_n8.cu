// Instantiation of the fused DBP block kernel for N = 2^8.
#include "launch.h"
#include "ssfm_kernels.cuh"

namespace dbp {

template <>
cudaError_t launch_block_kernel<8>(const KernelParams& kp, long long n_ctas, size_t smem_bytes,
                                    cudaStream_t stream) {
  return launch_block_kernel_impl<8>(kp, n_ctas, smem_bytes, stream);
}

template <>
cudaError_t launch_ssfm_row<8>(const SimParams& sp, long long n_ctas, size_t smem_bytes, cudaStream_t stream,
                                bool column) {
  using G = Geo<8>;
  if (column) {
    smem_bytes = col_smem_bytes<8>(smem_bytes);
    if (smem_bytes > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(ssfm_row_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem_bytes);
      if (e != cudaSuccess) return e;
    }
    ssfm_row_kernel<8, true><<<dim3((unsigned)n_ctas), dim3(SimShape<8, true>::THREADS), smem_bytes,
                                  stream>>>(sp);
    return cudaGetLastError();
  }
  if (smem_bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(ssfm_row_kernel<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem_bytes);
    if (e != cudaSuccess) return e;
  }
  ssfm_row_kernel<8, false><<<dim3((unsigned)n_ctas), dim3(G::THREADS), smem_bytes, stream>>>(sp);
  return cudaGetLastError();
}

}  // namespace dbp
