// The nonlinear sub-steps as standalone operators on ONE (2, n) block of any
// length (dbp.py:49-75 nonlinear_substep_essfm, channel.py:61-71
// nonlinear_substep_ssfm): float64 like the reference, cyclic FIR indices
// inside the block, block * exp(-j gamma dz_eff F).  The DBP path applies the
// same operator inside the fused block kernel (float32, power-of-two N); this
// entry point serves the reference's sub-step API for any n > 2 N_c.
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "../../include/dbp_b200.h"

namespace dbp_capi_internal {
int fail(int code, const std::string& msg);
void add_launches(long long n);
}
using dbp_capi_internal::fail;

namespace {

__global__ void intensity_kernel(const double2* __restrict__ blk, double* __restrict__ inten, long long n) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double2 x = blk[k], y = blk[n + k];
  const double ax = hypot(x.x, x.y), ay = hypot(y.x, y.y);   // numpy's abs(z) ** 2
  inten[k] = ax * ax + ay * ay;
}

// F_k = c0 I_k + sum_i c_i (I_{k-i} + I_{k+i}), in the reference's summation
// order; out = blk * exp(j phi), phi = -gamma dz_eff F
__global__ void rotate_kernel(const double2* __restrict__ blk, const double* __restrict__ inten,
                              const double* __restrict__ c, int nc, double a, double2* __restrict__ out,
                              long long n) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  double f = __dmul_rn(c[0], inten[k]);
  for (int i = 1; i <= nc; ++i) {
    long long lo = k - i, hi = k + i;
    if (lo < 0) lo += n;
    if (hi >= n) hi -= n;
    f = __dadd_rn(f, __dmul_rn(c[i], __dadd_rn(inten[lo], inten[hi])));
  }
  double s, co;
  sincos(__dmul_rn(a, f), &s, &co);
  const double2 x = blk[k], y = blk[n + k];
  out[k] = make_double2(x.x * co - x.y * s, x.x * s + x.y * co);
  out[n + k] = make_double2(y.x * co - y.y * s, y.x * s + y.y * co);
}

}  // namespace

extern "C" int dbp_nonlinear_substep_c128(int device, const void* h_block, void* h_out, int64_t n, double gamma,
                                          double dz_eff, const double* coeffs, int n_coeffs) {
  if (!h_block || !h_out || !coeffs) return fail(DBP_EINVAL, "null buffer");
  if (n < 1) return fail(DBP_EINVAL, "block must contain at least one sample");
  if (n_coeffs < 0) return fail(DBP_EINVAL, "n_coeffs must be >= 0");
  if (n <= 2LL * n_coeffs)
    return fail(DBP_EINVAL, "block length " + std::to_string(n) + " too short for " + std::to_string(n_coeffs) +
                                " side coefficients");
  if (!std::isfinite(gamma) || !std::isfinite(dz_eff)) return fail(DBP_EINVAL, "gamma and dz_eff must be finite");
  for (int i = 0; i <= n_coeffs; ++i)
    if (!std::isfinite(coeffs[i])) return fail(DBP_EINVAL, "coefficients must be finite");
  int prev = -1;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return fail(DBP_ECUDA, "cudaSetDevice failed");
  const size_t bytes = (size_t)2 * n * sizeof(double2);
  double2* d = nullptr;
  double* di = nullptr;
  double* dc = nullptr;
  int rc = DBP_OK;
  if (cudaMalloc(&d, 2 * bytes) != cudaSuccess || cudaMalloc(&di, n * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&dc, (n_coeffs + 1) * sizeof(double)) != cudaSuccess) {
    rc = fail(DBP_ENOMEM, "device allocation failed");
  } else if (cudaMemcpy(d, h_block, bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
             cudaMemcpy(dc, coeffs, (n_coeffs + 1) * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
    rc = fail(DBP_ECUDA, "H2D failed");
  } else {
    const unsigned blocks = (unsigned)((n + 255) / 256);
    intensity_kernel<<<blocks, 256>>>(d, di, n);
    // reference: block * exp(-1j * gamma * dz_eff * F)
    rotate_kernel<<<blocks, 256>>>(d, di, dc, n_coeffs, -gamma * dz_eff, d + 2 * n, n);
    dbp_capi_internal::add_launches(2);
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpy(h_out, d + 2 * n, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
      rc = fail(DBP_ECUDA, "nonlinear sub-step kernel failed");
  }
  cudaFree(d);
  cudaFree(di);
  cudaFree(dc);
  if (prev >= 0) cudaSetDevice(prev);
  return rc;
}
