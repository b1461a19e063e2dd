// Float64 DFT utility (dbp_fft_c2c, include/dbp_b200.h): the reference's
// spectral.fft / spectral.ifft (pkg/src/fiberdbp/spectral.py:37-48, numpy
// pocketfft along the last axis, inverse scaled by 1/n) on the repo's own
// float64 Stockham FFT (fft64.cuh; no cuFFT in the product library).  Not on
// the DBP path (the block kernel has its own FFT); it completes the spectral
// module's API for callers of the drop-in.
#include <cuda_runtime.h>

#include "fft64.cuh"

#include <mutex>
#include <string>

#include "../../include/dbp_b200.h"

namespace dbp_capi_internal {
int fail(int code, const std::string& msg);
void add_launches(long long n);
}
using dbp_capi_internal::fail;

namespace {

// phi = cumsum(incr) over one block of 1024 threads (contiguous chunks, then
// a scan of the chunk sums); out = in * exp(j phi) for both polarisations
__global__ void phase_noise_kernel(const double2* __restrict__ in, const double* __restrict__ incr,
                                   double2* __restrict__ out, long long n) {
  __shared__ double part[1024];
  const long long chunk = (n + blockDim.x - 1) / blockDim.x;
  const long long lo = threadIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
  double s = 0.0;
  for (long long k = lo; k < hi; ++k) s += incr[k];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double run = 0.0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      const double v = part[t];
      part[t] = run;
      run += v;
    }
  }
  __syncthreads();
  double phi = part[threadIdx.x];
  for (long long k = lo; k < hi; ++k) {
    phi += incr[k];
    double sn, cs;
    sincos(phi, &sn, &cs);
    const double2 a = in[k], b = in[n + k];
    out[k] = make_double2(a.x * cs - a.y * sn, a.x * sn + a.y * cs);
    out[n + k] = make_double2(b.x * cs - b.y * sn, b.x * sn + b.y * cs);
  }
}

std::mutex g_mu;

}  // namespace

extern "C" int dbp_fft_c2c(int device, const void* h_in, void* h_out, int64_t n, int64_t batch, int inverse) {
  if (!h_in || !h_out) return fail(DBP_EINVAL, "null buffer");
  if (n < 1 || (n & (n - 1))) return fail(DBP_EINVAL, "block length must be a power of two, got " + std::to_string(n));
  if (batch < 1) return fail(DBP_EINVAL, "batch must be >= 1");
  if (n > (1LL << 30) || batch * n > (1LL << 31)) return fail(DBP_EINVAL, "transform too large for one call");
  int prev = -1;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return fail(DBP_ECUDA, "cudaSetDevice failed");
  std::lock_guard<std::mutex> lock(g_mu);
  const size_t bytes = (size_t)batch * n * sizeof(double2);
  double2* d = nullptr;
  int rc = DBP_OK;
  double2* res = nullptr;
  long long launches = 0;
  if (cudaMalloc(&d, 2 * bytes) != cudaSuccess) {
    rc = fail(DBP_ENOMEM, "device allocation failed");
    goto done;
  }
  if (cudaMemcpy(d, h_in, bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
    rc = fail(DBP_ECUDA, "H2D failed");
    goto done;
  }
  res = fft64::transform(d, d + (size_t)batch * n, n, batch, inverse != 0, true, 0, &launches);
  dbp_capi_internal::add_launches(launches);
  if (!res) {
    rc = fail(DBP_ECUDA, "fft64 transform launch failed");
    goto done;
  }
  if (cudaMemcpy(h_out, res, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) rc = fail(DBP_ECUDA, "D2H failed");
done:
  if (d) cudaFree(d);
  if (prev >= 0) cudaSetDevice(prev);
  return rc;
}

extern "C" int dbp_phase_noise(int device, const void* h_in, const double* h_incr, void* h_out, int64_t n) {
  if (!h_in || !h_incr || !h_out || n < 1) return fail(DBP_EINVAL, "invalid phase-noise arguments");
  int prev = -1;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return fail(DBP_ECUDA, "cudaSetDevice failed");
  double2* d = nullptr;
  double* di = nullptr;
  int rc = DBP_OK;
  const size_t bytes = (size_t)2 * n * sizeof(double2);
  if (cudaMalloc(&d, 2 * bytes) != cudaSuccess || cudaMalloc(&di, n * sizeof(double)) != cudaSuccess) {
    rc = fail(DBP_ENOMEM, "device allocation failed");
  } else if (cudaMemcpy(d, h_in, bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
             cudaMemcpy(di, h_incr, n * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
    rc = fail(DBP_ECUDA, "H2D failed");
  } else {
    phase_noise_kernel<<<1, 1024>>>(d, di, d + 2 * n, n);
    dbp_capi_internal::add_launches(1);
    if (cudaGetLastError() != cudaSuccess || cudaMemcpy(h_out, d + 2 * n, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
      rc = fail(DBP_ECUDA, "phase_noise_kernel failed");
  }
  if (d) cudaFree(d);
  if (di) cudaFree(di);
  if (prev >= 0) cudaSetDevice(prev);
  return rc;
}
