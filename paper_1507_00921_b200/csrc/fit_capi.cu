// Device-side residual algebra of the ESSFM coefficient fit:
// dbp_fit_* in include/dbp_b200.h.
//
// Reference: pkg/src/fiberdbp/train.py:130-178 -- residual(c) = (DBP_c(x) -
// target)[window] / ||target[window]||, a forward-difference Jacobian and
// numpy.linalg.lstsq for the Gauss-Newton step, squared errors for the line
// search.  The GPU fit (training.py) keeps the DBP outputs of every
// coefficient set on the device and reduces them here: per-set squared
// residual norms for the line search, and the Gauss-Newton normal equations
// J^T J, J^T r (float64, central differences) for the step, so only
// (P + 1) P numbers cross PCIe per iteration instead of the outputs.
// Reductions are two-stage with a fixed order (deterministic).
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/dbp_b200.h"

namespace dbp_capi_internal {
int fail(int code, const std::string& msg);
void add_launches(long long n);
}
using dbp_capi_internal::fail;

#define FIT_CUDA(expr, what)                                                                      \
  do {                                                                                            \
    cudaError_t e_ = (expr);                                                                      \
    if (e_ != cudaSuccess) return fail(DBP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace fit {

constexpr int kThreads = 256;
constexpr int kMaxP = 65;              // n_coeffs <= 64
constexpr int kRows = 128;             // residual rows per block in the normal-equation kernel

// partial[s][blk] = sum over this block's samples of |(out_s - target) scale|^2
__global__ void sumsq_partial(const float2* __restrict__ out, long long n, const float2* __restrict__ target,
                              long long w0, long long w, double scale, double* __restrict__ partial) {
  __shared__ double sh[kThreads / 32];
  const int s = blockIdx.y;
  const float2* o = out + (long long)s * 2 * n;
  double acc = 0.0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < 2 * w; k += (long long)gridDim.x * blockDim.x) {
    const long long pol = k / w, idx = w0 + (k - pol * w);
    const float2 a = o[pol * n + idx], t = target[pol * n + idx];
    const double dr = ((double)a.x - (double)t.x) * scale, di = ((double)a.y - (double)t.y) * scale;
    acc += dr * dr + di * di;
  }
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) v += sh[i];
    partial[(long long)s * gridDim.x + blockIdx.x] = v;
  }
}

// sums[s] = sum_b partial[s][b] in block order
__global__ void reduce_rows(const double* __restrict__ partial, int cols, int rows, double* __restrict__ sums) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double v = 0.0;
  for (int c = 0; c < cols; ++c) v += partial[(long long)r * cols + c];
  sums[r] = v;
}

// Normal equations over kRows residual rows per block: row k (2 pols x w
// samples x re/im) has J_i = part((out_{+i} - out_{-i}) scale / (2 h)) and
// r = part((base - target) scale).  partial[blk][q] for the P (P + 1) / 2
// upper-triangle products then the P products with r.
__global__ void normal_partial(const float2* __restrict__ out, int P, long long n, const float2* __restrict__ target,
                               const float2* __restrict__ base, long long w0, long long w, double scale, double inv2h,
                               double* __restrict__ partial, int n_terms) {
  extern __shared__ double js[];   // [kRows][P + 1]
  const long long rows = 4 * w;
  const long long r0 = (long long)blockIdx.x * kRows;
  const int stride = P + 1;
  for (int e = threadIdx.x; e < kRows * stride; e += blockDim.x) {
    const int rr = e / stride, col = e - rr * stride;
    const long long k = r0 + rr;
    double v = 0.0;
    if (k < rows) {
      const long long smp = k >> 1, pol = smp / w, idx = w0 + (smp - pol * w);
      const bool im = k & 1;
      if (col < P) {
        const float2 a = out[((long long)col * 2 + pol) * n + idx];
        const float2 b = out[((long long)(P + col) * 2 + pol) * n + idx];
        v = ((double)(im ? a.y : a.x) - (double)(im ? b.y : b.x)) * scale * inv2h;
      } else {
        const float2 a = base[pol * n + idx], t = target[pol * n + idx];
        v = ((double)(im ? a.y : a.x) - (double)(im ? t.y : t.x)) * scale;
      }
    }
    js[e] = v;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < n_terms; q += blockDim.x) {
    int i, j;
    const int tri = P * (P + 1) / 2;
    if (q < tri) {   // upper triangle, row-major: (i, j), j >= i
      i = 0;
      int rem = q;
      while (rem >= P - i) {
        rem -= P - i;
        ++i;
      }
      j = i + rem;
    } else {         // J^T r
      i = q - tri;
      j = P;
    }
    double acc = 0.0;
    for (int rr = 0; rr < kRows; ++rr) acc += js[rr * stride + i] * js[rr * stride + j];
    partial[(long long)blockIdx.x * n_terms + q] = acc;
  }
}

// column sums of partial[blocks][terms] in block order
__global__ void reduce_cols(const double* __restrict__ partial, int blocks, int terms, double* __restrict__ sums) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= terms) return;
  double v = 0.0;
  for (int b = 0; b < blocks; ++b) v += partial[(long long)b * terms + q];
  sums[q] = v;
}

}  // namespace fit

namespace {

int check_window(int64_t n_total, int64_t w0, int64_t w1) {
  if (n_total < 1 || w0 < 0 || w1 <= w0 || w1 > n_total) return fail(DBP_EINVAL, "fit window outside the signal");
  return DBP_OK;
}

}  // namespace

extern "C" {

int dbp_fit_sumsq(const void* d_out, int n_sets, int64_t n_total, const void* d_target, int64_t w0, int64_t w1,
                  double scale, double* h_sums, void* stream) {
  if (!d_out || !d_target || !h_sums || n_sets < 1) return fail(DBP_EINVAL, "invalid fit arguments");
  int rc = check_window(n_total, w0, w1);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long w = w1 - w0;
  int blocks = (int)((2 * w + fit::kThreads * 8 - 1) / (fit::kThreads * 8));
  if (blocks > 1024) blocks = 1024;
  double* d_part = nullptr;
  FIT_CUDA(cudaMallocAsync(&d_part, ((size_t)n_sets * blocks + n_sets) * sizeof(double), st), "cudaMallocAsync");
  fit::sumsq_partial<<<dim3(blocks, n_sets), fit::kThreads, 0, st>>>(static_cast<const float2*>(d_out), n_total,
                                                                     static_cast<const float2*>(d_target), w0, w,
                                                                     scale, d_part);
  double* d_sums = d_part + (size_t)n_sets * blocks;
  fit::reduce_rows<<<(n_sets + 127) / 128, 128, 0, st>>>(d_part, blocks, n_sets, d_sums);
  dbp_capi_internal::add_launches(2);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(h_sums, d_sums, n_sets * sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_part, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  FIT_CUDA(e, "dbp_fit_sumsq");
  return DBP_OK;
}

int dbp_fit_normal(const void* d_out, int n_params, int64_t n_total, const void* d_target, const void* d_base,
                   int64_t w0, int64_t w1, double scale, double fd_step, double* h_ata, double* h_atr,
                   void* stream) {
  if (!d_out || !d_target || !d_base || !h_ata || !h_atr) return fail(DBP_EINVAL, "invalid fit arguments");
  if (n_params < 1 || n_params > fit::kMaxP) return fail(DBP_EINVAL, "n_params outside [1, 65]");
  if (!(fd_step > 0.0)) return fail(DBP_EINVAL, "fd_step must be positive");
  int rc = check_window(n_total, w0, w1);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int P = n_params;
  const int tri = P * (P + 1) / 2, terms = tri + P;
  const long long w = w1 - w0, rows = 4 * w;
  const int blocks = (int)((rows + fit::kRows - 1) / fit::kRows);
  const size_t smem = (size_t)fit::kRows * (P + 1) * sizeof(double);
  if (smem > 48 * 1024)
    FIT_CUDA(cudaFuncSetAttribute(fit::normal_partial, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
             "cudaFuncSetAttribute");
  double* d_part = nullptr;
  FIT_CUDA(cudaMallocAsync(&d_part, ((size_t)blocks * terms + terms) * sizeof(double), st), "cudaMallocAsync");
  fit::normal_partial<<<blocks, fit::kThreads, smem, st>>>(static_cast<const float2*>(d_out), P, n_total,
                                                           static_cast<const float2*>(d_target),
                                                           static_cast<const float2*>(d_base), w0, w, scale,
                                                           0.5 / fd_step, d_part, terms);
  double* d_sums = d_part + (size_t)blocks * terms;
  fit::reduce_cols<<<(terms + 127) / 128, 128, 0, st>>>(d_part, blocks, terms, d_sums);
  dbp_capi_internal::add_launches(2);
  std::vector<double> sums(terms);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(sums.data(), d_sums, terms * sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_part, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  FIT_CUDA(e, "dbp_fit_normal");
  int q = 0;
  for (int i = 0; i < P; ++i)
    for (int j = i; j < P; ++j, ++q) {
      h_ata[i * P + j] = sums[q];
      h_ata[j * P + i] = sums[q];
    }
  for (int i = 0; i < P; ++i) h_atr[i] = sums[tri + i];
  return DBP_OK;
}

}  // extern "C"
