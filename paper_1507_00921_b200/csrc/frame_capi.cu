// Overlap-save framing as standalone device operators, for block processors
// the fused kernel cannot run (the reference's overlap_save_run accepts any
// callable, spectral.py:84-92): frame = cyclic extension + cut into blocks
// (spectral.py:122-131: lead = M // 2, idx = arange(-lead, nb step + N - lead)
// % n, block b = ext[:, b step : b step + N]); unframe = keep the centre of
// each processed block (spectral.py:138-145: out[:, b step : (b + 1) step] =
// blk[:, lead : lead + step], trimmed to n).  Pure data movement, so any
// element width works bit-exactly: 8 bytes (complex64) or 16 (complex128, the
// reference's own dtype).  HBM-bound copies: one 16-byte element (or two
// 8-byte ones) per thread-iteration, consecutive threads on consecutive
// samples of a block row, grid sized to the SM count.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/dbp_b200.h"

namespace dbp_capi_internal {
int fail(int code, const std::string& msg);
void add_launches(long long n);
}
using dbp_capi_internal::fail;

namespace {

// blocks[item][b][pol][j] = sig[item][pol][(b0 + b) step - lead + j mod n]
template <class E>
__global__ void frame_kernel(const E* __restrict__ sig, E* __restrict__ blocks, long long n, int N, int step,
                             int lead, long long b0, long long nblk, long long total) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += stride) {
    const int j = (int)(o % N);
    const long long row = o / N;          // (item, b, pol)
    const int pol = (int)(row & 1);
    const long long ib = row >> 1;        // item * nblk + b
    const long long item = ib / nblk, b = ib - item * nblk;
    long long src = ((b0 + b) * step - lead + j) % n;
    if (src < 0) src += n;
    blocks[o] = __ldg(sig + (item * 2 + pol) * n + src);
  }
}

// out[item][pol][k] = blocks[item][k / step - b0][pol][lead + k % step] for
// k in [b0 step, min(n, b1 step))
template <class E>
__global__ void unframe_kernel(const E* __restrict__ blocks, E* __restrict__ out, long long n, int N, int step,
                               int lead, long long b0, long long nblk, long long k0, long long klen,
                               long long total) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += stride) {
    const long long r = o / klen, kk = o - r * klen;   // r = item * 2 + pol
    const long long item = r >> 1;
    const int pol = (int)(r & 1);
    const long long k = k0 + kk;
    const long long b = k / step;
    const int i = (int)(k - b * step);
    out[r * n + k] = __ldg(blocks + ((item * nblk + (b - b0)) * 2 + pol) * N + lead + i);
  }
}

int grid_for(long long total, int threads, int device) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const long long want = (total + threads - 1) / threads;
  const long long cap = (long long)sms * 8;     // 8 x 256-thread CTAs per SM, grid-stride beyond
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

int check_geometry(int64_t n_total, int batch, int N, int M, int64_t b0, int64_t b1, int elem_bytes,
                   int64_t* nb) {
  if (N < 1 || (N & (N - 1)) != 0) return fail(DBP_EINVAL, "block length must be a power of two");
  if (M < 0 || M >= N) return fail(DBP_EINVAL, "overlap must satisfy 0 <= overlap < block length");
  if (n_total < 1) return fail(DBP_EINVAL, "signal must contain at least one sample");
  if (batch < 0) return fail(DBP_EINVAL, "batch must be >= 0");
  if (elem_bytes != 8 && elem_bytes != 16) return fail(DBP_EINVAL, "elem_bytes must be 8 (complex64) or 16 (complex128)");
  const int step = N - M;
  *nb = (n_total + step - 1) / step;
  if (b0 < 0 || b1 < b0 || b1 > *nb) return fail(DBP_EINVAL, "block range out of bounds");
  return DBP_OK;
}

}  // namespace

extern "C" int dbp_frame_blocks(const void* d_sig, void* d_blocks, int64_t n_total, int batch, int block_len,
                                int overlap, int64_t block_begin, int64_t block_end, int elem_bytes,
                                void* stream) {
  int64_t nb = 0;
  int rc = check_geometry(n_total, batch, block_len, overlap, block_begin, block_end, elem_bytes, &nb);
  if (rc) return rc;
  const long long nblk = block_end - block_begin;
  const long long total = (long long)batch * nblk * 2 * block_len;
  if (total == 0) return DBP_OK;
  if (!d_sig || !d_blocks) return fail(DBP_EINVAL, "null device buffer");
  int dev = 0;
  cudaGetDevice(&dev);
  const int step = block_len - overlap, lead = overlap / 2;
  const int threads = 256, grid = grid_for(total, threads, dev);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (elem_bytes == 8)
    frame_kernel<float2><<<grid, threads, 0, s>>>(static_cast<const float2*>(d_sig), static_cast<float2*>(d_blocks),
                                                  n_total, block_len, step, lead, block_begin, nblk, total);
  else
    frame_kernel<double2><<<grid, threads, 0, s>>>(static_cast<const double2*>(d_sig),
                                                   static_cast<double2*>(d_blocks), n_total, block_len, step,
                                                   lead, block_begin, nblk, total);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DBP_ECUDA, std::string("frame_kernel: ") + cudaGetErrorString(e));
  dbp_capi_internal::add_launches(1);
  return DBP_OK;
}

extern "C" int dbp_unframe_blocks(const void* d_blocks, void* d_out, int64_t n_total, int batch, int block_len,
                                  int overlap, int64_t block_begin, int64_t block_end, int elem_bytes,
                                  void* stream) {
  int64_t nb = 0;
  int rc = check_geometry(n_total, batch, block_len, overlap, block_begin, block_end, elem_bytes, &nb);
  if (rc) return rc;
  const int step = block_len - overlap, lead = overlap / 2;
  const long long k0 = (long long)block_begin * step;
  long long k1 = (long long)block_end * step;
  if (k1 > n_total) k1 = n_total;
  const long long klen = k1 - k0;
  const long long total = (long long)batch * 2 * (klen > 0 ? klen : 0);
  if (total == 0) return DBP_OK;
  if (!d_blocks || !d_out) return fail(DBP_EINVAL, "null device buffer");
  int dev = 0;
  cudaGetDevice(&dev);
  const long long nblk = block_end - block_begin;
  const int threads = 256, grid = grid_for(total, threads, dev);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (elem_bytes == 8)
    unframe_kernel<float2><<<grid, threads, 0, s>>>(static_cast<const float2*>(d_blocks),
                                                    static_cast<float2*>(d_out), n_total, block_len, step, lead,
                                                    block_begin, nblk, k0, klen, total);
  else
    unframe_kernel<double2><<<grid, threads, 0, s>>>(static_cast<const double2*>(d_blocks),
                                                     static_cast<double2*>(d_out), n_total, block_len, step,
                                                     lead, block_begin, nblk, k0, klen, total);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DBP_ECUDA, std::string("unframe_kernel: ") + cudaGetErrorString(e));
  dbp_capi_internal::add_launches(1);
  return DBP_OK;
}
