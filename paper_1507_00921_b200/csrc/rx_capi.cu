// Post-DBP receiver DSP on the GPU: dbp_rx_* in include/dbp_b200.h.
//
// Reference: pkg/src/fiberdbp/modem.py -- butterfly_equalize / _cma_pass
// (:183-271), carrier_recover / _vv_phase (:274-351), qpsk_decide (:116-125),
// measure_ber (:358-413) -- chained as cli.py:677-685.  Float64 throughout,
// like the reference, so equalised symbols agree to ~1e-12 and decisions,
// shifts and error counts are identical.
//
// The equaliser is an adaptive filter whose taps change after every output
// symbol: sequential within a waveform, so one warp owns one waveform (a
// batch of waveforms fills the GPU).  The x and y outputs are computed by
// the two half-warps (lane j holds taps j, j + 16, ... of the filter pair
// feeding that output); one symbol costs a 4-level half-warp butterfly
// reduction plus the tap update, with the next symbol's inputs prefetched.
// Spectral searches (4th-power frequency peak, reference and bit-alignment
// correlations) are float64 Stockham transforms (fft64.cuh, no cuFFT) followed
// by arg-max kernels; the sliding-window phase estimate, the unwrap prefix scan,
// decisions and error counting are elementwise / reduction kernels.
#include <cuda_runtime.h>
#include "fft64.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "../../include/dbp_b200.h"

namespace dbp_capi_internal {
int fail(int code, const std::string& msg);
void add_launches(long long n);
}
using dbp_capi_internal::fail;
#define RX_LAUNCHED() dbp_capi_internal::add_launches(1)

#define RX_CUDA(expr, what)                                                                      \
  do {                                                                                           \
    cudaError_t e_ = (expr);                                                                     \
    if (e_ != cudaSuccess) return fail(DBP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace rx {

constexpr double kPi = 3.14159265358979311600;   // == numpy.pi
constexpr double kSqrt1_2 = 0.70710678118654757; // == 1 / math.sqrt(2.0) (modem.py:31)

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// block-wide sum of NV doubles (blockDim.x a multiple of 32, <= 1024)
template <int NV>
__device__ void block_sum(double (&v)[NV], double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i)
    for (int o = 16; o; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  __syncthreads();
  if (lane == 0)
    for (int i = 0; i < NV; ++i) sh[w * NV + i] = v[i];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < NV; ++i) {
      double s = 0.0;
      for (int k = 0; k < nw; ++k) s += sh[k * NV + i];
      v[i] = s;
    }
}

// per-waveform mean power of the dual-pol input, (|x|^2 + |y|^2) / 2 averaged (modem.py:236)
__global__ void power_kernel(const double2* __restrict__ in, long long n, double* __restrict__ p) {
  __shared__ double sh[32];
  const double2* x = in + (long long)blockIdx.x * 2 * n;
  double v[1] = {0.0};
  for (long long k = threadIdx.x; k < n; k += blockDim.x) {
    const double2 a = x[k], b = x[n + k];
    v[0] += a.x * a.x + a.y * a.y + b.x * b.x + b.y * b.y;
  }
  block_sum<1>(v, sh);
  if (threadIdx.x == 0) p[blockIdx.x] = v[0] / (double)n / 2.0;
}

// circularly padded, power-normalised equaliser input (modem.py:240-243)
__global__ void ext_kernel(const double2* __restrict__ in, long long n, int half, const double* __restrict__ p,
                           double2* __restrict__ ext, long long ext_len, int batch) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ext_len * 2 * batch) return;
  const long long plane = i / ext_len, k = i - plane * ext_len;
  const double g = 1.0 / sqrt(p[plane >> 1]);
  long long s = (k - half) % n;
  if (s < 0) s += n;
  const double2 v = in[plane * n + s];
  ext[i] = make_double2(v.x * g, v.y * g);
}

// One CMA sweep (modem.py:183-204) over the waveforms listed in ``items``:
// warp w owns waveform items[w]; half-warp h computes output h (x, y) with
// taps (h_{h x}, h_{h y}); lane j holds taps j + 16 k, k < K.
constexpr int kCmaChunk = 32;                     // symbols per staged chunk
constexpr int kCmaWin = 2 * kCmaChunk + 64;       // samples per polarisation window (taps <= 64)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}

// One CMA sweep (modem.py:183-204) over the waveforms listed in ``items``:
// warp w owns waveform items[w]; half-warp h computes output h (x, y) with
// taps (h_{h x}, h_{h y}); lane j holds taps j + 16 k, k < K.  The input
// window of the next 32 symbols is staged into shared memory with cp.async
// while the current chunk runs, so the per-symbol recursion only sees
// shared-memory latency (an L2 round trip is longer than one symbol update).
template <int K>
__global__ void __launch_bounds__(128) cma_kernel(const double2* __restrict__ ext, long long ext_len,
                                                  double2* __restrict__ taps_buf, int taps, double mu,
                                                  long long m, double2* __restrict__ out,
                                                  const int* __restrict__ items, int n_items) {
  __shared__ double2 win[4][2][2][kCmaWin];   // [warp][buffer][pol][sample]
  __shared__ double2 zero_col[2 * kCmaChunk + 2];   // read by lanes beyond the tap count
  const int w = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
  for (int e = threadIdx.x; e < 2 * kCmaChunk + 2; e += blockDim.x) zero_col[e] = make_double2(0.0, 0.0);
  __syncthreads();
  if (w >= n_items) return;
  const int b = items[w];
  const int lane = threadIdx.x & 31, h = lane >> 4, j = lane & 15, wl = threadIdx.x >> 5;
  const double2* ex = ext + (long long)b * 2 * ext_len;
  double2* tb = taps_buf + (long long)b * 4 * taps;
  double2 h1[K], h2[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int i = j + 16 * k;
    const bool ok = i < taps;
    h1[k] = ok ? tb[(2 * h) * taps + i] : make_double2(0.0, 0.0);
    h2[k] = ok ? tb[(2 * h + 1) * taps + i] : make_double2(0.0, 0.0);
  }
  double2* o = out + ((long long)b * 2 + h) * m;
  const long long nch = (m + kCmaChunk - 1) / kCmaChunk;
  auto stage = [&](long long c) {   // ext[2 c CH, + 2 CH + taps - 1) of both polarisations -> buffer c & 1
    const long long s0 = 2 * c * kCmaChunk;
    long long len = 2 * kCmaChunk + taps - 1;
    if (s0 + len > ext_len) len = ext_len - s0;
    for (int e = lane; e < 2 * len; e += 32) {
      const int pl = e >= len ? 1 : 0;
      const int r = pl ? (int)(e - len) : e;
      cp_async16(&win[wl][c & 1][pl][r], ex + pl * ext_len + s0 + r);
    }
  };
  stage(0);
  asm volatile("cp.async.commit_group;");
  for (long long c = 0; c < nch; ++c) {
    if (c + 1 < nch) stage(c + 1);
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 1;");
    __syncwarp();
    const long long n0 = c * kCmaChunk;
    const int cnt = (int)(m - n0 < kCmaChunk ? m - n0 : kCmaChunk);
    // per-tap column pointers: real taps read the window, the rest a zero column
    // (no per-symbol predicates; the read one symbol past a chunk is never used)
    const double2* px[K];
    const double2* py[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int i = j + 16 * k;
      px[k] = i < taps ? win[wl][c & 1][0] + i : zero_col;
      py[k] = i < taps ? win[wl][c & 1][1] + i : zero_col;
    }
    double2 ux[K], uy[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      ux[k] = px[k][0];
      uy[k] = py[k][0];
    }
    for (int n = 0; n < cnt; ++n) {
      double2 nx[K], ny[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        nx[k] = px[k][2 * (n + 1)];
        ny[k] = py[k][2 * (n + 1)];
      }
      double ar = 0.0, ai = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        ar += (h1[k].x * ux[k].x - h1[k].y * ux[k].y) + (h2[k].x * uy[k].x - h2[k].y * uy[k].y);
        ai += (h1[k].x * ux[k].y + h1[k].y * ux[k].x) + (h2[k].x * uy[k].y + h2[k].y * uy[k].x);
      }
#pragma unroll
      for (int off = 8; off; off >>= 1) {
        ar += __shfl_xor_sync(0xffffffffu, ar, off);
        ai += __shfl_xor_sync(0xffffffffu, ai, off);
      }
      const double a = mu * (1.0 - (ar * ar + ai * ai));
      const double er = a * ar, ei = a * ai;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        h1[k].x += er * ux[k].x + ei * ux[k].y;   // e * conj(u)
        h1[k].y += ei * ux[k].x - er * ux[k].y;
        h2[k].x += er * uy[k].x + ei * uy[k].y;
        h2[k].y += ei * uy[k].x - er * uy[k].y;
        ux[k] = nx[k];
        uy[k] = ny[k];
      }
      if (j == 0) o[n0 + n] = make_double2(ar, ai);
    }
    __syncwarp();   // every lane is done with this buffer before it is refilled
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int i = j + 16 * k;
    if (i < taps) {
      tb[(2 * h) * taps + i] = h1[k];
      tb[(2 * h + 1) * taps + i] = h2[k];
    }
  }
}

__global__ void init_taps_kernel(double2* __restrict__ taps_buf, int taps, int batch) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= batch * 4 * taps) return;
  const int f = (i / taps) & 3, t = i % taps;   // filters hxx, hxy, hyx, hyy
  const bool centre = t == taps / 2 && (f == 0 || f == 3);
  taps_buf[i] = make_double2(centre ? 1.0 : 0.0, 0.0);
}

// collapsed-output re-initialisation (modem.py:262-264): h_yy = conj(rev h_xx), h_yx = -conj(rev h_xy)
__global__ void reinit_kernel(double2* __restrict__ taps_buf, int taps, const int* __restrict__ items, int n_items) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_items * taps) return;
  double2* tb = taps_buf + (long long)items[i / taps] * 4 * taps;
  const int t = i % taps;
  const double2 xx = tb[taps - 1 - t], xy = tb[taps + taps - 1 - t];
  tb[3 * taps + t] = make_double2(xx.x, -xx.y);
  tb[2 * taps + t] = make_double2(-xy.x, xy.y);
}

// (vdot(x, y), vdot(x, x), vdot(y, y)) per waveform (modem.py:259-261)
__global__ void xcorr_kernel(const double2* __restrict__ s, long long m, double* __restrict__ r) {
  __shared__ double sh[32 * 4];
  const double2* x = s + (long long)blockIdx.x * 2 * m;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (long long k = threadIdx.x; k < m; k += blockDim.x) {
    const double2 a = x[k], b = x[m + k];
    v[0] += a.x * b.x + a.y * b.y;   // conj(a) b
    v[1] += a.x * b.y - a.y * b.x;
    v[2] += a.x * a.x + a.y * a.y;
    v[3] += b.x * b.x + b.y * b.y;
  }
  block_sum<4>(v, sh);
  if (threadIdx.x == 0)
    for (int i = 0; i < 4; ++i) r[blockIdx.x * 4 + i] = v[i];
}

// s^4 (numpy complex power: (s^2)^2)
__global__ void pow4_kernel(const double2* __restrict__ s, double2* __restrict__ q, long long total) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const double2 a = s[i];
  const double2 a2 = cmul(a, a);
  q[i] = cmul(a2, a2);
}

// Arg-max of a per-index score with numpy's first-index tie rule; one block
// per problem.  mode 0: |F0|^2 + |F1|^2 of two spectra (modem.py:314);
// mode 1: |c| of one sequence; mode 2: Re c.  Writes (index, value) and,
// for mode 0, the scores at index -1 and +1 (circular).
__device__ __forceinline__ double score(const double2* a, const double2* b, long long k, int mode) {
  if (mode == 0) {
    const double u = hypot(a[k].x, a[k].y), v = hypot(b[k].x, b[k].y);
    return u * u + v * v;
  }
  if (mode == 1) return hypot(a[k].x, a[k].y);
  return a[k].x;
}

__global__ void argmax_kernel(const double2* __restrict__ data, long long m, long long stride_a, long long stride_b,
                              int mode, long long* __restrict__ idx_out, double* __restrict__ val_out) {
  __shared__ double sv[32];
  __shared__ long long si[32];
  const double2* a = data + blockIdx.x * stride_a;
  const double2* b = a + stride_b;
  double best = -INFINITY;
  long long bi = m;
  for (long long k = threadIdx.x; k < m; k += blockDim.x) {
    const double v = score(a, b, k, mode);
    if (v > best) {   // strictly greater: keeps the first index per thread
      best = v;
      bi = k;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (sv[k] > best || (sv[k] == best && si[k] < bi)) {
        best = sv[k];
        bi = si[k];
      }
    idx_out[blockIdx.x] = bi;
    if (mode == 0) {
      val_out[3 * blockIdx.x + 0] = score(a, b, (bi - 1 + m) % m, 0);
      val_out[3 * blockIdx.x + 1] = best;
      val_out[3 * blockIdx.x + 2] = score(a, b, (bi + 1) % m, 0);
    } else if (mode == 1) {
      val_out[2 * blockIdx.x + 0] = a[bi].x;   // the complex value at the peak
      val_out[2 * blockIdx.x + 1] = a[bi].y;
    }
  }
}

// d[k] = s[k] exp(-2 pi j f k / Rs) (modem.py:330-331); per waveform f
__global__ void derotate_kernel(const double2* __restrict__ s, double2* __restrict__ d, long long m, int batch,
                                const double* __restrict__ f_off, double symbol_rate) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * m * batch) return;
  const long long k = i % m;
  const double ang = -2.0 * kPi * f_off[i / (2 * m)] * (double)k / symbol_rate;
  double sn, cs;
  sincos(ang, &sn, &cs);
  d[i] = cmul(s[i], make_double2(cs, sn));
}

// angle of the circular sliding mean of d^4 over ``window`` symbols,
// starting ``pad`` = window / 2 before k (modem.py:274-280)
__global__ void vv_angle_kernel(const double2* __restrict__ d, double* __restrict__ ang, long long m, int planes,
                                int window) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m * planes) return;
  const long long plane = i / m, k = i - plane * m;
  const double2* x = d + plane * m;
  const double inv = 1.0 / (double)window;
  const int pad = window / 2;
  double sr = 0.0, si = 0.0;
  for (int t = 0; t < window; ++t) {
    long long s = (k - pad + t) % m;
    if (s < 0) s += m;
    const double2 a = x[s];
    const double2 a2 = cmul(a, a);
    const double2 q = cmul(a2, a2);
    sr += q.x * inv;
    si += q.y * inv;
  }
  ang[i] = atan2(si, sr);
}

// numpy.unwrap (period 2 pi) as a prefix scan of the per-step corrections,
// then phi = (unwrapped - pi) / 4 and out = d exp(-j phi) (modem.py:280, 333-337).
// One block per polarisation plane; each thread scans a contiguous chunk.
__global__ void unwrap_apply_kernel(const double* __restrict__ ang, const double2* __restrict__ d,
                                    double2* __restrict__ out, long long m) {
  __shared__ double part[1024];
  const long long plane = blockIdx.x;
  const double* p = ang + plane * m;
  const int nt = blockDim.x;
  const long long chunk = (m + nt - 1) / nt;
  const long long lo = threadIdx.x * chunk, hi = lo + chunk < m ? lo + chunk : m;
  auto corr = [&](long long k) -> double {   // correction between k - 1 and k, k >= 1
    const double dd = p[k] - p[k - 1];
    double md = fmod(dd + kPi, 2.0 * kPi);
    if (md < 0.0) md += 2.0 * kPi;
    double ddmod = md - kPi;
    if (ddmod == -kPi && dd > 0.0) ddmod = kPi;
    return fabs(dd) < kPi ? 0.0 : ddmod - dd;
  };
  double s = 0.0;
  for (long long k = lo < 1 ? 1 : lo; k < hi; ++k) s += corr(k);
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double run = 0.0;
    for (int t = 0; t < nt; ++t) {
      const double v = part[t];
      part[t] = run;
      run += v;
    }
  }
  __syncthreads();
  double c = part[threadIdx.x];
  for (long long k = lo; k < hi; ++k) {
    if (k >= 1) c += corr(k);
    const double phi = (p[k] + c - kPi) / 4.0;
    double sn, cs;
    sincos(phi, &sn, &cs);
    out[plane * m + k] = cmul(d[plane * m + k], make_double2(cs, -sn));
  }
}

// out[b][p] *= (-j)^turns[b][p]
__global__ void quarter_turn_kernel(double2* __restrict__ s, long long m, int planes, const int* __restrict__ turns) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m * planes) return;
  const int t = turns[i / m];
  const double ang = -(double)t * kPi / 2.0;
  double sn, cs;
  sincos(ang, &sn, &cs);
  s[i] = cmul(s[i], make_double2(cs, sn));
}

// c[b][p][r][k] = a[b][p][k] * conj(r[r][k]) / m  (ifft normalisation folded in)
__global__ void xspec_kernel(const double2* __restrict__ a, const double2* __restrict__ ref, double2* __restrict__ c,
                             long long m, int batch) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 4 * m * batch) return;
  const long long k = i % m, q = i / m;     // q = (b * 2 + p) * 2 + r
  const int r = (int)(q & 1);
  const long long bp = q >> 1;
  const double2 x = a[bp * m + k], y = ref[r * m + k];
  const double inv = 1.0 / (double)m;
  c[i] = make_double2((x.x * y.x + x.y * y.y) * inv, (x.y * y.x - x.x * y.y) * inv);
}

__global__ void decide_kernel(const double2* __restrict__ s, uint8_t* __restrict__ bits, long long total) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const double2 v = s[i];
  bits[2 * i] = v.x < 0.0;
  bits[2 * i + 1] = v.y < 0.0;
}

// bits -> ((1 - 2 b_I) + j (1 - 2 b_Q)) / sqrt 2 (modem.py:354-355, 112-113)
__global__ void bits_to_symbols_kernel(const uint8_t* __restrict__ bits, double2* __restrict__ s, long long total) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  s[i] = make_double2((1.0 - 2.0 * bits[2 * i]) * kSqrt1_2, (1.0 - 2.0 * bits[2 * i + 1]) * kSqrt1_2);
}

// errors of decided plane (b, p) against reference plane r rolled by shift,
// symbols k >= skip (modem.py:394-399); one block per (b, p, r)
__global__ void count_kernel(const uint8_t* __restrict__ dec, const uint8_t* __restrict__ ref, long long m,
                             long long skip, const long long* __restrict__ shift, long long* __restrict__ errors) {
  __shared__ double sh[32];
  const long long q = blockIdx.x;   // (b * 2 + p) * 2 + r
  const int r = (int)(q & 1);
  const uint8_t* d = dec + (q >> 1) * 2 * m;
  const uint8_t* f = ref + (long long)r * 2 * m;
  const long long sft = shift[q];
  double v[1] = {0.0};
  for (long long k = skip + threadIdx.x; k < m; k += blockDim.x) {
    long long s = (k - sft) % m;
    if (s < 0) s += m;
    v[0] += (double)((d[2 * k] != f[2 * s]) + (d[2 * k + 1] != f[2 * s + 1]));
  }
  block_sum<1>(v, sh);
  if (threadIdx.x == 0) errors[q] = (long long)v[0];
}

// EVM against the scaled nearest constellation point (cli.py:691-695):
// pass 0 sums |s|^2 per waveform; pass 1 sums |s - nearest|^2 and |nearest|^2
__global__ void evm_kernel(const double2* __restrict__ s, long long m, int pass, double* __restrict__ acc) {
  __shared__ double sh[64];
  const double2* x = s + (long long)blockIdx.x * 2 * m;
  double v[2] = {0.0, 0.0};
  const double scale = pass ? sqrt(acc[3 * blockIdx.x] / (double)(2 * m)) : 0.0;
  for (long long k = threadIdx.x; k < 2 * m; k += blockDim.x) {
    const double2 a = x[k];
    if (pass == 0) {
      v[0] += a.x * a.x + a.y * a.y;
    } else {
      const double nr = scale * ((1.0 - 2.0 * (a.x < 0.0)) * kSqrt1_2);
      const double ni = scale * ((1.0 - 2.0 * (a.y < 0.0)) * kSqrt1_2);
      v[0] += (a.x - nr) * (a.x - nr) + (a.y - ni) * (a.y - ni);
      v[1] += nr * nr + ni * ni;
    }
  }
  block_sum<2>(v, sh);
  if (threadIdx.x == 0) {
    if (pass == 0) acc[3 * blockIdx.x] = v[0];
    else {
      acc[3 * blockIdx.x + 1] = v[0];
      acc[3 * blockIdx.x + 2] = v[1];
    }
  }
}

__global__ void widen_kernel(const float2* __restrict__ in, double2* __restrict__ out, long long total) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) out[i] = make_double2(in[i].x, in[i].y);
}

}  // namespace rx

struct dbp_rx {
  int device = 0, max_batch = 0;
  long long m = 0;             // symbols per polarisation
  cudaStream_t stream = nullptr;
  double2* in = nullptr;       // [B][2][2m] samples
  double2* ext = nullptr;      // [B][2][2m + taps - 1]
  long long ext_cap = 0;
  double2* sym = nullptr;      // [B][2][m]
  double2* work = nullptr;     // [B][2][m]
  double2* corr = nullptr;     // [B][2][2][m]
  double2* refs = nullptr;     // [2][m] reference symbols -> spectra
  double2* taps = nullptr;     // [B][4][taps]
  int taps_cap = 0;
  uint8_t* bits = nullptr;     // [B][2][2m]
  uint8_t* ref_bits = nullptr; // [2][2m]
  double* red = nullptr;       // [B][8]
  long long* idx = nullptr;    // [B][4]
  long long* cnt = nullptr;    // [B][4]
  int* items = nullptr;        // [B]
  int* turns = nullptr;        // [B][2]
  double2* fftbuf = nullptr;   // fft64::scratch_elems(m, 4 B): Stockham / Bluestein scratch
};

namespace {

struct Guard {
  int prev = -1;
  explicit Guard(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~Guard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

unsigned blocks(long long n, int t = 256) { return (unsigned)((n + t - 1) / t); }

// float64 DFT of `count` rows of length m (fft64.cuh Stockham, no cuFFT):
// out = F(in) (kForward) or the unnormalised inverse (kInverse), in == out allowed
constexpr int kForward = 0, kInverse = 1;

int fft(dbp_rx* r, double2* in, double2* out, int count, int dir) {
  const size_t bytes = (size_t)count * r->m * sizeof(double2);
  if (in != out) RX_CUDA(cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, r->stream), "D2D(fft)");
  long long launches = 0;
  if (!fft64::transform_any(out, r->fftbuf, r->m, count, dir == kInverse, false, r->stream, &launches))
    return fail(DBP_ECUDA, "fft64 transform launch failed");
  for (long long i = 0; i < launches; ++i) RX_LAUNCHED();
  return DBP_OK;
}

int check_batch(const dbp_rx* r, int batch) {
  if (!r) return fail(DBP_EINVAL, "null receiver");
  if (batch < 1 || batch > r->max_batch) return fail(DBP_EINVAL, "batch outside [1, max_batch]");
  return DBP_OK;
}

// equaliser on r->in (device) -> r->sym; reinits per item (host)
int equalize_dev(dbp_rx* r, int batch, int taps, double mu, int passes, int* reinits) {
  if (taps < 1 || taps % 2 == 0) return fail(DBP_EINVAL, "taps must be odd and positive");
  if (taps > 64) return fail(DBP_EINVAL, "taps above 64 are not supported by the GPU equaliser");
  if (!(mu > 0.0)) return fail(DBP_EINVAL, "step_size must be positive");
  if (passes < 1) return fail(DBP_EINVAL, "passes must be >= 1");
  cudaStream_t st = r->stream;
  const long long n = 2 * r->m, m = r->m;
  const long long ext_len = n + taps - 1;
  if (ext_len > r->ext_cap) {
    cudaFree(r->ext);
    r->ext = nullptr;
    RX_CUDA(cudaMalloc(&r->ext, (size_t)r->max_batch * 2 * ext_len * sizeof(double2)), "cudaMalloc(ext)");
    r->ext_cap = ext_len;
  }
  if (taps > r->taps_cap) {
    cudaFree(r->taps);
    r->taps = nullptr;
    RX_CUDA(cudaMalloc(&r->taps, (size_t)r->max_batch * 4 * taps * sizeof(double2)), "cudaMalloc(taps)");
    r->taps_cap = taps;
  }
  rx::power_kernel<<<batch, 256, 0, st>>>(r->in, n, r->red);
  RX_LAUNCHED();
  std::vector<double> p(batch);
  RX_CUDA(cudaMemcpyAsync(p.data(), r->red, batch * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H(power)");
  RX_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  for (int b = 0; b < batch; ++b)
    if (!(p[b] > 0.0)) return fail(DBP_EINVAL, "cannot equalize an all-zero signal");
  rx::ext_kernel<<<blocks(ext_len * 2 * batch), 256, 0, st>>>(r->in, n, taps / 2, r->red, r->ext, ext_len, batch);
  RX_LAUNCHED();
  rx::init_taps_kernel<<<blocks(batch * 4 * taps), 256, 0, st>>>(r->taps, taps, batch);
  RX_LAUNCHED();
  std::vector<int> all(batch);
  for (int b = 0; b < batch; ++b) all[b] = b;
  auto sweep = [&](const std::vector<int>& list) -> int {
    RX_CUDA(cudaMemcpyAsync(r->items, list.data(), list.size() * sizeof(int), cudaMemcpyHostToDevice, st),
            "H2D(items)");
    const int warps = (int)list.size();
    const unsigned grid = (unsigned)((warps + 3) / 4);
    if (taps <= 16)
      rx::cma_kernel<1><<<grid, 128, 0, st>>>(r->ext, ext_len, r->taps, taps, mu, m, r->sym, r->items, warps);
    else if (taps <= 32)
      rx::cma_kernel<2><<<grid, 128, 0, st>>>(r->ext, ext_len, r->taps, taps, mu, m, r->sym, r->items, warps);
    else
      rx::cma_kernel<4><<<grid, 128, 0, st>>>(r->ext, ext_len, r->taps, taps, mu, m, r->sym, r->items, warps);
    RX_LAUNCHED();
    RX_CUDA(cudaGetLastError(), "cma_kernel");
    RX_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");   // list is a host temporary
    return DBP_OK;
  };
  std::vector<int> nre(batch, 0);
  for (int pass = 0; pass < passes; ++pass) {
    int rc = sweep(all);
    if (rc) return rc;
    rx::xcorr_kernel<<<batch, 256, 0, st>>>(r->sym, m, r->red);
    RX_LAUNCHED();
    std::vector<double> xc(4 * batch);
    RX_CUDA(cudaMemcpyAsync(xc.data(), r->red, xc.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H(xcorr)");
    RX_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    std::vector<int> collapsed;
    for (int b = 0; b < batch; ++b) {
      const double num = std::hypot(xc[4 * b], xc[4 * b + 1]);
      const double den = std::sqrt(xc[4 * b + 2] * xc[4 * b + 3]);
      if (den > 0.0 && num / den > 0.95) collapsed.push_back(b);
    }
    if (!collapsed.empty()) {
      RX_CUDA(cudaMemcpyAsync(r->items, collapsed.data(), collapsed.size() * sizeof(int), cudaMemcpyHostToDevice, st),
              "H2D(items)");
      rx::reinit_kernel<<<blocks((long long)collapsed.size() * taps), 256, 0, st>>>(r->taps, taps, r->items,
                                                                                    (int)collapsed.size());
      RX_LAUNCHED();
      for (int b : collapsed) ++nre[b];
      if ((rc = sweep(collapsed))) return rc;
    }
  }
  if (reinits)
    for (int b = 0; b < batch; ++b) reinits[b] = nre[b];
  return DBP_OK;
}

// carrier recovery of r->sym in place; r->refs holds the reference spectra when have_ref
int carrier_dev(dbp_rx* r, int batch, double rs, bool have_ref, int window, double* f_off_out, int* status) {
  const long long m = r->m;
  if (window < 1 || window > m) return fail(DBP_EINVAL, "window must be in [1, n]");
  if (!(rs > 0.0)) return fail(DBP_EINVAL, "symbol_rate must be positive");
  cudaStream_t st = r->stream;
  int rc;
  rx::pow4_kernel<<<blocks(2 * m * batch), 256, 0, st>>>(r->sym, r->work, 2 * m * batch);
  RX_LAUNCHED();
  if ((rc = fft(r, r->work, r->work, 2 * batch, kForward))) return rc;
  rx::argmax_kernel<<<batch, 1024, 0, st>>>(r->work, m, 2 * m, m, 0, r->idx, r->red);
  RX_LAUNCHED();
  std::vector<long long> peak(batch);
  std::vector<double> sv(3 * batch);
  RX_CUDA(cudaMemcpyAsync(peak.data(), r->idx, batch * sizeof(long long), cudaMemcpyDeviceToHost, st), "D2H(peak)");
  RX_CUDA(cudaMemcpyAsync(sv.data(), r->red, sv.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H(peak)");
  RX_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  std::vector<double> f_off(batch, 0.0);
  const double bin_step = rs / (double)m;
  for (int b = 0; b < batch; ++b) {   // modem.py:315-329, host double arithmetic
    const double s0 = std::log(std::max(sv[3 * b], 1e-300)), s1 = std::log(std::max(sv[3 * b + 1], 1e-300)),
                 s2 = std::log(std::max(sv[3 * b + 2], 1e-300));
    const double denom = s0 - 2.0 * s1 + s2;
    const double frac = denom != 0.0 ? 0.5 * (s0 - s2) / denom : 0.0;
    const long long pk = peak[b];
    // numpy.fft.fftfreq(n, d=1/rs)[pk]: results = [0..(n-1)/2, -(n/2)..-1] * (1 / (n * d))
    const long long kk = pk <= (m - 1) / 2 ? pk : pk - m;
    const double val = 1.0 / ((double)m * (1.0 / rs));
    const double f4 = (double)kk * val + frac * bin_step;
    status[b] = std::fabs(f4) >= rs / 2.0 - 2.0 * bin_step ? 1 : 0;
    f_off[b] = f4 / 4.0;
  }
  if (f_off_out)
    for (int b = 0; b < batch; ++b) f_off_out[b] = f_off[b];
  RX_CUDA(cudaMemcpyAsync(r->red, f_off.data(), batch * sizeof(double), cudaMemcpyHostToDevice, st), "H2D(f_off)");
  rx::derotate_kernel<<<blocks(2 * m * batch), 256, 0, st>>>(r->sym, r->work, m, batch, r->red, rs);
  RX_LAUNCHED();
  double* ang = reinterpret_cast<double*>(r->corr);   // scratch: 2 m batch doubles
  rx::vv_angle_kernel<<<blocks(2 * m * batch), 256, 0, st>>>(r->work, ang, m, 2 * batch, window);
  RX_LAUNCHED();
  rx::unwrap_apply_kernel<<<2 * batch, 1024, 0, st>>>(ang, r->work, r->sym, m);
  RX_LAUNCHED();
  RX_CUDA(cudaGetLastError(), "carrier kernels");
  RX_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");   // f_off is a host temporary
  if (!have_ref) return DBP_OK;
  // 90-degree ambiguity against the better-correlating reference (modem.py:339-350)
  if ((rc = fft(r, r->sym, r->work, 2 * batch, kForward))) return rc;
  rx::xspec_kernel<<<blocks(4 * m * batch), 256, 0, st>>>(r->work, r->refs, r->corr, m, batch);
  RX_LAUNCHED();
  if ((rc = fft(r, r->corr, r->corr, 4 * batch, kInverse))) return rc;
  rx::argmax_kernel<<<4 * batch, 1024, 0, st>>>(r->corr, m, m, 0, 1, r->idx, r->red);
  RX_LAUNCHED();
  std::vector<double> pv(8 * batch);
  RX_CUDA(cudaMemcpyAsync(pv.data(), r->red, pv.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H(corr)");
  RX_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  std::vector<int> turns(2 * batch);
  for (int bp = 0; bp < 2 * batch; ++bp) {
    double br = pv[4 * bp], bi = pv[4 * bp + 1];
    if (std::hypot(pv[4 * bp + 2], pv[4 * bp + 3]) > std::hypot(br, bi)) {
      br = pv[4 * bp + 2];
      bi = pv[4 * bp + 3];
    }
    turns[bp] = (int)std::nearbyint(std::atan2(bi, br) / (rx::kPi / 2.0));   // round half to even, like round()
  }
  RX_CUDA(cudaMemcpyAsync(r->turns, turns.data(), turns.size() * sizeof(int), cudaMemcpyHostToDevice, st),
          "H2D(turns)");
  rx::quarter_turn_kernel<<<blocks(2 * m * batch), 256, 0, st>>>(r->sym, m, 2 * batch, r->turns);
  RX_LAUNCHED();
  RX_CUDA(cudaGetLastError(), "quarter_turn_kernel");
  RX_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  return DBP_OK;
}

// best-pairing error count of r->bits against r->ref_bits (modem.py:385-405)
int count_dev(dbp_rx* r, int batch, long long skip_bits, long long* errors, long long* counted) {
  const long long m = r->m, n_bits = 2 * m;
  if (skip_bits < 0 || skip_bits >= n_bits) return fail(DBP_EINVAL, "skip must be in [0, n_bits)");
  cudaStream_t st = r->stream;
  int rc;
  rx::bits_to_symbols_kernel<<<blocks(2 * m * batch), 256, 0, st>>>(r->bits, r->work, 2 * m * batch);
  RX_LAUNCHED();
  if ((rc = fft(r, r->work, r->work, 2 * batch, kForward))) return rc;
  rx::xspec_kernel<<<blocks(4 * m * batch), 256, 0, st>>>(r->work, r->refs, r->corr, m, batch);
  RX_LAUNCHED();
  if ((rc = fft(r, r->corr, r->corr, 4 * batch, kInverse))) return rc;
  rx::argmax_kernel<<<4 * batch, 1024, 0, st>>>(r->corr, m, m, 0, 2, r->idx, nullptr);
  RX_LAUNCHED();
  const long long skip_sym = (skip_bits + 1) / 2;
  rx::count_kernel<<<4 * batch, 256, 0, st>>>(r->bits, r->ref_bits, m, skip_sym, r->idx, r->cnt);
  RX_LAUNCHED();
  RX_CUDA(cudaGetLastError(), "count kernels");
  std::vector<long long> e(4 * batch);
  RX_CUDA(cudaMemcpyAsync(e.data(), r->cnt, e.size() * sizeof(long long), cudaMemcpyDeviceToHost, st), "D2H(errors)");
  RX_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  for (int b = 0; b < batch; ++b) {
    // pairings (0, 1) then (1, 0); q = (b * 2 + p) * 2 + r; first minimum wins
    const long long straight = e[(b * 2 + 0) * 2 + 0] + e[(b * 2 + 1) * 2 + 1];
    const long long swapped = e[(b * 2 + 0) * 2 + 1] + e[(b * 2 + 1) * 2 + 0];
    errors[b] = swapped < straight ? swapped : straight;
  }
  *counted = 2 * (m - skip_sym);
  return DBP_OK;
}

int upload_ref_spectra(dbp_rx* r, const double2* h_ref) {
  RX_CUDA(cudaMemcpyAsync(r->refs, h_ref, 2 * r->m * sizeof(double2), cudaMemcpyHostToDevice, r->stream), "H2D(ref)");
  return fft(r, r->refs, r->refs, 2, kForward);
}

}  // namespace

extern "C" {

int dbp_rx_create(dbp_rx** out, int device, int64_t n_symbols, int max_batch) {
  if (!out) return fail(DBP_EINVAL, "null output pointer");
  *out = nullptr;
  if (n_symbols < 2 || n_symbols > (1LL << 28)) return fail(DBP_EINVAL, "n_symbols outside [2, 2^28]");
  if (max_batch < 1) return fail(DBP_EINVAL, "max_batch must be >= 1");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(DBP_ECUDA, "no CUDA device available");
  }
  if (device < 0 || device >= ndev) return fail(DBP_EINVAL, "device index out of range");
  Guard g(device);
  dbp_rx* r = new (std::nothrow) dbp_rx();
  if (!r) return fail(DBP_ENOMEM, "host allocation failed");
  r->device = device;
  r->m = n_symbols;
  r->max_batch = max_batch;
  const size_t B = (size_t)max_batch, m = (size_t)n_symbols;
  bool ok = cudaMalloc(&r->in, B * 4 * m * sizeof(double2)) == cudaSuccess &&
            cudaMalloc(&r->sym, B * 2 * m * sizeof(double2)) == cudaSuccess &&
            cudaMalloc(&r->work, B * 2 * m * sizeof(double2)) == cudaSuccess &&
            cudaMalloc(&r->corr, B * 4 * m * sizeof(double2)) == cudaSuccess &&
            cudaMalloc(&r->fftbuf, fft64::scratch_elems(m, 4 * B) * sizeof(double2)) == cudaSuccess &&
            cudaMalloc(&r->refs, 2 * m * sizeof(double2)) == cudaSuccess &&
            cudaMalloc(&r->bits, B * 4 * m) == cudaSuccess && cudaMalloc(&r->ref_bits, 4 * m) == cudaSuccess &&
            cudaMalloc(&r->red, B * 8 * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&r->idx, B * 4 * sizeof(long long)) == cudaSuccess &&
            cudaMalloc(&r->cnt, B * 4 * sizeof(long long)) == cudaSuccess &&
            cudaMalloc(&r->items, B * sizeof(int)) == cudaSuccess &&
            cudaMalloc(&r->turns, B * 2 * sizeof(int)) == cudaSuccess &&
            cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    dbp_rx_destroy(r);
    return fail(DBP_ENOMEM, "device allocation of the receiver buffers failed");
  }
  *out = r;
  return DBP_OK;
}

int dbp_rx_destroy(dbp_rx* r) {
  if (!r) return DBP_OK;
  Guard g(r->device);
  if (r->stream) cudaStreamSynchronize(r->stream);
  cudaFree(r->fftbuf);
  cudaFree(r->in);
  cudaFree(r->ext);
  cudaFree(r->sym);
  cudaFree(r->work);
  cudaFree(r->corr);
  cudaFree(r->refs);
  cudaFree(r->taps);
  cudaFree(r->bits);
  cudaFree(r->ref_bits);
  cudaFree(r->red);
  cudaFree(r->idx);
  cudaFree(r->cnt);
  cudaFree(r->items);
  cudaFree(r->turns);
  if (r->stream) cudaStreamDestroy(r->stream);
  delete r;
  return DBP_OK;
}

int dbp_rx_equalize(dbp_rx* r, const void* h_in, int batch, int taps, double step_size, int passes, void* h_out,
                    int* reinits, void* h_taps) {
  int rc = check_batch(r, batch);
  if (rc) return rc;
  if (!h_in || !h_out) return fail(DBP_EINVAL, "null buffer");
  Guard g(r->device);
  const size_t in_bytes = (size_t)batch * 4 * r->m * sizeof(double2);
  RX_CUDA(cudaMemcpyAsync(r->in, h_in, in_bytes, cudaMemcpyHostToDevice, r->stream), "H2D(samples)");
  if ((rc = equalize_dev(r, batch, taps, step_size, passes, reinits))) return rc;
  RX_CUDA(cudaMemcpyAsync(h_out, r->sym, (size_t)batch * 2 * r->m * sizeof(double2), cudaMemcpyDeviceToHost,
                          r->stream), "D2H(symbols)");
  if (h_taps)
    RX_CUDA(cudaMemcpyAsync(h_taps, r->taps, (size_t)batch * 4 * taps * sizeof(double2), cudaMemcpyDeviceToHost,
                            r->stream), "D2H(taps)");
  RX_CUDA(cudaStreamSynchronize(r->stream), "cudaStreamSynchronize");
  return DBP_OK;
}

int dbp_rx_carrier_recover(dbp_rx* r, const void* h_sym, int batch, double symbol_rate, const void* h_ref,
                           int window, void* h_out, double* f_off, int* status) {
  int rc = check_batch(r, batch);
  if (rc) return rc;
  if (!h_sym || !h_out || !status) return fail(DBP_EINVAL, "null buffer");
  Guard g(r->device);
  RX_CUDA(cudaMemcpyAsync(r->sym, h_sym, (size_t)batch * 2 * r->m * sizeof(double2), cudaMemcpyHostToDevice,
                          r->stream), "H2D(symbols)");
  if (h_ref && (rc = upload_ref_spectra(r, static_cast<const double2*>(h_ref)))) return rc;
  if ((rc = carrier_dev(r, batch, symbol_rate, h_ref != nullptr, window, f_off, status))) return rc;
  RX_CUDA(cudaMemcpyAsync(h_out, r->sym, (size_t)batch * 2 * r->m * sizeof(double2), cudaMemcpyDeviceToHost,
                          r->stream), "D2H(symbols)");
  RX_CUDA(cudaStreamSynchronize(r->stream), "cudaStreamSynchronize");
  return DBP_OK;
}

int dbp_rx_decide(dbp_rx* r, const void* h_sym, int batch, uint8_t* h_bits) {
  int rc = check_batch(r, batch);
  if (rc) return rc;
  if (!h_sym || !h_bits) return fail(DBP_EINVAL, "null buffer");
  Guard g(r->device);
  const long long total = (long long)batch * 2 * r->m;
  RX_CUDA(cudaMemcpyAsync(r->sym, h_sym, total * sizeof(double2), cudaMemcpyHostToDevice, r->stream), "H2D(symbols)");
  rx::decide_kernel<<<blocks(total), 256, 0, r->stream>>>(r->sym, r->bits, total);
  RX_LAUNCHED();
  RX_CUDA(cudaGetLastError(), "decide_kernel");
  RX_CUDA(cudaMemcpyAsync(h_bits, r->bits, 2 * total, cudaMemcpyDeviceToHost, r->stream), "D2H(bits)");
  RX_CUDA(cudaStreamSynchronize(r->stream), "cudaStreamSynchronize");
  return DBP_OK;
}

int dbp_rx_count_errors(dbp_rx* r, const uint8_t* h_dec, int batch, const uint8_t* h_ref, int64_t skip_bits,
                        int64_t* errors, int64_t* counted) {
  int rc = check_batch(r, batch);
  if (rc) return rc;
  if (!h_dec || !h_ref || !errors || !counted) return fail(DBP_EINVAL, "null buffer");
  Guard g(r->device);
  const long long m = r->m;
  RX_CUDA(cudaMemcpyAsync(r->bits, h_dec, (size_t)batch * 4 * m, cudaMemcpyHostToDevice, r->stream), "H2D(bits)");
  RX_CUDA(cudaMemcpyAsync(r->ref_bits, h_ref, (size_t)4 * m, cudaMemcpyHostToDevice, r->stream), "H2D(ref bits)");
  rx::bits_to_symbols_kernel<<<blocks(2 * m), 256, 0, r->stream>>>(r->ref_bits, r->refs, 2 * m);
  RX_LAUNCHED();
  if ((rc = fft(r, r->refs, r->refs, 2, kForward))) return rc;
  std::vector<long long> e(batch);
  long long c = 0;
  if ((rc = count_dev(r, batch, skip_bits, e.data(), &c))) return rc;
  for (int b = 0; b < batch; ++b) errors[b] = e[b];
  *counted = c;
  return DBP_OK;
}

int dbp_rx_chain(dbp_rx* r, const void* h_in, int in_is_c64, int batch, int taps, double step_size, int passes,
                 double symbol_rate, const void* h_ref_sym, int window, int64_t skip_bits, double* metrics,
                 int* status) {
  int rc = check_batch(r, batch);
  if (rc) return rc;
  if (!h_in || !h_ref_sym || !metrics || !status) return fail(DBP_EINVAL, "null buffer");
  Guard g(r->device);
  cudaStream_t st = r->stream;
  const long long m = r->m, n = 2 * m;
  if (in_is_c64) {   // complex64 DBP output: stage it in the upper half of corr, widen on the device
    float2* tmp = reinterpret_cast<float2*>(r->corr);
    RX_CUDA(cudaMemcpyAsync(tmp, h_in, (size_t)batch * 2 * n * sizeof(float2), cudaMemcpyHostToDevice, st),
            "H2D(samples)");
    const long long total = (long long)batch * 2 * n;
    rx::widen_kernel<<<blocks(total), 256, 0, st>>>(tmp, r->in, total);
    RX_LAUNCHED();
    RX_CUDA(cudaGetLastError(), "widen");
  } else {
    RX_CUDA(cudaMemcpyAsync(r->in, h_in, (size_t)batch * 2 * n * sizeof(double2), cudaMemcpyHostToDevice, st),
            "H2D(samples)");
  }
  std::vector<int> reinits(batch);
  if ((rc = equalize_dev(r, batch, taps, step_size, passes, reinits.data()))) return rc;
  if ((rc = upload_ref_spectra(r, static_cast<const double2*>(h_ref_sym)))) return rc;
  std::vector<double> f_off(batch);
  if ((rc = carrier_dev(r, batch, symbol_rate, true, window, f_off.data(), status))) return rc;
  // EVM against the scaled nearest constellation point
  rx::evm_kernel<<<batch, 256, 0, st>>>(r->sym, m, 0, r->red);
  RX_LAUNCHED();
  rx::evm_kernel<<<batch, 256, 0, st>>>(r->sym, m, 1, r->red);
  RX_LAUNCHED();
  std::vector<double> ev(3 * batch);
  RX_CUDA(cudaMemcpyAsync(ev.data(), r->red, ev.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H(evm)");
  // decisions of the recovered symbols and of the reference (modem.py:116-125)
  rx::decide_kernel<<<blocks(2 * m * batch), 256, 0, st>>>(r->sym, r->bits, 2 * m * batch);
  RX_LAUNCHED();
  RX_CUDA(cudaMemcpyAsync(r->work, h_ref_sym, 2 * m * sizeof(double2), cudaMemcpyHostToDevice, st), "H2D(ref)");
  rx::decide_kernel<<<blocks(2 * m), 256, 0, st>>>(r->work, r->ref_bits, 2 * m);
  RX_LAUNCHED();
  rx::bits_to_symbols_kernel<<<blocks(2 * m), 256, 0, st>>>(r->ref_bits, r->refs, 2 * m);
  RX_LAUNCHED();
  if ((rc = fft(r, r->refs, r->refs, 2, kForward))) return rc;
  std::vector<long long> errors(batch);
  long long counted = 0;
  if ((rc = count_dev(r, batch, skip_bits, errors.data(), &counted))) return rc;
  for (int b = 0; b < batch; ++b) {
    const double ber = (double)errors[b] / (double)(2 * counted);
    metrics[6 * b + 0] = ber;
    metrics[6 * b + 1] = (double)errors[b];
    metrics[6 * b + 2] = (double)(2 * counted);
    metrics[6 * b + 3] = 100.0 * std::sqrt((ev[3 * b + 1] / (double)(2 * m)) / (ev[3 * b + 2] / (double)(2 * m)));
    metrics[6 * b + 4] = f_off[b];
    metrics[6 * b + 5] = (double)reinits[b];
    if (status[b] == 0 && ber >= 0.4) status[b] = 2;
  }
  return DBP_OK;
}

}  // extern "C"
