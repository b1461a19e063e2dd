// Overlap-save DBP for block lengths outside the fused kernel's range
// (N < 16 or N > 8192): the reference's own algorithm (spectral.py:87-145,
// dbp.py:160-235) as a multi-kernel float64 pipeline on the device.
//
// The reference accepts any power-of-two block length (spectral.py:72-76);
// the fused block kernel holds a block in one CTA's registers and shared
// memory, which bounds it to 16 <= N <= 8192.  Longer (and shorter) blocks
// take this path instead -- no CPU fallback: a chunk of blocks is gathered
// with the cyclic extension into a complex128 workspace [block][pol][N],
// every operator of the decoded program (KernelParams: conv_all / conv_parity
// / half_ends / sidx_shift) runs over the whole chunk -- the linear step as
// the library's float64 Stockham FFT (fft64.cuh), the filter multiply (1/N
// folded into the table) and the unscaled inverse; the nonlinear step as an
// intensity pass and a cyclic-FIR + rotation pass -- and the kept centres are
// written back as complex64.  Float64 throughout, so results agree with the
// reference to ~1e-12 before the final complex64 rounding.  HBM-bound
// (log4 N passes per transform), for generality rather than speed.
#pragma once
#include <cuda_runtime.h>

#include "dbp_common.cuh"

namespace dbp_general {

constexpr int kThreads = 256;
constexpr int kMaxTaps = 64 + 1;   // c_0 .. c_64 (DBP_MAX_SIDE_COEFFS)

struct Taps {
  double c[kMaxTaps];
};

__device__ __forceinline__ void locate(const dbp::KernelParams& kp, long long blk, long long& item, long long& b) {
  item = blk / kp.blocks_per_item;
  b = kp.block_begin + (blk - item * kp.blocks_per_item);
}

// ws[(blk - blk0) * 2 + pol][j] = block sample j of global block blk (spectral.py:124-131)
__global__ void frame_kernel(const dbp::KernelParams kp, long long blk0, long long nblk, long long n,
                             double2* __restrict__ ws) {
  const long long total = nblk * 2 * n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long j = i % n, row = i / n;
    const int pol = (int)(row & 1);
    long long item, b;
    locate(kp, blk0 + (row >> 1), item, b);
    long long gi = b * kp.step - kp.lead + j;
    if (kp.cyclic) {
      gi %= kp.n_total;
      if (gi < 0) gi += kp.n_total;
    } else {
      gi -= kp.in_origin;
    }
    const float2 v = kp.in[item * kp.in_item_stride + pol * kp.in_pol_stride + gi];
    ws[i] = make_double2((double)v.x, (double)v.y);
  }
}

// x[row][k] *= tab[k]
__global__ void mul_kernel(double2* __restrict__ x, const double2* __restrict__ tab, long long total, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const double2 a = x[i], h = tab[i % n];
    x[i] = make_double2(fma(a.x, h.x, -a.y * h.y), fma(a.x, h.y, a.y * h.x));
  }
}

// inten[blk][k] = |x_k|^2 + |y_k|^2 (dbp.py:71)
__global__ void intensity_kernel(const double2* __restrict__ ws, double* __restrict__ inten, long long nblk,
                                 long long n) {
  const long long total = nblk * n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long blk = i / n, k = i - blk * n;
    const double2 x = ws[(2 * blk) * n + k], y = ws[(2 * blk + 1) * n + k];
    inten[i] = x.x * x.x + x.y * x.y + (y.x * y.x + y.y * y.y);
  }
}

// F_k = c_0 I_k + sum_i c_i (I_{k-i} + I_{k+i}) (cyclic in the block, dbp.py:72-74);
// both polarisations of position k times exp(+j a F_k), then times g when g != 1
// (dbp.py:75, 202-207, 220-221); per-item coefficient sets when kp.coeff_stride
__global__ void rotate_kernel(double2* __restrict__ ws, const double* __restrict__ inten, long long nblk,
                              long long n, const dbp::KernelParams kp, long long blk0, Taps taps, int nc,
                              double a, double g) {
  const long long total = nblk * n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long blk = i / n, k = i - blk * n;
    const double* ib = inten + blk * n;
    const float* cset = nullptr;
    if (kp.coeff_stride) {
      long long item, b;
      locate(kp, blk0 + blk, item, b);
      cset = kp.coeff + item * kp.coeff_stride;
    }
    double f = (cset ? (double)cset[0] : taps.c[0]) * ib[k];
    for (int t = 1; t <= nc; ++t) {
      long long lo = k - t, hi = k + t;
      lo %= n;
      if (lo < 0) lo += n;
      hi %= n;
      const double ct = cset ? (double)cset[t] : taps.c[t];
      f = f + ct * (ib[lo] + ib[hi]);
    }
    double s, c;
    sincos(a * f, &s, &c);
    for (int pol = 0; pol < 2; ++pol) {
      double2& v = ws[(2 * blk + pol) * n + k];
      double2 r = make_double2(v.x * c - v.y * s, v.x * s + v.y * c);
      if (g != 1.0) r = make_double2(r.x * g, r.y * g);
      v = r;
    }
  }
}

// kept centre [lead, lead + len) of each block to its output position (spectral.py:143-145)
__global__ void store_kernel(const double2* __restrict__ ws, const dbp::KernelParams kp, long long blk0,
                             long long nblk, long long n) {
  const long long total = nblk * 2 * (long long)kp.step;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i % kp.step, row = i / kp.step;
    const int pol = (int)(row & 1);
    long long item, b;
    locate(kp, blk0 + (row >> 1), item, b);
    const long long o = b * kp.step + r;           // output sample index
    if (o >= kp.n_total) continue;                 // trim to the signal length
    const double2 v = ws[row * n + kp.lead + r];
    kp.out[item * kp.out_item_stride + pol * kp.out_pol_stride + (o - kp.out_origin)] =
        make_float2((float)v.x, (float)v.y);
  }
}

inline unsigned grid_for(long long total) {
  long long g = (total + kThreads - 1) / kThreads;
  if (g > 148LL * 64) g = 148LL * 64;   // grid-stride beyond this
  return (unsigned)(g > 0 ? g : 1);
}

}  // namespace dbp_general
