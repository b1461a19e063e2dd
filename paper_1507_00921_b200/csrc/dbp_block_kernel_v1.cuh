// Fused overlap-save DBP block kernel for sm_100a.
//
// One overlap-save block of N dual-polarisation samples per thread slice
// (T = N/16 threads, 16 samples of BOTH polarisations per thread).  The
// whole multi-step program -- dispersion filter (FFT -> x H -> IFFT), the
// SSFM/ESSFM nonlinear rotation with the in-block cyclic intensity FIR,
// gains -- runs on-chip between ONE coalesced load of the block (with its
// halo, cyclic wrap of the whole signal) and ONE store of its centre.
//
// Reference behaviour reproduced (pkg/src/fiberdbp/...):
//   framing  spectral.py:122-145  block b = samples [b*step - M/2, +N) mod n,
//                                 keep [M/2, M/2 + step), trim to n
//   FFE      dbp.py:185-191       ifft(fft(b) * H)
//   SSFM     dbp.py:193-235       symmetric / linear-first / nonlinear-first
//   rotate   dbp.py:49-75, channel.py:61-71
//            b * exp(-j g w (c0 I_k + sum_i c_i (I_{k-i} + I_{k+i}))), cyclic in-block
//
// FFT: mixed radix, passes of radix 16 (last pass 2..16).  Forward passes
// are decimation-in-frequency, so the spectrum ends digit-reversed across
// threads; the dispersion table is read at each register's natural bin
// index, and the inverse transform is the exact adjoint walk back, so no
// reordering pass exists.  Between passes data moves through shared memory
// as float4 {x.re, x.im, y.re, y.im} with an XOR swizzle that makes every
// exchange bank-conflict free.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <vector>

#include "dbp_common.cuh"
#include "dft_small.cuh"

namespace dbp {

// host helpers (same interface as the v2 header)
inline std::vector<float2> make_twiddles(int logn) {
  const int np = (logn + 3) / 4;
  std::vector<float2> tw;
  for (int p = 0; p < np - 1; ++p) {
    const int ls = logn - 4 * (p + 1);
    const long long S = 1LL << ls;
    const long long period = 16 * S;
    for (int k = 1; k < 16; ++k)
      for (long long ns = 0; ns < S; ++ns) {
        const double ang = -2.0 * M_PI * (double)((ns * k) % period) / (double)period;
        tw.push_back(make_float2((float)std::cos(ang), (float)std::sin(ang)));
      }
  }
  if (tw.empty()) tw.push_back(make_float2(1.f, 0.f));
  return tw;
}

inline int slice_floats(int N, int pw) {
  auto phys = [](int u) { return u + ((u >> 4) << 2); };
  int fir = phys(N + 2 * pw) + 4 + phys(N);
  int v = 4 * N > fir ? 4 * N : fir;
  return (v + 3) & ~3;
}

template <int LOGN>
struct Geo {
  static constexpr int N = 1 << LOGN;
  static constexpr int T = N / 16;                      // threads per block slice
  static constexpr int NP = (LOGN + 3) / 4;             // FFT passes
  static constexpr int RLAST = 1 << (LOGN - 4 * (NP - 1));
#ifndef DBP_CTA_THREADS
#define DBP_CTA_THREADS 128
#endif
  static constexpr int BPC = T >= DBP_CTA_THREADS ? 1 : DBP_CTA_THREADS / T;  // block slices per CTA
  static constexpr int THREADS = T * BPC;
#ifndef DBP_THREADS_PER_SM
#define DBP_THREADS_PER_SM 384
#endif
  // resident-thread target per SM sets the register budget (65536 / target)
  static constexpr int MIN_CTAS = DBP_THREADS_PER_SM / THREADS > 0 ? DBP_THREADS_PER_SM / THREADS : 1;
  __host__ __device__ static constexpr int radix(int p) { return p < NP - 1 ? 16 : RLAST; }
  __host__ __device__ static constexpr int log_s(int p) { return p < NP - 1 ? LOGN - 4 * (p + 1) : 0; }
  __host__ __device__ static constexpr int tw_offset(int p) {
    int off = 0;
    for (int q = 0; q < p; ++q) off += 15 << log_s(q);
    return off;
  }
  static constexpr int TW_ENTRIES = tw_offset(NP - 1);
};

// Swizzle of the exchange between pass P and P+1 (see header comment).
template <int LOGN, int P>
__device__ __forceinline__ int swz(int i) {
  using G = Geo<LOGN>;
  constexpr int ls = G::log_s(P), ls1 = G::log_s(P + 1);
  if constexpr (ls1 >= 3) {
    return i;
  } else {
    return i ^ (((i >> ls) << ls1) & 7);
  }
}

// ---------------------------------------------------------------------------
// FFT -> x table -> IFFT, recursive over passes (forward on the way down,
// adjoint on the way back up).  On entry and exit thread t holds samples
// n*T + t (n = 0..15) of its block in x[n], y[n].
// ---------------------------------------------------------------------------
template <int LOGN, int P>
__device__ __forceinline__ void conv_pass(float2 (&x)[16], float2 (&y)[16], float4* sm,
                                          const float2* __restrict__ tab,
                                          const float2* __restrict__ tw, int t) {
  using G = Geo<LOGN>;
  constexpr int N = G::N, T = G::T;
  if constexpr (P < G::NP - 1) {
    // forward radix-16 over one group (g = t), then twiddle W_{16 S}^{ns k}
    constexpr int LS = G::log_s(P);
    constexpr int S = 1 << LS;
    dft<16, false>(x);
    dft<16, false>(y);
    const int ns = t & (S - 1);
    const float2* twp = tw + G::tw_offset(P) + ns;
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      const float2 wk = __ldg(twp + (k - 1) * S);
      x[k] = c_mul(x[k], wk);
      y[k] = c_mul(y[k], wk);
    }
    // exchange into pass P+1 layout
    constexpr int R1 = G::radix(P + 1);
    constexpr int LS1 = G::log_s(P + 1);
    constexpr int GRP = 16 / R1;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k)
      sm[swz<LOGN, P>(t + k * (N / 16))] = make_float4(x[k].x, x[k].y, y[k].x, y[k].y);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < GRP; ++q) {
      const int g = t + T * q;
      const int base = ((g >> LS1) << LS) + (g & ((1 << LS1) - 1));
#pragma unroll
      for (int e = 0; e < R1; ++e) {
        const float4 v = sm[swz<LOGN, P>(base + (e << LS1))];
        x[q * R1 + e] = make_float2(v.x, v.y);
        y[q * R1 + e] = make_float2(v.z, v.w);
      }
    }

    conv_pass<LOGN, P + 1>(x, y, sm, tab, tw, t);

    // adjoint exchange back into pass P layout
    __syncthreads();
#pragma unroll
    for (int q = 0; q < GRP; ++q) {
      const int g = t + T * q;
      const int base = ((g >> LS1) << LS) + (g & ((1 << LS1) - 1));
#pragma unroll
      for (int e = 0; e < R1; ++e)
        sm[swz<LOGN, P>(base + (e << LS1))] =
            make_float4(x[q * R1 + e].x, x[q * R1 + e].y, y[q * R1 + e].x, y[q * R1 + e].y);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float4 v = sm[swz<LOGN, P>(t + k * (N / 16))];
      x[k] = make_float2(v.x, v.y);
      y[k] = make_float2(v.z, v.w);
    }
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      const float2 wk = __ldg(twp + (k - 1) * S);  // reloaded: keeps registers free below
      x[k] = c_mulc(x[k], wk);
      y[k] = c_mulc(y[k], wk);
    }
    dft<16, true>(x);
    dft<16, true>(y);
  } else {
    // last pass: S = 1, GRP groups of radix RL per thread, group g = t + T q
    constexpr int RL = G::RLAST;
    constexpr int GRP = 16 / RL;
    constexpr int LL = N / RL;  // bin index k = g + LL * e
#pragma unroll
    for (int q = 0; q < GRP; ++q) {
      dft<RL, false>(x + q * RL);
      dft<RL, false>(y + q * RL);
    }
#pragma unroll
    for (int q = 0; q < GRP; ++q) {
#pragma unroll
      for (int e = 0; e < RL; ++e) {
        const float2 h = __ldg(tab + (t + T * q) + LL * e);
        x[q * RL + e] = c_mul(x[q * RL + e], h);
        y[q * RL + e] = c_mul(y[q * RL + e], h);
      }
    }
#pragma unroll
    for (int q = 0; q < GRP; ++q) {
      dft<RL, true>(x + q * RL);
      dft<RL, true>(y + q * RL);
    }
  }
}

// ---------------------------------------------------------------------------
// Nonlinear rotation with the in-block cyclic intensity FIR.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int fir_phys(int u) { return u + ((u >> 4) << 2); }  // pad 4 per 16

// F for 8 consecutive outputs p0 .. p0+7 (p0 = 16 t + 8 q) from a register
// window of the padded intensity buffer; results go straight to fbuf.
// Only 8 outputs per call keeps the unrolled code small (instruction-cache
// footprint) at the price of re-reading 2 PW window floats per chunk.
template <int NC>
__device__ __forceinline__ void fir8_fixed(const float* __restrict__ ibuf, float* __restrict__ fbuf,
                                           int p0, const KernelParams& kp) {
  constexpr int PW = (NC + 3) & ~3;
  constexpr int W = 8 + 2 * PW;
  float w[W];
#pragma unroll
  for (int m = 0; m < W / 4; ++m) {
    const float4 v = *reinterpret_cast<const float4*>(ibuf + fir_phys(p0 + 4 * m));
    w[4 * m] = v.x; w[4 * m + 1] = v.y; w[4 * m + 2] = v.z; w[4 * m + 3] = v.w;
  }
  float f[8];
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    float acc = kp.c[0] * w[o + PW];
#pragma unroll
    for (int i = 1; i <= NC; ++i) acc = fmaf(kp.c[i], w[o + PW - i] + w[o + PW + i], acc);
    f[o] = acc;
  }
  *reinterpret_cast<float4*>(fbuf + fir_phys(p0)) = make_float4(f[0], f[1], f[2], f[3]);
  *reinterpret_cast<float4*>(fbuf + fir_phys(p0 + 4)) = make_float4(f[4], f[5], f[6], f[7]);
}

// any nc: taps in chunks of four, windows re-read per chunk (same summation
// order as fir8_fixed, so every path gives identical bits for a given c)
__device__ __forceinline__ void fir8_generic(const float* __restrict__ ibuf, float* __restrict__ fbuf,
                                             int p0, int pw, const KernelParams& kp) {
  float f[8];
  {
    const float4 a = *reinterpret_cast<const float4*>(ibuf + fir_phys(p0 + pw));
    const float4 b = *reinterpret_cast<const float4*>(ibuf + fir_phys(p0 + pw + 4));
    const float c0 = kp.c[0];
    f[0] = c0 * a.x; f[1] = c0 * a.y; f[2] = c0 * a.z; f[3] = c0 * a.w;
    f[4] = c0 * b.x; f[5] = c0 * b.y; f[6] = c0 * b.z; f[7] = c0 * b.w;
  }
#pragma unroll 1
  for (int i0 = 1; i0 <= kp.nc; i0 += 4) {
    // left: positions p0 - i0 - 3 .. p0 + 7 - i0  ->  window u from p0 + pw - i0 - 3
    // right: positions p0 + i0 .. p0 + 10 + i0     ->  window u from p0 + pw + i0 - 1
    float l[12], r[12];
    const int ul = p0 + pw - i0 - 3;
    const int ur = p0 + pw + i0 - 1;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const float4 a = *reinterpret_cast<const float4*>(ibuf + fir_phys(ul + 4 * m));
      const float4 b = *reinterpret_cast<const float4*>(ibuf + fir_phys(ur + 4 * m));
      l[4 * m] = a.x; l[4 * m + 1] = a.y; l[4 * m + 2] = a.z; l[4 * m + 3] = a.w;
      r[4 * m] = b.x; r[4 * m + 1] = b.y; r[4 * m + 2] = b.z; r[4 * m + 3] = b.w;
    }
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const float ci = __ldg(kp.coeff + i0 + d);
      // tap i = i0 + d: left value at position p - i -> l[o + 3 - d]; right p + i -> r[o + 1 + d]
#pragma unroll
      for (int o = 0; o < 8; ++o) f[o] = fmaf(ci, l[o + 3 - d] + r[o + 1 + d], f[o]);
    }
  }
  *reinterpret_cast<float4*>(fbuf + fir_phys(p0)) = make_float4(f[0], f[1], f[2], f[3]);
  *reinterpret_cast<float4*>(fbuf + fir_phys(p0 + 4)) = make_float4(f[4], f[5], f[6], f[7]);
}

template <int LOGN>
__device__ __forceinline__ void rotate(float2 (&x)[16], float2 (&y)[16], float* smf,
                                       const KernelParams& kp, int step_idx, int t) {
  using G = Geo<LOGN>;
  constexpr int N = G::N, T = G::T;
  float inten[16];
#pragma unroll
  for (int n = 0; n < 16; ++n)
    inten[n] = fmaf(x[n].x, x[n].x, x[n].y * x[n].y) + fmaf(y[n].x, y[n].x, y[n].y * y[n].y);

  float f[16];
  if (kp.nc == 0) {
#pragma unroll
    for (int n = 0; n < 16; ++n) f[n] = kp.c[0] * inten[n];
  } else {
    const int pw = kp.fir_pad;
    float* ibuf = smf;                                        // logical [-pw, N + pw)
    float* fbuf = smf + fir_phys(N + 2 * pw) + 4;             // logical [0, N)
    __syncthreads();
#pragma unroll
    for (int n = 0; n < 16; ++n) {
      const int j = n * T + t;
      ibuf[fir_phys(j + pw)] = inten[n];
      if (j < pw) ibuf[fir_phys(j + N + pw)] = inten[n];
      if (j >= N - pw) ibuf[fir_phys(j - N + pw)] = inten[n];
    }
    __syncthreads();
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
      const int p0 = 16 * t + 8 * q;
      switch (kp.nc) {
        case 1: fir8_fixed<1>(ibuf, fbuf, p0, kp); break;
        case 9: fir8_fixed<9>(ibuf, fbuf, p0, kp); break;
        case 17: fir8_fixed<17>(ibuf, fbuf, p0, kp); break;
        case 32: fir8_fixed<32>(ibuf, fbuf, p0, kp); break;
        case 33: fir8_fixed<33>(ibuf, fbuf, p0, kp); break;
        default: fir8_generic(ibuf, fbuf, p0, pw, kp); break;
      }
    }
    __syncthreads();
#pragma unroll
    for (int n = 0; n < 16; ++n) f[n] = fbuf[fir_phys(n * T + t)];
  }

  const float2 sg = __ldg(kp.steps + step_idx);  // (a_j, g_j)
#pragma unroll
  for (int n = 0; n < 16; ++n) {
    const float th = sg.x * f[n];
    const float k = rintf(th * 0.159154943091895336f);
    float r = fmaf(k, -6.28318548202514648f, th);
    r = fmaf(k, 1.74845553e-7f, r);
    float s, c;
    __sincosf(r, &s, &c);
    c *= sg.y;
    s *= sg.y;
    x[n] = make_float2(fmaf(x[n].x, c, -x[n].y * s), fmaf(x[n].x, s, x[n].y * c));
    y[n] = make_float2(fmaf(y[n].x, c, -y[n].y * s), fmaf(y[n].x, s, y[n].y * c));
  }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <int LOGN>
__global__ void __launch_bounds__(Geo<LOGN>::THREADS, Geo<LOGN>::MIN_CTAS)
dbp_block_kernel(const KernelParams kp) {
  using G = Geo<LOGN>;
  constexpr int N = G::N, T = G::T;
  extern __shared__ float4 smem_raw[];
  const int t = threadIdx.x;
  float* smf = reinterpret_cast<float*>(smem_raw) + threadIdx.y * kp.slice_floats;
  float4* sm = reinterpret_cast<float4*>(smf);

  const long long blk = (long long)blockIdx.x * G::BPC + threadIdx.y;
  const bool active = blk < kp.total_blocks;
  long long item = 0, b = 0;
  if (active) {
    item = blk / kp.blocks_per_item;
    b = kp.block_begin + (blk - item * kp.blocks_per_item);
  }

  float2 x[16], y[16];
  const long long s0 = b * kp.step - kp.lead;  // global index of block sample 0
  if (active) {
    const float2* px = kp.in + item * kp.in_item_stride;
    const float2* py = px + kp.in_pol_stride;
    if (!kp.cyclic || (s0 >= 0 && s0 + N <= kp.n_total)) {
      // interior block (or pre-extended chunk): one contiguous window, immediate offsets
      const long long base = (kp.cyclic ? s0 : s0 - kp.in_origin) + t;
#pragma unroll
      for (int n = 0; n < 16; ++n) {
        x[n] = ld_stream(px + base + n * T);
        y[n] = ld_stream(py + base + n * T);
      }
    } else {
      // edge block: circular extension of the whole signal (spectral.py:128)
#pragma unroll
      for (int n = 0; n < 16; ++n) {
        long long gi = s0 + n * T + t;
        if (gi < 0 || gi >= kp.n_total) {
          gi %= kp.n_total;
          if (gi < 0) gi += kp.n_total;
        }
        x[n] = ld_stream(px + gi);
        y[n] = ld_stream(py + gi);
      }
    }
  } else {
#pragma unroll
    for (int n = 0; n < 16; ++n) x[n] = y[n] = make_float2(0.f, 0.f);
  }

  // operator program (dbp.py:212-233)
  int n_ops;
  if (kp.program == kFFE) n_ops = 1;
  else if (kp.program == kRotateOnly) n_ops = kp.n_steps;
  else n_ops = 2 * kp.n_steps + (kp.arrangement == kSymmetric ? 1 : 0);

  for (int op = 0; op < n_ops; ++op) {
    bool is_conv;
    int sidx = 0;
    const float2* tab = kp.tab_full;
    if (kp.program == kFFE) {
      is_conv = true;
    } else if (kp.program == kRotateOnly) {
      is_conv = false;
      sidx = op;
    } else if (kp.arrangement == kSymmetric) {
      is_conv = (op & 1) == 0;
      sidx = op >> 1;
      if (op == 0 || op == n_ops - 1) tab = kp.tab_half;
    } else if (kp.arrangement == kLinearFirst) {
      is_conv = (op & 1) == 0;
      sidx = op >> 1;
    } else {
      is_conv = (op & 1) == 1;
      sidx = op >> 1;
    }
    if (is_conv) {
      conv_pass<LOGN, 0>(x, y, sm, tab, kp.twiddle, t);
    } else {
      rotate<LOGN>(x, y, smf, kp, sidx, t);
    }
  }

  if (active) {
    float2* ox = kp.out + item * kp.out_item_stride;
    float2* oy = ox + kp.out_pol_stride;
    const long long ob = b * kp.step - kp.lead - kp.out_origin;  // output index of block sample 0
    const bool whole = (b + 1) * kp.step <= kp.n_total;
#pragma unroll
    for (int n = 0; n < 16; ++n) {
      const int j = n * T + t;
      const bool keep = j >= kp.lead && j < kp.lead + kp.step &&
                        (whole || b * kp.step + (j - kp.lead) < kp.n_total);
      if (keep) {
        st_stream(ox + ob + j, x[n]);
        st_stream(oy + ob + j, y[n]);
      }
    }
  }
}

}  // namespace dbp
