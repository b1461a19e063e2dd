// Whole-waveform split-step Fourier link simulator on sm_100a.
//
// Reference: pkg/src/fiberdbp/channel.py:74-94 propagate_span -- per step
// x <- ifft(fft(x) * exp(-j 2 pi^2 beta2 f^2 dz)); x <- x exp(-j gamma
// dz_eff (|x|^2 + |y|^2)); x <- x exp(-alpha dz / 2) -- on ONE circular
// block of n = 2^k samples (2^17 .. 2^21 in the reference experiments), and
// channel.py:97-153 (amplifier with ASE, Jones rotation) at span ends.
//
// n = N1 N2 four-step FFT built from the DBP kernel's block-FFT halves
// (fft_fwd / fft_inv: radix-16 register DFTs + shared-memory exchanges):
//
//   At[n2][n1] = x[n1 N2 + n2]   (N2 rows of length N1)
//   K_a  row of At : fft_fwd over n1, x W_n^{k1 n2}, store in register order
//                    (W_n from full tables in both layouts, rounded for |w| ~ 1)
//   transpose      -> B[p][n2]  (row p = register position of bin k1)
//   K_b  row of B  : fft_fwd over n2, x Lin[k1 + N1 k2] (1/n folded in),
//                    fft_inv, x W_n^{-k1 n2}, store natural
//   transpose      -> At'
//   K_c  row of At': fft_inv over n1, x e^{-j gamma dz_eff I} x loss, and
//                    for every step but the last K_a again (fused, mode CA)
//
// One SSFM step = two row kernels + two transposes over the waveform in this
// transposed layout (n > 2^21).  For 2^11 <= n <= 2^21 the column layout
// keeps the waveform in natural [N1][N2] order: K_a / K_c become column
// kernels (COL = true: a tile of adjacent columns staged through shared
// memory with coalesced row segments) and K_b runs on the natural rows --
// two kernels per step, no transposes (ssfm_capi.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dbp_block_kernel.cuh"

namespace dbp {

enum SimMode : int { kSimA = 0, kSimCA = 1, kSimC = 2, kSimB = 3, kSimFull = 4 };

struct SimParams {
  float2* data;             // rows of row_len samples, [item][pol][rows][row_len]
  long long pol_stride;     // n
  long long total_rows;     // rows * items (both polarisations handled per row)
  int rows;                 // rows per polarisation
  int log_n;                // log2 n
  int log_n1;               // log2 N1 (At row length)
  int mode;                 // SimMode
  const float2* tw;         // block-FFT twiddles of this row length
  const float2* wtab;       // W_n^{k1 n2} by row and position (A/CA: [n2][p], B: [p][n2])
  const float2* lin;        // kSimB: per-row permuted linear table [row][tab_index] ...
  const float2* lin_lo;     // ... as a double-float pair (hi, lo)
  float nl_a;               // rotation exp(+j nl_a I) (= -gamma dz_eff)
  float loss;               // amplitude factor per step ...
  float loss_last;          // ... and on the span's last step (kSimC), absorbing the
                            // float rounding of loss^(steps-1): the span gain is then
                            // exact to one rounding instead of drifting by steps ulp
  int nonlinear;
  int slice_floats;
  int n2;                   // column kernels: row stride / number of columns (N2)
  int steps;                // kSimFull: SSFM steps of the span, all in one launch
};

// x e^{-j gamma dz_eff (|x|^2 + |y|^2)} x loss (channel.py:61-71, 93); the
// partner lane (lane ^ 16) holds the other polarisation of the same sample
__device__ __forceinline__ void sim_nonlinear(float2 (&v)[16], const SimParams& sp, int pol, bool last) {
  const float loss = last ? sp.loss_last : sp.loss;
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const float own = fmaf(v[m].x, v[m].x, v[m].y * v[m].y);
    const float other = __shfl_xor_sync(0xffffffffu, own, 16);
    const float inten = pol ? other + own : own + other;
    v[m] = sp.nonlinear ? c_mul(v[m], rot_factor<true>(sp.nl_a, loss, inten))
                        : make_float2(v[m].x * loss, v[m].y * loss);
  }
}

// after fft_fwd over the At row n2: position p = t + T e holds bin k1(p)
template <int LOGN>
__device__ __forceinline__ void sim_twiddle_rows(float2 (&v)[16], const float2* __restrict__ w, int t) {
  constexpr int T = Geo<LOGN>::T;
#pragma unroll
  for (int e = 0; e < 16; ++e) v[e] = c_mul(v[e], ldg_table(w + t + T * e));
}

// Row kernels (COL = false): slice s of a CTA owns one contiguous row of
// ``row_len`` = 2^LOGN samples.  Column kernels (COL = true): the CTA owns a
// tile of BPC adjacent columns of the natural [N1][N2] layout (column length
// 2^LOGN = N1, row stride N2), loaded and stored with coalesced row
// segments through a padded shared-memory tile; slice s then holds column
// c0 + s in the same register layout as a row, so the four-step FFT needs no
// global transposes.
// Column tile width: the block-FFT slice count 2048 / N1.  (8 columns at
// N1 = 512 -- 64-byte row segments, 512-thread CTAs -- measured no faster
// than 4: 2^21 73.0 vs 68.6 us per step, tools/sim_sweep2.sh.)
__host__ __device__ constexpr int col_width(int logn) { return 1 << (11 - logn); }

template <int LOGN, bool COL>
struct SimShape {
  static constexpr int C = COL ? col_width(LOGN) : Geo<LOGN>::BPC;   // slices per CTA
  static constexpr int THREADS = 2 * Geo<LOGN>::T * C;
  static constexpr int MIN_CTAS = threads_per_sm(LOGN) / THREADS > 0 ? threads_per_sm(LOGN) / THREADS : 1;
};

template <int LOGN, bool COL>
__global__ void __launch_bounds__(SimShape<LOGN, COL>::THREADS, SimShape<LOGN, COL>::MIN_CTAS)
ssfm_row_kernel(const SimParams sp) {
  using G = Geo<LOGN>;
  constexpr int N = G::N, T = G::T, C = SimShape<LOGN, COL>::C, THREADS = SimShape<LOGN, COL>::THREADS;
  extern __shared__ float4 smem_raw[];
  const int lane = threadIdx.x & 31;
  const int pol = lane >> 4;
  const int q = ((threadIdx.x >> 5) << 4) + (lane & 15);
  const int t = q % T;
  const int slice = q / T;
  Shm<LOGN> sh;   // single region (the column tile aliases it)
  sh.init(reinterpret_cast<float*>(smem_raw) + slice * sp.slice_floats, sp.slice_floats, pol);

  float2 v[16];
  bool active;
  int row;            // W-table row: n2 (A/CA/C) or the register position p (B)
  float2* rp = nullptr;
  long long item = 0;
  int c0 = 0;
  if constexpr (COL) {
    // tile = (item, column group); columns c0 .. c0 + C - 1 of both polarisations
    const long long groups = sp.n2 / C;
    item = blockIdx.x / groups;
    c0 = (int)(blockIdx.x - item * groups) * C;
    active = true;
    row = c0 + slice;
    float2* tile = reinterpret_cast<float2*>(smem_raw);
    const float2* src = sp.data + item * 2 * sp.pol_stride + c0;
#pragma unroll 4
    for (int i = threadIdx.x; i < 2 * N * C; i += THREADS) {
      const int c = i % C, r = (i / C) % N, pl = i / (N * C);
      DBP_CHECK((pl * N + r) * (C + 1) + c < 2 * N * (C + 1));
      DBP_CHECK(item * 2 * sp.pol_stride + c0 + pl * sp.pol_stride + (long long)r * sp.n2 + c <
                (item + 1) * 2 * sp.pol_stride);
      tile[(pl * N + r) * (C + 1) + c] = src[pl * sp.pol_stride + (long long)r * sp.n2 + c];
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      DBP_CHECK((pol * N + t + T * m) * (C + 1) + slice < 2 * N * (C + 1));
      v[m] = tile[(pol * N + t + T * m) * (C + 1) + slice];
    }
    __syncthreads();   // the tile region is reused by the FFT exchange planes
  } else {
    const long long gr = (long long)blockIdx.x * G::BPC + slice;
    active = gr < sp.total_rows;
    item = active ? gr / sp.rows : 0;
    row = active ? (int)(gr - item * sp.rows) : 0;
    rp = sp.data + (item * 2 + pol) * sp.pol_stride + (long long)row * N + t;
    // natural (A, B) or register order (CA, C): both are position t + T m
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = active ? rp[T * m] : make_float2(0.f, 0.f);
  }

  if (sp.mode == kSimFull) {
    // whole waveform in this slice (n = row length <= 2^13): every step of
    // the span on-chip -- FFT, dispersion (double-float table, bins in
    // register order), inverse FFT, Manakov rotation and loss
    for (int k = 0; k < sp.steps; ++k) {
      const int tf = opaque(t);
      fft_fwd<LOGN, 0, 0>(v, sh, sp.tw, tf);
      apply_table_df<LOGN>(v, sp.lin, sp.lin_lo, G::NP == 1 ? 0 : tf);
      fft_inv<LOGN, 0, 0>(v, sh, sp.tw, opaque(t));
      sim_nonlinear(v, sp, pol, k + 1 == sp.steps);
    }
  } else if (sp.mode == kSimB) {
    fft_fwd<LOGN, 0, 0>(v, sh, sp.tw, t);
    apply_table_df<LOGN>(v, sp.lin + (long long)row * N, sp.lin_lo + (long long)row * N, G::NP == 1 ? 0 : t);
    const int ti = opaque(t);
    fft_inv<LOGN, 0, 0>(v, sh, sp.tw, ti);
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = c_mulc(v[m], ldg_table(sp.wtab + (long long)row * N + ti + T * m));
  } else {
    if (sp.mode != kSimA) {
      fft_inv<LOGN, 0, 0>(v, sh, sp.tw, t);
      sim_nonlinear(v, sp, pol, sp.mode == kSimC);
    }
    if (sp.mode != kSimC) {
      const int tf = opaque(t);
      fft_fwd<LOGN, 0, 0>(v, sh, sp.tw, tf);
      sim_twiddle_rows<LOGN>(v, sp.wtab + (long long)row * N, tf);
    }
  }
  if constexpr (COL) {
    float2* tile = reinterpret_cast<float2*>(smem_raw);
    __syncthreads();   // exchange planes -> tile
#pragma unroll
    for (int m = 0; m < 16; ++m) tile[(pol * N + t + T * m) * (C + 1) + slice] = v[m];
    __syncthreads();
    float2* dst = sp.data + item * 2 * sp.pol_stride + c0;
#pragma unroll 4
    for (int i = threadIdx.x; i < 2 * N * C; i += THREADS) {
      const int c = i % C, r = (i / C) % N, pl = i / (N * C);
      dst[pl * sp.pol_stride + (long long)r * sp.n2 + c] = tile[(pl * N + r) * (C + 1) + c];
    }
  } else if (active) {
#pragma unroll
    for (int m = 0; m < 16; ++m) rp[T * m] = v[m];
  }
}

// shared memory of a column-kernel CTA: the padded tile or the exchange planes
template <int LOGN>
inline size_t col_smem_bytes(size_t planes_bytes) {
  using G = Geo<LOGN>;
  const size_t tile = (size_t)2 * G::N * (col_width(LOGN) + 1) * sizeof(float2);
  return tile > planes_bytes ? tile : planes_bytes;
}

}  // namespace dbp
