// N = 8192 blocks as a radix-2 step around two 4096-point transforms held by
// the same thread ("R2" kernel).
//
// The pol-pair block kernel runs N = 8192 as R0 = 2 x 16^3: four passes, two
// CTA-wide exchanges (four barriers) per transform, every barrier spanning a
// 1024-thread CTA (profiles/r2/ncu_8192_ssfm20_summary.txt: MIO throttle and
// barrier stalls lead).  Here each thread of a 512-thread CTA holds 32 samples
// of each polarisation lane -- the even and the odd subsequence at positions
// 2 (t + 256 m) + a, a = 0, 1 -- and transforms both with the 4096-point
// machinery (16^3: ONE CTA-wide exchange plus one half-warp tile per
// transform, shared by the two subsequences).  The radix-2 step joining them
// never leaves the thread: with E, O the 4096-point spectra of the even and
// odd samples, X[k] = E[k] + W^k O[k], X[k + 4096] = E[k] - W^k O[k]
// (W = W_8192), and after the dispersion multiply K the inverse split is
// E' = X[k] + X[k + 4096], O' = W^-k (X[k] - X[k + 4096]), so
//
//   E' = A E + C O,  O' = D E + A O,
//   A = K[k] + K[k + 4096],  C = W^k (K[k] - K[k + 4096]),  D = W^-k (K[k] - K[k + 4096])
//
// with A, C, D tabled on the host from the float64 filter (1/N folded in).
// Per transform pair: two CTA-wide exchanges instead of four, half the
// barriers, each over 16 warps instead of 32.
#pragma once
#include "dbp_block_kernel.cuh"

// Measured against the pol-pair kernel (profiles/r2/r2/ab_r2a.txt): ESSFM
// 8192/1400 +13%, SSFM-20 8192/1024 +20%, N_s = 4 N_c = 33 +11%, N_s = 2
// N_c = 9 +12%; the FFE program keeps the polarisation-split pairs (R2 -6%).
// Default for every split-step program at N = 8192; env DBP_R2=0 (off) /
// 1 (also FFE) overrides.
#ifndef DBP_R2
#define DBP_R2 1
#endif
#ifndef DBP_R2_LOOP_BARRIER
#define DBP_R2_LOOP_BARRIER 0
#endif
#ifndef DBP_R2_TMA_STORE
#define DBP_R2_TMA_STORE 1    // kept centres out through shared memory and the TMA bulk engine
#endif
#ifndef DBP_R2_PAIR_STORE
#define DBP_R2_PAIR_STORE 1   // 16-byte (even, odd) output pairs; 0: 8-byte stores
#endif

namespace dbp {

struct R2Geo {
  static constexpr int N = 8192, H = 4096, T = 256, THREADS = 512;
  using G = Geo<12>;
  // exchange planes: [subsequence][pol] x plane_elems(4096) float2
  static constexpr int PLANE_FLOATS = 2 * plane_elems(4096);
};
inline int r2_slice_floats(int pw) {
  const int planes = 2 * 2 * R2Geo::PLANE_FLOATS;
  const int fir = fir_floats(R2Geo::N, pw);
  return ((planes > fir ? planes : fir) + 3) & ~3;
}

// acc + a b (two FFMA2)
__device__ __forceinline__ float2 c_mul_add(float2 a, float2 b, float2 acc) {
#if DBP_F32X2
  const unsigned long long t = f2_fma(f2_pack(a.x, a.x), f2_pack(b.x, b.y), f2_pack(acc.x, acc.y));
  return f2_unpack(f2_fma(f2_pack(-a.y, a.y), f2_pack(b.y, b.x), t));
#else
  return make_float2(fmaf(-a.y, b.y, fmaf(a.x, b.x, acc.x)), fmaf(a.y, b.x, fmaf(a.x, b.y, acc.y)));
#endif
}

template <int TWP>
__device__ __forceinline__ void r2_fft_fwd(float2 (&v)[2][16], Shm<12, kShmSync>& s0, Shm<12, kShmSync>& s1,
                                           const float2* __restrict__ tw, int t) {
  using G = Geo<12>;
  // pass 0: radix 16 over positions t + 256 e
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    dft<16, false>(v[a]);
    if constexpr (TWP != kTwDit) twiddle<16, false, true, TWP>(v[a], tw + 2 * t, 2 * 256);
  }
  DitBase nb = dit_zero();
  if constexpr (TWP == kTwDit) nb = dit_base(tw, G::dit_fwd_offset(1), t >> 4);
  __syncthreads();   // write-after-read: every warp is done with the region
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    float2* plane = (a ? s1 : s0).template plane<1>();
#pragma unroll
    for (int m = 0; m < 16; ++m) plane[side_index<12, 0>(t, m)] = v[a][m];
  }
  __syncthreads();
  const int base = ((t >> 4) << 8) + (t & 15);
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const float2* plane = (a ? s1 : s0).template plane<1>();
#pragma unroll
    for (int e = 0; e < 16; ++e) v[a][e] = plane[xchg_index<12, 0>(base + (e << 4))];
  }
  // pass 1, the half-warp tile, pass 2
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    if constexpr (TWP != kTwDit) {
      dft<16, false>(v[a]);
      twiddle<16, false, false, TWP>(v[a], tw + G::tw_offset(1) + 2 * (t & 15), 2 * 16);
    } else {
      dft_tw<16, false>(v[a], nb);
    }
  }
  DitBase nb2 = dit_zero();
  if constexpr (TWP == kTwDit) nb2 = dit_base(tw, G::dit_fwd_offset(2), t);
  const int l = t & 15;
  __syncwarp();
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    float2* tile = (a ? s1 : s0).template plane<1>() + kTileLen * (t >> 4);
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[l + kTilePitch * k] = v[a][k];
  }
  __syncwarp();
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const float2* tile = (a ? s1 : s0).template plane<1>() + kTileLen * (t >> 4);
#pragma unroll
    for (int e = 0; e < 16; e += 2) ld_pair(tile + kTilePitch * l + e, v[a][e], v[a][e + 1]);
    if constexpr (TWP != kTwDit) dft<16, false>(v[a]);
    else dft_tw<16, false>(v[a], nb2);
  }
}

template <int TWP>
__device__ __forceinline__ void r2_fft_inv(float2 (&v)[2][16], Shm<12, kShmSync>& s0, Shm<12, kShmSync>& s1,
                                           const float2* __restrict__ tw, int t) {
  using G = Geo<12>;
  const int l = t & 15;
#pragma unroll
  for (int a = 0; a < 2; ++a) dft<16, true>(v[a]);   // last pass first
  DitBase pb = dit_zero();
  if constexpr (TWP == kTwDit) pb = dit_base(tw, G::dit_inv_offset(1), t & 15);
  __syncwarp();
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    float2* tile = (a ? s1 : s0).template plane<1>() + kTileLen * (t >> 4);
#pragma unroll
    for (int e = 0; e < 16; e += 2) st_pair(tile + kTilePitch * l + e, v[a][e], v[a][e + 1]);
  }
  __syncwarp();
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const float2* tile = (a ? s1 : s0).template plane<1>() + kTileLen * (t >> 4);
#pragma unroll
    for (int k = 0; k < 16; ++k) v[a][k] = tile[l + kTilePitch * k];
    if constexpr (TWP != kTwDit) {
      twiddle<16, true, false, TWP>(v[a], tw + G::tw_offset(1) + 2 * (t & 15), 2 * 16);
      dft<16, true>(v[a]);
    } else {
      dft_tw<16, true>(v[a], pb);
    }
  }
  DitBase pre = dit_zero();
  if constexpr (TWP == kTwDit) pre = dit_base(tw, G::dit_inv_offset(0), t);
  __syncthreads();   // every warp has left the tiles (and the previous phase)
  const int base = ((t >> 4) << 8) + (t & 15);
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    float2* plane = (a ? s1 : s0).template plane<0>();
#pragma unroll
    for (int e = 0; e < 16; ++e) plane[xchg_index<12, 0>(base + (e << 4))] = v[a][e];
  }
  __syncthreads();
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const float2* plane = (a ? s1 : s0).template plane<0>();
#pragma unroll
    for (int m = 0; m < 16; ++m) v[a][m] = plane[side_index<12, 0>(t, m)];
    if constexpr (TWP != kTwDit) {
      twiddle<16, true, true, TWP>(v[a], tw + 2 * t, 2 * 256);
      dft<16, true>(v[a]);
    } else {
      dft_tw<16, true>(v[a], pre);
    }
  }
}

// forward transforms, the 2 x 2 radix-2 / dispersion / inverse-split step, inverse transforms
template <int TWP>
__device__ __forceinline__ void r2_conv(float2 (&v)[2][16], Shm<12, kShmSync>& s0, Shm<12, kShmSync>& s1,
                                        const float2* __restrict__ tab, const float2* __restrict__ tw, int t) {
  r2_fft_fwd<TWP>(v, s0, s1, tw, t);
#pragma unroll
  for (int e = 0; e < 16; e += 2) {
    float2 a0, a1, c0, c1, d0, d1;
    ldg_table_pair(tab + tab_index(12, t, e), a0, a1);
    ldg_table_pair(tab + R2Geo::H + tab_index(12, t, e), c0, c1);
    ldg_table_pair(tab + 2 * R2Geo::H + tab_index(12, t, e), d0, d1);
    const float2 e0 = v[0][e], o0 = v[1][e], e1 = v[0][e + 1], o1 = v[1][e + 1];
    v[0][e] = c_mul_add(c0, o0, c_mul(a0, e0));
    v[1][e] = c_mul_add(a0, o0, c_mul(d0, e0));
    v[0][e + 1] = c_mul_add(c1, o1, c_mul(a1, e1));
    v[1][e + 1] = c_mul_add(a1, o1, c_mul(d1, e1));
  }
  r2_fft_inv<TWP>(v, s0, s1, tw, opaque(t));
}

// Nonlinear step (dbp.py:63-70 / 72-80) on positions n = 2 (t + 256 m) + a.
// Each lane of an x/y pair forms the total intensity of half the positions
// (m = 8 pol .. 8 pol + 7), every lane produces 16 FIR outputs, the
// factors come back through shared memory as (n, n + 1) pairs.
template <int PROG>
__device__ __forceinline__ void r2_rotate(float2 (&v)[2][16], float* smem, const KernelParams& kp, int step_idx,
                                          int t, int pol, const float* __restrict__ cptr) {
  constexpr int N = R2Geo::N;
  const float c0 = kp.coeff_stride ? __ldg(cptr) : kp.c[0];
  const float2 sg = __ldg(kp.steps + step_idx);
  float inten[2][8];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const float lo = fmaf(v[a][m].x, v[a][m].x, v[a][m].y * v[a][m].y);
      const float hi = fmaf(v[a][m + 8].x, v[a][m + 8].x, v[a][m + 8].y * v[a][m + 8].y);
      const float other = __shfl_xor_sync(0xffffffffu, pol ? lo : hi, 16);
      inten[a][m] = (pol ? hi : lo) + other;
    }
  if (PROG == kProgNoFir || kp.nc == 0) {
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float2 mine = kp.precise_sincos ? rot_factor<true>(sg.x, sg.y, c0 * inten[a][i])
                                              : rot_factor<false>(sg.x, sg.y, c0 * inten[a][i]);
        const float2 oth = make_float2(__shfl_xor_sync(0xffffffffu, mine.x, 16),
                                       __shfl_xor_sync(0xffffffffu, mine.y, 16));
        v[a][i] = c_mul(v[a][i], pol ? oth : mine);
        v[a][8 + i] = c_mul(v[a][8 + i], pol ? mine : oth);
      }
    return;
  }
  const int pw = kp.fir_pad;
  float* ibuf = smem;
  float* nlbuf = ibuf + fir_phys(N + 2 * pw) + 4;
  __syncthreads();   // the exchange planes (aliased) are free
  const int m0 = 8 * pol;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int j = 2 * (t + 256 * (m0 + m));   // even position; (j, j + 1) share a 16-float group (pw % 4 == 0)
    *reinterpret_cast<float2*>(ibuf + fir_phys(j + pw)) = make_float2(inten[0][m], inten[1][m]);
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int n = j + a;
      if (n < pw) ibuf[fir_phys(n + N + pw)] = inten[a][m];
      if (n >= N - pw) ibuf[fir_phys(n - N + pw)] = inten[a][m];
    }
  }
  __syncthreads();
  constexpr bool kDirectFir = DBP_FIR_DIRECT;
  // outputs p0 .. p0 + 7 with p0 = 16 (t + 256 h) + 8 pol: consecutive lanes
  // 16 positions apart, so each quarter warp's 16-byte window reads hit eight
  // distinct bank groups (fir_phys stride 20 floats) as in the pol-pair kernel
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    const int p0 = 16 * (t + 256 * h) + 8 * pol;
    switch (kp.coeff_stride ? -1 : kp.nc) {
      case 1: fir8_fixed<1, kDirectFir>(ibuf, nlbuf, p0, sg.x, sg.y, kp, N, true); break;
      case 9: fir8_fixed<9, kDirectFir>(ibuf, nlbuf, p0, sg.x, sg.y, kp, N, true); break;
      case 17: fir8_fixed<17, kDirectFir>(ibuf, nlbuf, p0, sg.x, sg.y, kp, N, true); break;
      case 32: fir8_fixed<32, kDirectFir>(ibuf, nlbuf, p0, sg.x, sg.y, kp, N, true); break;
      case 33: fir8_fixed<33, kDirectFir>(ibuf, nlbuf, p0, sg.x, sg.y, kp, N, true); break;
      default:
        if constexpr (PROG == kProgGenericFir) fir8_generic(ibuf, nlbuf, p0, pw, sg.x, sg.y, kp, cptr, c0, true);
        else __trap();
        break;
    }
  }
  __syncthreads();
  const float2* cs = reinterpret_cast<const float2*>(nlbuf);
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int j = 2 * (t + 256 * m);
    const float4 f = *reinterpret_cast<const float4*>(cs + cs_phys(j));
    v[0][m] = c_mul(v[0][m], make_float2(f.x, f.y));
    v[1][m] = c_mul(v[1][m], make_float2(f.z, f.w));
  }
}

template <int PROG, int TWP>
__global__ void __launch_bounds__(R2Geo::THREADS, 1) dbp_r2_kernel(const KernelParams kp) {
  constexpr int N = R2Geo::N, T = R2Geo::T;
  extern __shared__ float4 smem_raw[];
  const int lane = threadIdx.x & 31;
  const int pol = lane >> 4;
  const int t = ((threadIdx.x >> 5) << 4) + (lane & 15);
  float* smem = reinterpret_cast<float*>(smem_raw);
  Shm<12, kShmSync> s0, s1;
  s0.init(smem, kp.slice_floats, pol);
  s1.init(smem + 2 * R2Geo::PLANE_FLOATS, kp.slice_floats, pol);
  const float2* tw = kp.r2_tw;
  for (long long blk = blockIdx.x; blk < kp.total_blocks; blk += gridDim.x) {
    const long long item = kp.bpi_magic ? (long long)__umul64hi(kp.bpi_magic, (unsigned long long)blk)
                                        : blk / kp.blocks_per_item;
    const long long b = kp.block_begin + (blk - item * kp.blocks_per_item);
    const float* cptr = kp.coeff + (kp.coeff_stride ? item * kp.coeff_stride : 0);
    const float2* pin = kp.in + item * kp.in_item_stride + pol * kp.in_pol_stride;
    const long long s0i = b * kp.step - kp.lead;
    float2 v[2][16];
    if (!kp.cyclic || (s0i >= 0 && s0i + N <= kp.n_total)) {
      const float2* src = pin + (kp.cyclic ? s0i : s0i - kp.in_origin);
      if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          float4 q;
          asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w)
                       : "l"(src + 2 * (t + T * m)));
          v[0][m] = make_float2(q.x, q.y);
          v[1][m] = make_float2(q.z, q.w);
        }
      } else {
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          v[0][m] = ld_stream(src + 2 * (t + T * m));
          v[1][m] = ld_stream(src + 2 * (t + T * m) + 1);
        }
      }
    } else {
#pragma unroll
      for (int m = 0; m < 16; ++m)
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          long long gi = s0i + 2 * (t + T * m) + a;
          if (gi < 0 || gi >= kp.n_total) {
            gi %= kp.n_total;
            if (gi < 0) gi += kp.n_total;
          }
          v[a][m] = ld_stream(pin + gi);
        }
    }
    if (blk + gridDim.x < kp.total_blocks) {
      // L2 prefetch of the next block: one 128-byte line per thread and polarisation
      const long long nblk = blk + gridDim.x;
      const long long nitem = kp.bpi_magic ? (long long)__umul64hi(kp.bpi_magic, (unsigned long long)nblk)
                                           : nblk / kp.blocks_per_item;
      const long long nb = kp.block_begin + (nblk - nitem * kp.blocks_per_item);
      const long long ns0 = nb * kp.step - kp.lead;
      if (!kp.cyclic || (ns0 >= 0 && ns0 + N <= kp.n_total)) {
        const float2* pn = kp.in + nitem * kp.in_item_stride + pol * kp.in_pol_stride +
                           (kp.cyclic ? ns0 : ns0 - kp.in_origin) + 32 * t;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pn));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pn + 16));
      }
    }

    if constexpr (PROG == kProgFFE) {
      r2_conv<TWP>(v, s0, s1, kp.r2_full, tw, t);
    } else {
      const int n_ops = kp.n_ops;
      for (int op = 0; op < n_ops; ++op) {
        const bool is_conv = kp.conv_all || (op & 1) == kp.conv_parity;
        const float2* tab = kp.half_ends && (op == 0 || op == n_ops - 1) ? kp.r2_half : kp.r2_full;
        if (is_conv) r2_conv<TWP>(v, s0, s1, tab, tw, t);
        else r2_rotate<PROG>(v, smem, kp, op >> kp.sidx_shift, t, pol, cptr);
      }
    }

    float2* pout = kp.out + item * kp.out_item_stride + pol * kp.out_pol_stride;
    const long long ob = b * kp.step - kp.lead - kp.out_origin;
    const long long rem = kp.n_total - b * kp.step;
    const int hi = kp.lead + (rem < kp.step ? (int)rem : kp.step);
    // positions 2 (t + 256 m) + a: the even / odd pair is adjacent in the output
    // row, so it leaves as one coalesced 16-byte store when the kept range and
    // the row are pair-aligned (8-byte stores, half a warp's sectors each, held
    // the LSU queue: lg_throttle was the top memory stall, profiles/r2/r2/)
    const bool pairs = DBP_R2_PAIR_STORE && ((ob | kp.lead | hi) & 1) == 0 &&
                       (reinterpret_cast<uintptr_t>(pout + ob) & 15) == 0;
    // TMA bulk store (CTA-uniform condition): the kept centres of both
    // polarisations staged in the free exchange planes as [pol][step], two
    // bulk copies issued by one thread, which alone waits for the engine to
    // have read them (the loop's closing barrier then frees the planes)
    float2* row_x = kp.out + item * kp.out_item_stride + (b * kp.step - kp.out_origin);
    const int len = hi - kp.lead;
    // (step even: the y row's staging starts 16-byte aligned; len even: whole 16-byte units)
    const bool bulk = DBP_R2_TMA_STORE && ((len | kp.lead | kp.step) & 1) == 0 && (kp.out_pol_stride & 1) == 0 &&
                      (reinterpret_cast<uintptr_t>(row_x) & 15) == 0;
    if (bulk) {
      __syncthreads();   // every warp has left the planes
      float2* stg = reinterpret_cast<float2*>(smem) + pol * kp.step - kp.lead;
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const int j = 2 * (t + T * m);
        if (j >= kp.lead && j < hi)
          *reinterpret_cast<float4*>(stg + j) = make_float4(v[0][m].x, v[0][m].y, v[1][m].x, v[1][m].y);
      }
      fence_proxy_async_smem();
      __syncthreads();
      if (threadIdx.x == 0) {
        const float2* src = reinterpret_cast<const float2*>(smem);
        bulk_store(row_x, src, (uint32_t)len * 8u);
        bulk_store(row_x + kp.out_pol_stride, src + kp.step, (uint32_t)len * 8u);
        bulk_store_commit_and_wait_read();
      }
    } else if (pairs) {
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const int j = 2 * (t + T * m);
        if (j >= kp.lead && j < hi)
          __stcs(reinterpret_cast<float4*>(pout + ob + j), make_float4(v[0][m].x, v[0][m].y, v[1][m].x, v[1][m].y));
      }
    } else {
#pragma unroll
      for (int m = 0; m < 16; ++m)
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const int j = 2 * (t + T * m) + a;
          if (j >= kp.lead && j < hi) __stcs(pout + ob + j, v[a][m]);
        }
    }
#if DBP_R2_LOOP_BARRIER
    __syncthreads();   // the next block's first exchange reuses the planes
#endif
    // (no barrier needed here: every first shared-memory write of the next
    // block -- the forward exchange, the FIR buffers, the store staging --
    // sits behind its own __syncthreads, which thread 0 reaches only after
    // its bulk store has read the staging)
  }
}

// host: the R2 step tables for a float64 filter K (natural bin order, re/im
// interleaved) of the 8192-point block: [A | C | D], each in the 4096-point
// kernel's e-paired register order, 1/N folded in
inline std::vector<float2> make_r2_tables(const double* k) {
  const int n = R2Geo::N, h = R2Geo::H;
  std::vector<float2> out(3 * h);
  for (int t = 0; t < h / 16; ++t)
    for (int e = 0; e < 16; ++e) {
      const int kk = last_pass_bin(12, t, e), idx = tab_index(12, t, e);
      const double lr = k[2 * kk] / n, li = k[2 * kk + 1] / n;
      const double hr = k[2 * (kk + h)] / n, hi = k[2 * (kk + h) + 1] / n;
      const double ar = lr + hr, ai = li + hi, br = lr - hr, bi = li - hi;
      const double ang = -2.0 * M_PI * kk / n, wr = std::cos(ang), wi = std::sin(ang);
      out[idx] = make_float2((float)ar, (float)ai);
      out[h + idx] = make_float2((float)(wr * br - wi * bi), (float)(wr * bi + wi * br));
      out[2 * h + idx] = make_float2((float)(wr * br + wi * bi), (float)(wr * bi - wi * br));
    }
  return out;
}

}  // namespace dbp
