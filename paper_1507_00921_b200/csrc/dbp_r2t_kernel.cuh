// N = 8192 blocks, two CTAs per SM: the R2 kernel's radix-2 step around two
// 4096-point transforms, with the subsequence a thread is not transforming
// parked in tensor memory ("R2T" kernel).
//
// The R2 kernel (dbp_r2_kernel.cuh) holds both 16-sample subsequences of a
// thread in registers: 128 registers, one 512-thread CTA per SM, so an SM has
// no second block to overlap with while a block waits at its exchange
// barriers (profiles/r2/ab_onecta.txt: that overlap is worth 25-40% at
// N = 2048 / 4096).  An 8192-sample dual-polarisation block is 128 KB, half
// the register file -- but the subsequence that is not being transformed
// only needs to be kept, not computed on, and TMEM (256 KB per SM, private
// to its lane, otherwise idle on this path) keeps it: each thread parks 16
// complex samples (32 columns of its TMEM lane) with one tcgen05.st and takes
// them back with one tcgen05.ld.  The live set is then exactly the 4096-point
// kernel's (16 samples, 64 registers), the exchange planes hold one
// subsequence (70 KB), and two CTAs fit an SM.
//
// Per transform pair (dbp.py:188-189 / 196-223 on the two subsequences
// E, O of positions 2 (t + 256 m) + a; see dbp_r2_kernel.cuh for the step):
//   live c: forward(c) -> park in Q; take the other from P; forward;
//   join with the R2 tables (R' = A R + X S, S' = A S + Y R, S streamed from Q
//   four samples at a time); inverse(R') -> park in P; take S' from Q;
//   inverse.  Both subsequences take the same 4096-point passes (fft_fwd /
//   fft_inv of dbp_block_kernel.cuh), so results equal the R2 kernel's up to
//   the rounding of the join.
// Nonlinear step: the intensities of both subsequences go to shared memory
// (one parked meanwhile), the FIR publishes F (4 bytes per position: the
// factor buffer would not leave room for two CTAs), each subsequence is
// rotated while live.  SSFM (no FIR): each subsequence is rotated while live
// from its own and the partner lane's |v|^2, and the two swap roles.
//
// Measured (profiles/r2/r2t/): parity-correct (the N = 8192 parity subset
// under DBP_R2T=2), but slower than the R2 kernel -- ESSFM 8192/1400 33.1 vs
// 36.4 GS/s, SSFM-20 8192/1024 3.70 vs 4.66, N_s = 4 N_c = 33 10.9 vs 13.4,
// FFE 46.2 vs 70.8.  Two CTAs per SM do run (32 warps), but the 4096-point
// passes alone already fill 64 registers (a bare forward/table/inverse
// kernel spills 12 bytes), so the parked-slot bookkeeping and the join spill
// 250-700 bytes per thread; the spill traffic (1024 threads x ~0.5 KB per SM)
// does not fit L1 next to 166 KB of shared memory and goes to L2 and DRAM
// (SSFM-20: 18.4 GB written per launch instead of 2.1).  Off by default;
// DBP_R2T=1 (split-step programs) / 2 (every program) selects it.
#pragma once
#include "dbp_r2_kernel.cuh"

#ifndef DBP_R2T
#define DBP_R2T 0
#endif

namespace dbp {

struct R2TGeo {
  static constexpr int N = 8192, H = 4096, T = 256, THREADS = 512;
  static constexpr int TMEM_COLS = 256;   // 4 warps per TMEM lane quarter x 2 slots x 32 columns
};

inline int r2t_slice_floats(int pw) {
  const int planes = 2 * 2 * plane_elems(4096);                 // one Shm<12>: 2 polarisation planes of float2
  const int fir = fir_phys(R2TGeo::N + 2 * pw) + 4 + fir_phys(R2TGeo::N) + 4;   // intensity + published F
  return ((planes > fir ? planes : fir) + 3) & ~3;
}

// ---- tensor memory: lane-private parking of 16 complex samples -------------
// in 8-column pieces: a 32-column tcgen05.ld / st needs 32 contiguous
// registers, which a 64-register thread cannot spare next to its other state
__device__ __forceinline__ void tm_st4(uint32_t taddr, float2 a, float2 b, float2 c, float2 d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y), "f"(d.x), "f"(d.y)
               : "memory");
}
__device__ __forceinline__ void tm_ld4_nowait(uint32_t taddr, float2& a, float2& b, float2& c, float2& d) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(b.x), "=f"(b.y), "=f"(c.x), "=f"(c.y), "=f"(d.x), "=f"(d.y)
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_ld4(uint32_t taddr, float2& a, float2& b, float2& c, float2& d) {
  tm_ld4_nowait(taddr, a, b, c, d);
  tm_wait_ld();
}
__device__ __forceinline__ void tm_st16(uint32_t taddr, const float2 (&v)[16]) {
#pragma unroll
  for (int e = 0; e < 16; e += 4) tm_st4(taddr + 2 * e, v[e], v[e + 1], v[e + 2], v[e + 3]);
}
__device__ __forceinline__ void tm_ld16(uint32_t taddr, float2 (&v)[16]) {
#pragma unroll
  for (int e = 0; e < 16; e += 4) tm_ld4_nowait(taddr + 2 * e, v[e], v[e + 1], v[e + 2], v[e + 3]);
  tm_wait_ld();
}
// every earlier tcgen05.st of this thread has landed (before reading a slot back)
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Slot addresses are rebuilt from shared memory at each use instead of being
// kept in registers through the transforms (the 64-register budget is the
// 4096-point kernel's): this warp's TMEM lane quarter (warp % 4), its
// 64-column pair (warp / 4), slot k at column 32 k.
__device__ __forceinline__ uint32_t tm_slot(const uint32_t* base_sh, int k) {
  uint32_t base, tid;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(base) : "r"((uint32_t)__cvta_generic_to_shared(base_sh)));
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
  const uint32_t warp = tid >> 5;
  return base + ((32u * (warp & 3u)) << 16) + 64u * (warp >> 2) + 32u * (uint32_t)k;
}

// swap the live subsequence with the one parked at `from`, parking the live one at `to`
__device__ __forceinline__ void tm_swap(float2 (&v)[16], uint32_t to, uint32_t from) {
  tm_st16(to, v);
  tm_wait_st();   // `from` may have been written by an earlier st of this thread
  tm_ld16(from, v);
}

// forward transforms of both subsequences, the radix-2 join with the filter,
// inverse transforms; the live subsequence (parity la) stays live, the other
// stays parked at slot P; slot Q is scratch
template <int TWP>
__device__ __forceinline__ void r2t_conv(float2 (&v)[16], Shm<12, kShmSync>& sh, const float2* __restrict__ tab,
                                         const float2* __restrict__ tw, int t, int la, const uint32_t* tb) {
  // the parked subsequence is in slot la (P), slot 1 - la (Q) is scratch
  fft_fwd<12, 0, TWP>(v, sh, tw, t);
  tm_swap(v, tm_slot(tb, 1 - la), tm_slot(tb, la));   // spectrum of the live one to Q; the other one's samples
  fft_fwd<12, 0, TWP>(v, sh, tw, opaque(t));   // (opaque: no addresses kept live across the first)
  // registers: R = spectrum of the other subsequence (parity 1 - la); Q: S (parity la)
  // E' = A E + C O, O' = D E + A O:  R' = A R + X S, S' = A S + Y R with
  // (X, Y) = (C, D) when R is E (la == 1), (D, C) when R is O (la == 0)
  const float2* tx = tab + (la ? R2Geo::H : 2 * R2Geo::H);
  const float2* ty = tab + (la ? 2 * R2Geo::H : R2Geo::H);
  tm_wait_st();
#pragma unroll
  for (int e = 0; e < 16; e += 4) {
    float2 s[4];
    const uint32_t Q = tm_slot(tb, 1 - la);
    tm_ld4(Q + 2 * e, s[0], s[1], s[2], s[3]);
#pragma unroll
    for (int k = 0; k < 4; k += 2) {
      float2 a0, a1, x0, x1, y0, y1;
      ldg_table_pair(tab + tab_index(12, t, e + k), a0, a1);
      ldg_table_pair(tx + tab_index(12, t, e + k), x0, x1);
      ldg_table_pair(ty + tab_index(12, t, e + k), y0, y1);
      const float2 r0 = v[e + k], r1 = v[e + k + 1];
      v[e + k] = c_mul_add(x0, s[k], c_mul(a0, r0));
      v[e + k + 1] = c_mul_add(x1, s[k + 1], c_mul(a1, r1));
      s[k] = c_mul_add(a0, s[k], c_mul(y0, r0));
      s[k + 1] = c_mul_add(a1, s[k + 1], c_mul(y1, r1));
    }
    tm_st4(Q + 2 * e, s[0], s[1], s[2], s[3]);
  }
  fft_inv<12, 0, TWP>(v, sh, tw, opaque(t));
  tm_swap(v, tm_slot(tb, la), tm_slot(tb, 1 - la));   // the other one back to P; S' live
  fft_inv<12, 0, TWP>(v, sh, tw, opaque(t));
}

// |v|^2 of this lane's positions m = 8 pol .. 8 pol + 7 plus the partner lane's
__device__ __forceinline__ void r2t_intensity(const float2 (&v)[16], float (&inten)[8], int pol) {
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const float lo = fmaf(v[m].x, v[m].x, v[m].y * v[m].y);
    const float hi = fmaf(v[m + 8].x, v[m + 8].x, v[m + 8].y * v[m + 8].y);
    const float other = __shfl_xor_sync(0xffffffffu, pol ? lo : hi, 16);
    inten[m] = (pol ? hi : lo) + other;
  }
}

// SSFM sub-step (F = c0 I) on the live subsequence: each lane of an x/y pair
// evaluates half the factors, then they swap (as the block kernel)
__device__ __forceinline__ void r2t_rotate_local(float2 (&v)[16], float a, float g, float c0, int pol,
                                                 bool precise) {
  float inten[8];
  r2t_intensity(v, inten, pol);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float2 mine = precise ? rot_factor<true>(a, g, c0 * inten[i]) : rot_factor<false>(a, g, c0 * inten[i]);
    const float2 oth = make_float2(__shfl_xor_sync(0xffffffffu, mine.x, 16),
                                   __shfl_xor_sync(0xffffffffu, mine.y, 16));
    v[i] = c_mul(v[i], pol ? oth : mine);
    v[8 + i] = c_mul(v[8 + i], pol ? mine : oth);
  }
}

// the live subsequence's intensities into the padded cyclic intensity buffer
__device__ __forceinline__ void r2t_store_intensity(float* ibuf, const float2 (&v)[16], int t, int pol, int a,
                                                    int pw) {
  constexpr int N = R2TGeo::N;
  float inten[8];
  r2t_intensity(v, inten, pol);
  const int m0 = 8 * pol;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int n = 2 * (t + 256 * (m0 + m)) + a;
    ibuf[fir_phys(n + pw)] = inten[m];
    if (n < pw) ibuf[fir_phys(n + N + pw)] = inten[m];
    if (n >= N - pw) ibuf[fir_phys(n - N + pw)] = inten[m];
  }
}

template <bool PRECISE>
__device__ __forceinline__ void r2t_rotate_by_f(float2 (&v)[16], const float* fbuf, int t, int a, float sa,
                                                float g) {
  float fv[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) fv[m] = fbuf[fir_phys(2 * (t + 256 * m) + a)];
  rotate_by_f<PRECISE>(v, fv, sa, g);
}

// ESSFM sub-step (dbp.py:63-75): both subsequences' intensities, the FIR over
// the block (each lane 16 outputs, as the R2 kernel), F published, each
// subsequence rotated while live.  Live parity and slots are unchanged on exit.
template <int PROG>
__device__ __forceinline__ void r2t_rotate_fir(float2 (&v)[16], float* smem, const KernelParams& kp, float2 sg,
                                               int t, int pol, int la, const uint32_t* tb,
                                               const float* __restrict__ cptr, float c0) {
  constexpr int N = R2TGeo::N;
  const int pw = kp.fir_pad;
  float* ibuf = smem;
  float* fbuf = ibuf + fir_phys(N + 2 * pw) + 4;
  __syncthreads();   // the exchange planes (aliased) are free
  r2t_store_intensity(ibuf, v, t, pol, la, pw);
  tm_swap(v, tm_slot(tb, 1 - la), tm_slot(tb, la));
  r2t_store_intensity(ibuf, v, t, pol, 1 - la, pw);
  __syncthreads();
  constexpr bool kDirectFir = DBP_FIR_DIRECT;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    const int p0 = 16 * (t + 256 * h) + 8 * pol;
    switch (kp.coeff_stride ? -1 : kp.nc) {
      case 1: fir8_fixed<1, kDirectFir>(ibuf, fbuf, p0, sg.x, sg.y, kp, N, false); break;
      case 9: fir8_fixed<9, kDirectFir>(ibuf, fbuf, p0, sg.x, sg.y, kp, N, false); break;
      case 17: fir8_fixed<17, kDirectFir>(ibuf, fbuf, p0, sg.x, sg.y, kp, N, false); break;
      case 32: fir8_fixed<32, kDirectFir>(ibuf, fbuf, p0, sg.x, sg.y, kp, N, false); break;
      case 33: fir8_fixed<33, kDirectFir>(ibuf, fbuf, p0, sg.x, sg.y, kp, N, false); break;
      default:
        if constexpr (PROG == kProgGenericFir) fir8_generic(ibuf, fbuf, p0, pw, sg.x, sg.y, kp, cptr, c0, false);
        else __trap();
        break;
    }
  }
  __syncthreads();
  if (kp.precise_sincos) {
    r2t_rotate_by_f<true>(v, fbuf, t, 1 - la, sg.x, sg.y);
    tm_swap(v, tm_slot(tb, la), tm_slot(tb, 1 - la));
    r2t_rotate_by_f<true>(v, fbuf, t, la, sg.x, sg.y);
  } else {
    r2t_rotate_by_f<false>(v, fbuf, t, 1 - la, sg.x, sg.y);
    tm_swap(v, tm_slot(tb, la), tm_slot(tb, 1 - la));
    r2t_rotate_by_f<false>(v, fbuf, t, la, sg.x, sg.y);
  }
}

__device__ __forceinline__ long long opaque64(long long x) {
  long long y;
  asm volatile("mov.b64 %0, %1;" : "=l"(y) : "l"(x));
  return y;
}
__device__ __forceinline__ void r2t_locate(const KernelParams& kp, long long blk, long long& item, long long& b) {
  item = kp.bpi_magic ? (long long)__umul64hi(kp.bpi_magic, (unsigned long long)blk) : blk / kp.blocks_per_item;
  b = kp.block_begin + (blk - item * kp.blocks_per_item);
}

template <int PROG, int TWP>
__global__ void __launch_bounds__(R2TGeo::THREADS, 2) dbp_r2t_kernel(const KernelParams kp) {
  static_assert(DBP_NL_PUBLISH_F, "the R2T kernel publishes F");
  constexpr int N = R2TGeo::N, T = R2TGeo::T;
  extern __shared__ float4 smem_raw[];
  __shared__ uint32_t tmem_base_sh;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int pol = lane >> 4;
  const int t = (warp << 4) + (lane & 15);
  float* smem = reinterpret_cast<float*>(smem_raw);
  Shm<12, kShmSync> sh;
  sh.init(smem, kp.slice_floats, pol);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base_sh)),
                 "n"(R2TGeo::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const float2* tw = kp.r2_tw;
  for (long long blk = blockIdx.x; blk < kp.total_blocks; blk += gridDim.x) {
    long long item, b;
    r2t_locate(kp, blk, item, b);
    const float* cptr = kp.coeff + (kp.coeff_stride ? item * kp.coeff_stride : 0);
    const float2* pin = kp.in + item * kp.in_item_stride + pol * kp.in_pol_stride;
    const long long s0i = b * kp.step - kp.lead;
    // la: parity of the live subsequence; the other one is parked in TMEM
    // slot la (P), slot 1 - la is scratch (Q) -- the two flip together
    int la = 0;
    float2 v[16];
    // load: the odd subsequence first (parked), then the even one
    if (!kp.cyclic || (s0i >= 0 && s0i + N <= kp.n_total)) {
      const float2* src = pin + (kp.cyclic ? s0i : s0i - kp.in_origin) + 2 * t;
#pragma unroll
      for (int m = 0; m < 16; ++m) v[m] = ld_stream(src + 2 * T * m + 1);
      tm_st16(tm_slot(&tmem_base_sh, la), v);
#pragma unroll
      for (int m = 0; m < 16; ++m) v[m] = ld_stream(src + 2 * T * m);
    } else {
      // cyclic edge block (rare): each subsequence of both polarisations is
      // staged through the exchange planes by a compact loop, odd one first
      const float2* pin0 = kp.in + item * kp.in_item_stride;
      float2* stage = reinterpret_cast<float2*>(smem);   // [2][4096] <= one Shm<12>
      for (int a = 1; a >= 0; --a) {
        __syncthreads();
#pragma unroll 1
        for (int i = threadIdx.x; i < 2 * R2TGeo::H; i += R2TGeo::THREADS) {
          long long gi = s0i + 2 * (i & (R2TGeo::H - 1)) + a;
          gi %= kp.n_total;
          if (gi < 0) gi += kp.n_total;
          stage[i] = ld_stream(pin0 + (i >> 12) * kp.in_pol_stride + gi);
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = stage[pol * R2TGeo::H + t + T * m];
        if (a) tm_st16(tm_slot(&tmem_base_sh, la), v);
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
      r2t_conv<TWP>(v, sh, kp.r2_full, tw, t, la, &tmem_base_sh);
    } else {
      const float c0 = kp.coeff_stride ? __ldg(cptr) : kp.c[0];
      const int n_ops = kp.n_ops;
      for (int op = 0; op < n_ops; ++op) {
        const bool is_conv = kp.conv_all || (op & 1) == kp.conv_parity;
        const float2* tab = kp.half_ends && (op == 0 || op == n_ops - 1) ? kp.r2_half : kp.r2_full;
        if (is_conv) {
          r2t_conv<TWP>(v, sh, tab, tw, t, la, &tmem_base_sh);
        } else {
          const float2 sg = __ldg(kp.steps + (op >> kp.sidx_shift));
          if (PROG == kProgNoFir || kp.nc == 0) {
            // rotate the live one, swap, rotate the other: the two exchange roles
            r2t_rotate_local(v, sg.x, sg.y, c0, pol, kp.precise_sincos);
            tm_swap(v, tm_slot(&tmem_base_sh, 1 - la), tm_slot(&tmem_base_sh, la));
            r2t_rotate_local(v, sg.x, sg.y, c0, pol, kp.precise_sincos);
            la ^= 1;
          } else {
            r2t_rotate_fir<PROG>(v, smem, kp, sg, t, pol, la, &tmem_base_sh, cptr, c0);
          }
        }
      }
    }

    // the block's coordinates again (recomputed, not kept live through the program)
    r2t_locate(kp, opaque64(blk), item, b);
    float2* pout = kp.out + item * kp.out_item_stride + pol * kp.out_pol_stride;
    const long long ob = b * kp.step - kp.lead - kp.out_origin;
    const long long rem = kp.n_total - b * kp.step;
    const int hi = kp.lead + (rem < kp.step ? (int)rem : kp.step);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int j = 2 * (t + T * m) + la;
      if (j >= kp.lead && j < hi) __stcs(pout + ob + j, v[m]);
    }
    tm_wait_st();
    tm_ld16(tm_slot(&tmem_base_sh, la), v);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int j = 2 * (t + T * m) + 1 - la;
      if (j >= kp.lead && j < hi) __stcs(pout + ob + j, v[m]);
    }
    __syncthreads();   // the next block's first exchange reuses the planes
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh), "n"(R2TGeo::TMEM_COLS)
                 : "memory");
}

}  // namespace dbp
