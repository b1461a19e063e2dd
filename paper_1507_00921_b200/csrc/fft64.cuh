// Batched float64 complex FFT for the off-hot-path spectral utilities
// (spectral.fft / ifft, pkg/src/fiberdbp/spectral.py:37-48) and the receiver's
// carrier-recovery spectra and correlations (modem.py:305-351): a Stockham
// autosort transform, radix 4 (one radix-2 pass first when log2 n is odd),
// one global-memory pass per radix step, twiddles from sincospi in float64.
// Replaces cuFFT so the product library links no FFT library; accuracy is
// that of a float64 radix-4 FFT (~1e-15 relative, like numpy's pocketfft).
#pragma once
#include <cuda_runtime.h>

namespace fft64 {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// multiply by -j (forward) / +j (inverse)
__device__ __forceinline__ double2 crot(double2 a, bool inv) {
  return inv ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// One Stockham pass of radix R over `batch` rows of length n: thread (row, j),
// j < n / R; inputs at stride n / R, outputs at stride ns (the current
// sub-transform length), twiddle W_{R ns}^{k r}, k = j mod ns.
template <int R>
__global__ void stockham_pass(const double2* __restrict__ in, double2* __restrict__ out, long long n,
                              long long ns, long long total, int inverse) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= total) return;
  const long long q = n / R;
  const long long row = tid / q, j = tid - row * q;
  const double2* src = in + row * n;
  double2* dst = out + row * n;
  const long long k = j % ns;
  // angle = -+ 2 pi k r / (R ns): sincospi of 2 k r / (R ns)
  const double base = (inverse ? 2.0 : -2.0) * (double)k / (double)(R * ns);
  double2 v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double2 a = src[j + r * q];
    if (r == 0) {
      v[r] = a;
    } else {
      double s, c;
      sincospi(base * r, &s, &c);
      v[r] = cmul(a, make_double2(c, s));
    }
  }
  const long long o = (j / ns) * R * ns + k;
  if constexpr (R == 2) {
    dst[o] = cadd(v[0], v[1]);
    dst[o + ns] = csub(v[0], v[1]);
  } else {
    const bool inv = inverse != 0;
    const double2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    const double2 t2 = cadd(v[1], v[3]), t3 = crot(csub(v[1], v[3]), inv);
    dst[o] = cadd(t0, t2);
    dst[o + ns] = cadd(t1, t3);
    dst[o + 2 * ns] = csub(t0, t2);
    dst[o + 3 * ns] = csub(t1, t3);
  }
}

static __global__ void scale_rows(double2* __restrict__ x, long long total, double s) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) x[i] = make_double2(x[i].x * s, x[i].y * s);
}

// Transform `batch` contiguous rows of length n (a power of two) from `in`;
// `work` is scratch of the same size.  The result lands in `in` or `work`:
// the return value (nullptr on a launch error) says which.  Unscaled inverse
// when scale_inverse is false; 1/n folded in otherwise.  launches: kernels issued.
inline double2* transform(double2* in, double2* work, long long n, long long batch, bool inverse,
                          bool scale_inverse, cudaStream_t s, long long* launches) {
  int lg = 0;
  while ((1LL << lg) < n) ++lg;
  double2* a = in;
  double2* b = work;
  long long ns = 1;
  const int threads = 256;
  if (lg % 2) {
    const long long total = batch * (n / 2);
    stockham_pass<2><<<(unsigned)((total + threads - 1) / threads), threads, 0, s>>>(a, b, n, ns, total, inverse);
    ++*launches;
    double2* t = a; a = b; b = t;
    ns *= 2;
  }
  for (int p = 0; p < lg / 2; ++p) {
    const long long total = batch * (n / 4);
    stockham_pass<4><<<(unsigned)((total + threads - 1) / threads), threads, 0, s>>>(a, b, n, ns, total, inverse);
    ++*launches;
    double2* t = a; a = b; b = t;
    ns *= 4;
  }
  if (inverse && scale_inverse) {
    const long long total = batch * n;
    scale_rows<<<(unsigned)((total + threads - 1) / threads), threads, 0, s>>>(a, total, 1.0 / (double)n);
    ++*launches;
  }
  if (cudaGetLastError() != cudaSuccess) return nullptr;
  return a;
}

// ---------------------------------------------------------------------------
// Any length m (the receiver's symbol count need not be a power of two):
// Bluestein's chirp-z transform on the power-of-two Stockham FFT of length
// L >= 2m - 1.  X_k = c_k sum_n (x_n c_n) conj(c_{k-n}), c_n = W_{2m}^{n^2}
// (n^2 reduced mod 2m in integers, so the chirp phase stays exact).
// ---------------------------------------------------------------------------
__host__ __device__ inline long long bluestein_len(long long m) {
  long long l = 1;
  while (l < 2 * m - 1) l <<= 1;
  return l;
}
inline bool is_pow2(long long n) { return n > 0 && (n & (n - 1)) == 0; }
// scratch (double2 elements) transform_any needs for `batch` rows of length m
inline long long scratch_elems(long long m, long long batch) {
  return is_pow2(m) ? batch * m : (2 * batch + 2) * bluestein_len(m);
}

__device__ __forceinline__ double2 chirp(long long n, long long m, bool inverse) {
  const long long e = (n % (2 * m)) * (n % (2 * m)) % (2 * m);   // n^2 mod 2m
  double s, c;
  sincospi((inverse ? 1.0 : -1.0) * (double)e / (double)m, &s, &c);
  return make_double2(c, s);
}

// a[row][j] = x[row][j] c_j (j < m), 0 up to L
static __global__ void bluestein_pre(const double2* __restrict__ x, double2* __restrict__ a, long long m, long long L,
                              long long total, int inverse) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const long long row = i / L, j = i - row * L;
  a[i] = j < m ? cmul(x[row * m + j], chirp(j, m, inverse != 0)) : make_double2(0.0, 0.0);
}

// b_j = conj(c_j) for j < m, b_{L-j} = conj(c_j) for 0 < j < m, else 0
static __global__ void bluestein_kernel_b(double2* __restrict__ b, long long m, long long L, int inverse) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= L) return;
  long long src = -1;
  if (j < m) src = j;
  else if (L - j < m) src = L - j;
  if (src < 0) {
    b[j] = make_double2(0.0, 0.0);
  } else {
    const double2 c = chirp(src, m, inverse != 0);
    b[j] = make_double2(c.x, -c.y);
  }
}

// A[row][j] *= B[j]
static __global__ void bluestein_mul(double2* __restrict__ a, const double2* __restrict__ bspec, long long L,
                              long long total) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) a[i] = cmul(a[i], bspec[i % L]);
}

// y[row][k] = c_k r[row][k] / L (k < m), times 1/m when scaling an inverse
static __global__ void bluestein_post(const double2* __restrict__ r, double2* __restrict__ y, long long m, long long L,
                               long long total, int inverse, double scale) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const long long row = i / m, k = i - row * m;
  const double2 v = cmul(r[row * L + k], chirp(k, m, inverse != 0));
  y[i] = make_double2(v.x * scale, v.y * scale);
}

// x: `batch` rows of length m (any m >= 1), transformed in place; scratch has
// scratch_elems(m, batch) elements.  Returns false on a launch error.
inline bool transform_any(double2* x, double2* scratch, long long m, long long batch, bool inverse,
                          bool scale_inverse, cudaStream_t s, long long* launches) {
  const int threads = 256;
  if (is_pow2(m)) {
    double2* res = transform(x, scratch, m, batch, inverse, scale_inverse, s, launches);
    if (!res) return false;
    if (res != x && cudaMemcpyAsync(x, res, (size_t)batch * m * sizeof(double2), cudaMemcpyDeviceToDevice, s) !=
                        cudaSuccess)
      return false;
    return true;
  }
  const long long L = bluestein_len(m);
  double2* a = scratch;                 // [batch][L]
  double2* a2 = a + batch * L;          // [batch][L] ping-pong
  double2* b = a2 + batch * L;          // [L]
  double2* b2 = b + L;                  // [L]
  const long long tot = batch * L;
  bluestein_kernel_b<<<(unsigned)((L + threads - 1) / threads), threads, 0, s>>>(b, m, L, inverse);
  ++*launches;
  double2* bspec = transform(b, b2, L, 1, false, false, s, launches);
  bluestein_pre<<<(unsigned)((tot + threads - 1) / threads), threads, 0, s>>>(x, a, m, L, tot, inverse);
  ++*launches;
  double2* aspec = transform(a, a2, L, batch, false, false, s, launches);
  if (!bspec || !aspec) return false;
  bluestein_mul<<<(unsigned)((tot + threads - 1) / threads), threads, 0, s>>>(aspec, bspec, L, tot);
  ++*launches;
  double2* other = aspec == a ? a2 : a;
  double2* r = transform(aspec, other, L, batch, true, false, s, launches);
  if (!r) return false;
  const long long totm = batch * m;
  const double scale = (inverse && scale_inverse ? 1.0 / (double)m : 1.0) / (double)L;
  bluestein_post<<<(unsigned)((totm + threads - 1) / threads), threads, 0, s>>>(r, x, m, L, totm, inverse, scale);
  ++*launches;
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace fft64
