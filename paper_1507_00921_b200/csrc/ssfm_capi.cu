// C ABI of the whole-waveform SSFM link simulator (dbp_sim_*, include/dbp_b200.h).
//
// The simulator owns its device buffers: the waveform batch
// [item][pol][n] complex64, a scratch buffer of the same size (transposed
// layout only), the noise and Jones buffers of the span-end amplifier, the
// block-FFT twiddles of both row lengths, the W_n^{k1 n2} tables in both
// layouts and the permuted double-float linear-step table (cached per
// (sample rate, beta2, dz)); spans run as cached CUDA graphs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dbp_b200.h"
#include "launch.h"
#include "ssfm_kernels.cuh"

namespace dbp {

// [planes][rows][cols] -> [planes][cols][rows], complex64, 32 x 32 tiles
__global__ void __launch_bounds__(256) ssfm_transpose_kernel(const float2* __restrict__ in,
                                                             float2* __restrict__ out, int rows, int cols) {
  __shared__ float2 tile[32][33];
  const long long plane = blockIdx.z;
  const float2* src = in + plane * (long long)rows * cols;
  float2* dst = out + plane * (long long)rows * cols;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int r = r0 + threadIdx.y + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[threadIdx.y + k][threadIdx.x] = src[(long long)r * cols + c];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int c = c0 + threadIdx.y + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[(long long)c * rows + r] = tile[threadIdx.x][threadIdx.y + k];
  }
}

// span-end amplifier: x <- J (g x + noise) (channel.py:97-128, 131-153)
__global__ void __launch_bounds__(256) ssfm_amplify_kernel(float2* __restrict__ data, long long n, long long items,
                                                           float g, const float2* __restrict__ noise,
                                                           const float2* __restrict__ jones) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * items) return;
  const long long item = i / n, s = i - item * n;
  float2* px = data + item * 2 * n + s;
  float2* py = px + n;
  float2 x = make_float2(px->x * g, px->y * g), y = make_float2(py->x * g, py->y * g);
  if (noise) {
    const float2* nx = noise + item * 2 * n + s;
    x = c_add(x, nx[0]);
    y = c_add(y, nx[n]);
  }
  if (jones) {  // one row-major 2x2 matrix per waveform
    const float2* j = jones + 4 * item;
    const float2 a = c_add(c_mul(x, __ldg(j)), c_mul(y, __ldg(j + 1)));
    const float2 b = c_add(c_mul(x, __ldg(j + 2)), c_mul(y, __ldg(j + 3)));
    x = a;
    y = b;
  }
  *px = x;
  *py = y;
}

}  // namespace dbp

namespace dbp_capi_internal {
int fail(int code, const std::string& msg);
void add_launches(long long n);
long long launch_total();
}

namespace {

using dbp_capi_internal::fail;

#define SIM_CUDA(call, what)                                                       \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) return fail(DBP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e_)); \
  } while (0)

using RowFn = cudaError_t (*)(const dbp::SimParams&, long long, size_t, cudaStream_t, bool);
using ShapeFn = dbp::LaunchShape (*)();

template <int L>
void fill(RowFn* rf, ShapeFn* sf) {
  rf[L] = &dbp::launch_ssfm_row<L>;
  sf[L] = &dbp::launch_shape<L>;
  if constexpr (L < dbp::kMaxLogN) fill<L + 1>(rf, sf);
}

struct SimDispatch {
  RowFn row[dbp::kMaxLogN + 1] = {};
  ShapeFn shape[dbp::kMaxLogN + 1] = {};
  SimDispatch() { fill<dbp::kMinLogN>(row, shape); }
};

const SimDispatch& sim_dispatch() {
  static SimDispatch d;
  return d;
}

struct Guard {
  int prev = -1;
  explicit Guard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    cudaSetDevice(dev);
  }
  ~Guard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

struct dbp_sim {
  int device = 0, log_n = 0, log_n1 = 0, log_n2 = 0, max_batch = 0;
  // column mode (n <= 2^22): the waveform stays in natural [N1][N2] order,
  // column kernels with shared-memory tiles do the N1-point transforms, no
  // global transposes.  Otherwise (or DBP_SIM_TRANSPOSE=1) the transposed
  // four-step layout with 32 x 33 tile transposes.
  bool column = false;
  // block mode (n <= 2^13): the whole waveform is one block-FFT row; a span
  // is ONE launch running every step on-chip (kSimFull)
  bool block = false;
  long long n = 0;
  float2* data = nullptr;
  float2* scratch = nullptr;
  float2* noise = nullptr;
  float2* jones = nullptr;   // [max_batch][2][2]
  float2* tw1 = nullptr;
  float2* tw2 = nullptr;
  float2* wa = nullptr;   // W_n^{k1(p) n2} at [n2][p] (row kernels over At)
  float2* wb = nullptr;   // the same at [p][n2] (row kernels over B)
  float2* lin = nullptr;
  float2* lin_lo = nullptr;
  double lin_key[3] = {0, 0, 0};
  bool lin_valid = false;
  cudaStream_t stream = nullptr;
  // one CUDA graph per span configuration: a span is 4 launches per step, so
  // small waveforms are launch-bound; the graph replays the whole span
  struct SpanGraph {
    int batch, steps, nonlinear;
    float nl_a, loss, loss_last;
    cudaGraphExec_t exec;
    long long launches;
  };
  std::vector<SpanGraph> graphs;
};

namespace {

int upload(float2** dst, const std::vector<float2>& h) {
  SIM_CUDA(cudaMalloc(dst, h.size() * sizeof(float2)), "cudaMalloc");
  SIM_CUDA(cudaMemcpy(*dst, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice), "cudaMemcpy");
  return DBP_OK;
}

// W_n^{k1(p) n2} in both layouts, p the register-order position of bin k1
// after the N1-point forward pass (host threads over n2 rows)
void make_four_step_twiddles(int log_n, int log_n1, std::vector<float2>& wa, std::vector<float2>& wb) {
  const long long n = 1LL << log_n, n1 = 1LL << log_n1, n2 = n >> log_n1;
  const int t1 = (int)(n1 / 16);
  wa.assign(n, make_float2(0.f, 0.f));
  wb.assign(n, make_float2(0.f, 0.f));
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (unsigned w = 0; w < hw; ++w)
    pool.emplace_back([&, w] {
      for (long long r = w; r < n2; r += hw)
        for (long long p = 0; p < n1; ++p) {
          const long long k1 = dbp::last_pass_bin(log_n1, (int)(p % t1), (int)(p / t1));
          const float2 v = dbp::unit_float2(-2.0 * M_PI * (double)((k1 * r) & (n - 1)) / (double)n);
          wa[r * n1 + p] = v;
          wb[p * n2 + r] = v;
        }
    });
  for (auto& th : pool) th.join();
}

int launch_row(dbp_sim* s, int logn_row, int mode, float2* buf, int batch, const dbp::SimParams& base,
               cudaStream_t st, bool column = false) {
  const SimDispatch& d = sim_dispatch();
  const dbp::LaunchShape sh = d.shape[logn_row]();
  dbp::SimParams sp = base;
  sp.data = buf;
  sp.mode = mode;
  sp.rows = (int)(s->n >> logn_row);
  sp.total_rows = (long long)sp.rows * batch;
  sp.n2 = 1 << s->log_n2;
  sp.tw = logn_row == s->log_n1 ? s->tw1 : s->tw2;
  sp.wtab = mode == dbp::kSimB ? s->wb : s->wa;
  sp.slice_floats = dbp::slice_floats(1 << logn_row, 0, false);
  // row kernels: one row per slice; column kernels: one tile of col_width columns per CTA
  const int slices = column ? dbp::col_width(logn_row) : sh.slices;
  const long long ctas = column ? (long long)batch * (sp.n2 / slices) : (sp.total_rows + slices - 1) / slices;
  const size_t smem = (size_t)sp.slice_floats * sizeof(float) * slices;
  cudaError_t e = d.row[logn_row](sp, ctas, smem, st, column);
  dbp_capi_internal::add_launches(1);
  if (e != cudaSuccess) return fail(DBP_ECUDA, std::string("ssfm_row_kernel: ") + cudaGetErrorString(e));
  return DBP_OK;
}

int transpose(const float2* in, float2* out, int rows, int cols, int planes, cudaStream_t st) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32, planes);
  dbp::ssfm_transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(in, out, rows, cols);
  dbp_capi_internal::add_launches(1);
  SIM_CUDA(cudaGetLastError(), "ssfm_transpose_kernel");
  return DBP_OK;
}

int ensure_lin(dbp_sim* s, double fs, double beta2, double dz) {
  if (s->lin_valid && s->lin_key[0] == fs && s->lin_key[1] == beta2 && s->lin_key[2] == dz) return DBP_OK;
  const long long n = s->n, n1 = 1LL << s->log_n1, n2 = 1LL << s->log_n2;
  const int t1 = (int)(n1 / 16), t2 = (int)(n2 / 16);
  std::vector<float2> h(n), l(n);
  const double inv_n = 1.0 / (double)n;
  auto entry = [&](long long k, long long slot) {
    const double f = (k < n / 2 ? (double)k : (double)(k - n)) * (fs / (double)n);
    const double ph = -2.0 * M_PI * M_PI * (beta2 * 1e-24) * f * f * dz;  // channel.py:57
    const double re = std::cos(ph) * inv_n, im = std::sin(ph) * inv_n;
    const float2 hi = make_float2((float)re, (float)im);
    h[slot] = hi;
    l[slot] = make_float2((float)(re - hi.x), (float)(im - hi.y));
  };
  if (s->block) {   // one row of n: bins in the block FFT's register order
    const int tt = (int)(n / 16);
    for (int t = 0; t < tt; ++t)
      for (int e = 0; e < 16; ++e) entry(dbp::last_pass_bin(s->log_n, t, e), dbp::tab_index(s->log_n, t, e));
  }
  for (long long p = 0; !s->block && p < n1; ++p) {
    const long long k1 = dbp::last_pass_bin(s->log_n1, (int)(p % t1), (int)(p / t1));
    for (int t = 0; t < t2; ++t)
      for (int e = 0; e < 16; ++e) {
        const long long k = k1 + n1 * dbp::last_pass_bin(s->log_n2, t, e);
        const double f = (k < n / 2 ? (double)k : (double)(k - n)) * (fs / (double)n);
        const double ph = -2.0 * M_PI * M_PI * (beta2 * 1e-24) * f * f * dz;  // channel.py:57
        const double re = std::cos(ph) * inv_n, im = std::sin(ph) * inv_n;
        const float2 hi = make_float2((float)re, (float)im);
        h[p * n2 + dbp::tab_index(s->log_n2, t, e)] = hi;
        l[p * n2 + dbp::tab_index(s->log_n2, t, e)] = make_float2((float)(re - hi.x), (float)(im - hi.y));
      }
  }
  if (!s->lin) SIM_CUDA(cudaMalloc(&s->lin, n * sizeof(float2)), "cudaMalloc(lin)");
  if (!s->lin_lo) SIM_CUDA(cudaMalloc(&s->lin_lo, n * sizeof(float2)), "cudaMalloc(lin_lo)");
  SIM_CUDA(cudaMemcpy(s->lin, h.data(), n * sizeof(float2), cudaMemcpyHostToDevice), "cudaMemcpy(lin)");
  SIM_CUDA(cudaMemcpy(s->lin_lo, l.data(), n * sizeof(float2), cudaMemcpyHostToDevice), "cudaMemcpy(lin_lo)");
  s->lin_key[0] = fs;
  s->lin_key[1] = beta2;
  s->lin_key[2] = dz;
  s->lin_valid = true;
  return DBP_OK;
}

}  // namespace

extern "C" {

int dbp_sim_create(dbp_sim** out, int device, int log2_n, int max_batch) {
  if (!out) return fail(DBP_EINVAL, "null output pointer");
  *out = nullptr;
  if (log2_n < 2 * dbp::kMinLogN || log2_n > dbp::kMaxLogN + 13)
    return fail(DBP_EINVAL, "waveform length 2^" + std::to_string(log2_n) + " outside [2^8, 2^26]");
  if (max_batch < 1) return fail(DBP_EINVAL, "max_batch must be >= 1");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(DBP_ECUDA, "no CUDA device available");
  }
  if (device < 0 || device >= ndev) return fail(DBP_EINVAL, "device index out of range");
  Guard g(device);
  dbp_sim* s = new (std::nothrow) dbp_sim();
  if (!s) return fail(DBP_ENOMEM, "host allocation failed");
  s->device = device;
  s->log_n = log2_n;
  s->n = 1LL << log2_n;
  const char* force_t = std::getenv("DBP_SIM_TRANSPOSE");
  const char* force_nb = std::getenv("DBP_SIM_NO_BLOCK");
  // (measured: 2^8 2.7, 2^10 3.5, 2^12 10.0 us per step; at 2^13 one 1024-thread
  // CTA per waveform is slower than the four-step split, 22 vs 11 us)
  s->block = log2_n <= 12 && !(force_nb && force_nb[0] == '1') && !(force_t && force_t[0] == '1');
  // Column tiles are BPC(N1) = 2048 / N1 columns wide, so N2 >= 2048 / N1,
  // i.e. n >= 2^11.  Split measured on B200 (tools/sim_sweep.sh,
  // profiles/r1/sim_sweep.txt): N1 = 2^7 up to 2^14, 2^8 up to 2^20, 2^9 at
  // 2^21; from 2^22 the transposed layout is faster (32-byte column rows).
  s->column = !s->block && log2_n >= 11 && log2_n <= 21 && !(force_t && force_t[0] == '1');
  const char* force_l1 = std::getenv("DBP_SIM_LOGN1");   // tuning experiments
  if (s->column) {
    s->log_n1 = log2_n <= 14 ? std::min(7, log2_n - 4) : log2_n <= 20 ? 8 : 9;   // N2 <= 2^13
    if (force_l1 && std::atoi(force_l1) >= dbp::kMinLogN && std::atoi(force_l1) <= 9 &&
        log2_n - std::atoi(force_l1) <= dbp::kMaxLogN && log2_n - std::atoi(force_l1) >= 11 - std::atoi(force_l1))
      s->log_n1 = std::atoi(force_l1);
    s->log_n2 = log2_n - s->log_n1;
  } else {
    s->log_n2 = (log2_n + 1) / 2;
    s->log_n1 = log2_n - s->log_n2;
    if (s->log_n2 > dbp::kMaxLogN) {
      s->log_n2 = dbp::kMaxLogN;
      s->log_n1 = log2_n - s->log_n2;
    }
  }
  if (s->block) {
    s->log_n1 = 0;
    s->log_n2 = log2_n;
  }
  s->max_batch = max_batch;
  const size_t bytes = (size_t)max_batch * 2 * s->n * sizeof(float2);
  int rc = DBP_OK;
  auto cleanup = [&](int code) {
    dbp_sim_destroy(s);
    return code;
  };
  if (cudaMalloc(&s->data, bytes) != cudaSuccess ||
      (!s->column && !s->block && cudaMalloc(&s->scratch, bytes) != cudaSuccess) ||
      cudaMalloc(&s->noise, bytes) != cudaSuccess ||
      cudaMalloc(&s->jones, (size_t)max_batch * 4 * sizeof(float2)) != cudaSuccess)
    return cleanup(fail(DBP_ENOMEM, "device allocation of the waveform buffers failed"));
  if (!s->block && (rc = upload(&s->tw1, dbp::make_twiddles(s->log_n1)))) return cleanup(rc);
  if ((rc = upload(&s->tw2, dbp::make_twiddles(s->log_n2)))) return cleanup(rc);
  if (!s->block) {
    std::vector<float2> wa, wb;
    make_four_step_twiddles(log2_n, s->log_n1, wa, wb);
    if ((rc = upload(&s->wa, wa))) return cleanup(rc);
    if ((rc = upload(&s->wb, wb))) return cleanup(rc);
  }
  if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess)
    return cleanup(fail(DBP_ECUDA, "cudaStreamCreate failed"));
  *out = s;
  return DBP_OK;
}

int dbp_sim_destroy(dbp_sim* s) {
  if (!s) return DBP_OK;
  Guard g(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  cudaFree(s->data);
  cudaFree(s->scratch);
  cudaFree(s->noise);
  cudaFree(s->jones);
  cudaFree(s->tw1);
  cudaFree(s->tw2);
  cudaFree(s->wa);
  cudaFree(s->wb);
  cudaFree(s->lin);
  cudaFree(s->lin_lo);
  for (auto& gr : s->graphs) cudaGraphExecDestroy(gr.exec);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
  return DBP_OK;
}

int dbp_sim_upload(dbp_sim* s, const void* h_in, int batch) {
  if (!s || !h_in) return fail(DBP_EINVAL, "null argument");
  if (batch < 1 || batch > s->max_batch) return fail(DBP_EINVAL, "batch outside [1, max_batch]");
  Guard g(s->device);
  SIM_CUDA(cudaMemcpyAsync(s->data, h_in, (size_t)batch * 2 * s->n * sizeof(float2), cudaMemcpyHostToDevice,
                           s->stream), "H2D");
  SIM_CUDA(cudaStreamSynchronize(s->stream), "cudaStreamSynchronize");
  return DBP_OK;
}

int dbp_sim_download(dbp_sim* s, void* h_out, int batch) {
  if (!s || !h_out) return fail(DBP_EINVAL, "null argument");
  if (batch < 1 || batch > s->max_batch) return fail(DBP_EINVAL, "batch outside [1, max_batch]");
  Guard g(s->device);
  SIM_CUDA(cudaMemcpyAsync(h_out, s->data, (size_t)batch * 2 * s->n * sizeof(float2), cudaMemcpyDeviceToHost,
                           s->stream), "D2H");
  SIM_CUDA(cudaStreamSynchronize(s->stream), "cudaStreamSynchronize");
  return DBP_OK;
}

int dbp_sim_span(dbp_sim* s, int batch, double sample_rate, double beta2, double gamma, double dz,
                 double dz_eff, double loss, int steps, int nonlinear) {
  if (!s) return fail(DBP_EINVAL, "null simulator");
  if (batch < 1 || batch > s->max_batch) return fail(DBP_EINVAL, "batch outside [1, max_batch]");
  if (steps < 1) return fail(DBP_EINVAL, "steps_per_span must be >= 1");
  if (!(sample_rate > 0.0) || !std::isfinite(beta2) || !std::isfinite(gamma) || !std::isfinite(dz) ||
      !std::isfinite(dz_eff) || !std::isfinite(loss))
    return fail(DBP_EINVAL, "span parameters must be finite (sample rate positive)");
  Guard g(s->device);
  int rc = ensure_lin(s, sample_rate, beta2, dz);
  if (rc) return rc;
  dbp::SimParams base;
  std::memset(&base, 0, sizeof(base));
  base.pol_stride = s->n;
  base.log_n = s->log_n;
  base.log_n1 = s->log_n1;
  base.lin = s->lin;
  base.lin_lo = s->lin_lo;
  base.nl_a = (float)(-gamma * dz_eff);  // channel.py:71 exp(-j gamma dz_eff I)
  base.loss = (float)loss;
  base.loss_last = (float)(std::pow(loss, steps) / std::pow((double)base.loss, steps - 1));
  base.nonlinear = nonlinear ? 1 : 0;
  const int n1 = 1 << s->log_n1, n2 = 1 << s->log_n2, planes = 2 * batch;
  cudaStream_t st = s->stream;
  auto enqueue = [&]() -> int {
    int r;
    if (s->block) {   // one launch: every step on-chip
      dbp::SimParams full = base;
      full.steps = steps;
      return launch_row(s, s->log_n, dbp::kSimFull, s->data, batch, full, st);
    }
    if (s->column) {   // natural layout throughout: column (N1) and row (N2) kernels in place
      if ((r = launch_row(s, s->log_n1, dbp::kSimA, s->data, batch, base, st, true))) return r;
      for (int k = 0; k < steps; ++k) {
        if ((r = launch_row(s, s->log_n2, dbp::kSimB, s->data, batch, base, st))) return r;
        if ((r = launch_row(s, s->log_n1, k + 1 < steps ? dbp::kSimCA : dbp::kSimC, s->data, batch, base, st,
                            true)))
          return r;
      }
      return DBP_OK;
    }
    // natural [N1][N2] -> At [N2][N1], first column FFT
    if ((r = transpose(s->data, s->scratch, n1, n2, planes, st))) return r;
    if ((r = launch_row(s, s->log_n1, dbp::kSimA, s->scratch, batch, base, st))) return r;
    for (int k = 0; k < steps; ++k) {
      if ((r = transpose(s->scratch, s->data, n2, n1, planes, st))) return r;   // -> B [N1][N2]
      if ((r = launch_row(s, s->log_n2, dbp::kSimB, s->data, batch, base, st))) return r;
      if ((r = transpose(s->data, s->scratch, n1, n2, planes, st))) return r;   // -> At
      if ((r = launch_row(s, s->log_n1, k + 1 < steps ? dbp::kSimCA : dbp::kSimC, s->scratch, batch, base, st)))
        return r;
    }
    return transpose(s->scratch, s->data, n2, n1, planes, st);                 // -> natural
  };
  dbp_sim::SpanGraph* gr = nullptr;
  for (auto& g2 : s->graphs)
    if (g2.batch == batch && g2.steps == steps && g2.nonlinear == base.nonlinear && g2.nl_a == base.nl_a &&
        g2.loss == base.loss && g2.loss_last == base.loss_last)
      gr = &g2;
  if (!gr) {
    if (s->graphs.size() >= 8) {
      cudaGraphExecDestroy(s->graphs.front().exec);
      s->graphs.erase(s->graphs.begin());
    }
    SIM_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    const long long before = dbp_capi_internal::launch_total();
    rc = enqueue();
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    SIM_CUDA(ce, "cudaStreamEndCapture");
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    SIM_CUDA(ie, "cudaGraphInstantiate");
    const long long launches = dbp_capi_internal::launch_total() - before;
    dbp_capi_internal::add_launches(-launches);   // counted when the graph runs
    s->graphs.push_back({batch, steps, base.nonlinear, base.nl_a, base.loss, base.loss_last, exec, launches});
    gr = &s->graphs.back();
  }
  SIM_CUDA(cudaGraphLaunch(gr->exec, st), "cudaGraphLaunch");
  dbp_capi_internal::add_launches(gr->launches);
  SIM_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  return DBP_OK;
}

int dbp_sim_amplify(dbp_sim* s, int batch, double g_amp, const void* h_noise, const double* jones) {
  if (!s) return fail(DBP_EINVAL, "null simulator");
  if (batch < 1 || batch > s->max_batch) return fail(DBP_EINVAL, "batch outside [1, max_batch]");
  Guard g(s->device);
  cudaStream_t st = s->stream;
  if (h_noise)
    SIM_CUDA(cudaMemcpyAsync(s->noise, h_noise, (size_t)batch * 2 * s->n * sizeof(float2), cudaMemcpyHostToDevice,
                             st), "H2D(noise)");
  if (jones) {
    std::vector<float2> j((size_t)batch * 4);
    for (size_t i = 0; i < j.size(); ++i) {
      if (!std::isfinite(jones[2 * i]) || !std::isfinite(jones[2 * i + 1]))
        return fail(DBP_EINVAL, "Jones matrices must be finite");
      j[i] = make_float2((float)jones[2 * i], (float)jones[2 * i + 1]);
    }
    SIM_CUDA(cudaMemcpyAsync(s->jones, j.data(), j.size() * sizeof(float2), cudaMemcpyHostToDevice, st),
             "H2D(jones)");
    SIM_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");   // j is a host temporary
  }
  const long long total = s->n * batch;
  dbp::ssfm_amplify_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
      s->data, s->n, batch, (float)g_amp, h_noise ? s->noise : nullptr, jones ? s->jones : nullptr);
  dbp_capi_internal::add_launches(1);
  SIM_CUDA(cudaGetLastError(), "ssfm_amplify_kernel");
  SIM_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  return DBP_OK;
}

int dbp_sim_length(const dbp_sim* s, int64_t* n) {
  if (!s || !n) return fail(DBP_EINVAL, "null argument");
  *n = s->n;
  return DBP_OK;
}

}  // extern "C"
