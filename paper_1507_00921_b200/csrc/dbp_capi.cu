// C ABI of libdbp_b200.so (declared in include/dbp_b200.h).
//
// The plan owns the device-resident tables of one DBP configuration
// (dispersion filters, FFT twiddles, step program, ESSFM coefficients) and
// the staging buffers of the host-buffer entry point.  Nothing here throws
// across the ABI: failures return a negative code and leave a message in a
// thread-local string (dbp_last_error).
#include <cuda_runtime.h>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include <algorithm>
#include <atomic>
#include <thread>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/dbp_b200.h"
#include "dbp_general.cuh"
#include "fft64.cuh"
#include "host_pool.h"
#include "launch.h"

namespace {

thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(DBP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define DBP_CUDA(call, what)                      \
  do {                                            \
    cudaError_t e_ = (call);                      \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

int ilog2_exact(int n) {
  if (n <= 0 || (n & (n - 1)) != 0) return -1;
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

// RAII device switch
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

using LaunchFn = cudaError_t (*)(const dbp::KernelParams&, long long, size_t, cudaStream_t);
using ShapeFn = dbp::LaunchShape (*)();

template <int L>
void fill_tables(LaunchFn* lf, ShapeFn* sf) {
  lf[L] = &dbp::launch_block_kernel<L>;
  sf[L] = &dbp::launch_shape<L>;
  if constexpr (L < dbp::kMaxLogN) fill_tables<L + 1>(lf, sf);
}

struct Dispatch {
  LaunchFn launch[dbp::kMaxLogN + 1] = {};
  ShapeFn shape[dbp::kMaxLogN + 1] = {};
  Dispatch() { fill_tables<dbp::kMinLogN>(launch, shape); }
};

const Dispatch& dispatch() {
  static Dispatch d;
  return d;
}

}  // namespace

namespace dbp_capi_internal {
// shared with ssfm_capi.cu: set the thread-local message, return the code
int fail(int code, const std::string& msg) { return ::fail(code, msg); }
void add_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_total() { return g_launches.load(); }
int run_host_staged(dbp_plan* p, const void* h_in, void* h_out, int64_t n_total, int batch);
}  // namespace dbp_capi_internal

struct dbp_plan {
  int device = 0;
  int N = 0, M = 0, logn = 0, step = 0, lead = 0;
  float2* d_full = nullptr;
  float2* d_half = nullptr;
  float2* d_tw = nullptr;
  float2* d_wtw = nullptr;   // warp FFE kernel bases (N = 1024 .. 4096)
  float2* d_full_nat = nullptr;   // the full-step filter in natural bin order (warp FFE kernel)
  float2* d_r2_full = nullptr;    // N = 8192 radix-2 step tables (dbp_r2_kernel.cuh)
  float2* d_r2_half = nullptr;
  float2* d_r2_tw = nullptr;      // N = 8192: the 4096-point twiddles
  bool have_r2_half = false;
  float2* d_steps = nullptr;
  int steps_cap = 0;
  float* d_coeff = nullptr;
  bool have_full = false, have_half = false, have_steps = false;
  int program = dbp::kFFE, arrangement = dbp::kSymmetric, n_steps = 0, nc = 0;
  float c[dbp::kMaxSideCoeffs + 4] = {};
  // per-item coefficient sets (dbp_plan_set_coeff_batch)
  float* d_coeff_batch = nullptr;
  int batch_sets = 0, batch_nc = 0, batch_stride = 0;
  size_t batch_cap = 0;
  // host-run staging
  size_t staging_budget = size_t(256) << 20;
  cudaStream_t streams[2] = {nullptr, nullptr};
  void* d_stage[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [slot][in/out]
  size_t stage_bytes = 0;
  // complex128 drop-in path (dbp_backpropagate_c128): pinned complex64
  // staging per slot [in/out], its size, completion events, host threads
  void* h_pin[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  size_t pin_bytes = 0;
  cudaEvent_t done[2] = {nullptr, nullptr};
  // dbp_run_host's whole-item pipeline: copy-in, compute and copy-out
  // streams joined per slot by events, so each copy engine runs back to back
  cudaStream_t pipe[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_k[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  dbp::HostPool* pool = nullptr;   // the process-wide conversion pool (not owned)
  // block lengths outside the fused kernel's [16, 8192]: the float64
  // multi-kernel path (dbp_general.cuh) with natural-order float64 tables
  bool general = false;
  double2* d_full64 = nullptr;
  double2* d_half64 = nullptr;
  std::vector<double2> steps64;   // (a_j, g_j) in float64
  double c64[dbp::kMaxSideCoeffs + 1] = {};
  double2* d_ws = nullptr;        // [block][pol][N] complex128 workspace ...
  double2* d_work = nullptr;      // ... the FFT's ping-pong partner ...
  double* d_inten = nullptr;      // ... and [block][N] intensities
  long long ws_blocks = 0;
  cudaEvent_t ws_done = nullptr;  // end of the last launch that used the workspace (any stream)
};

namespace {

int upload(float2** dst, const std::vector<float2>& src) {
  if (*dst == nullptr) {
    DBP_CUDA(cudaMalloc(dst, src.size() * sizeof(float2)), "cudaMalloc(table)");
  }
  DBP_CUDA(cudaMemcpy(*dst, src.data(), src.size() * sizeof(float2), cudaMemcpyHostToDevice),
           "cudaMemcpy(table)");
  return DBP_OK;
}

int check_ready(const dbp_plan* p) {
  if (!p) return fail(DBP_EINVAL, "null plan");
  if (!p->have_steps) return fail(DBP_ESTATE, "dbp_plan_set_steps has not been called");
  if (p->program != dbp::kRotateOnly && p->program != dbp::kIdentity && !p->have_full)
    return fail(DBP_ESTATE, "dbp_plan_set_linear has not been called");
  if (p->program != dbp::kFFE && p->program != dbp::kRotateOnly && p->program != dbp::kIdentity &&
      p->arrangement == dbp::kSymmetric && !p->have_half)
    return fail(DBP_ESTATE, "symmetric arrangement needs the half-step kernel");
  return DBP_OK;
}

// Fill the parameters shared by every launch mode.
void base_params(const dbp_plan* p, dbp::KernelParams& kp) {
  std::memset(&kp, 0, sizeof(kp));
  kp.program = p->program;
  kp.arrangement = p->arrangement;
  kp.n_steps = p->n_steps;
  if (p->program == dbp::kFFE) {
    kp.n_ops = 1;
    kp.conv_all = 1;
    kp.conv_parity = -1;
  } else if (p->program == dbp::kRotateOnly) {
    kp.n_ops = p->n_steps;
    kp.conv_parity = -1;
  } else if (p->program == dbp::kIdentity) {
    kp.n_ops = 0;             // framing only: load, keep the centre, store
    kp.conv_parity = -1;
  } else {
    kp.n_ops = 2 * p->n_steps + (p->arrangement == dbp::kSymmetric ? 1 : 0);
    kp.conv_parity = p->arrangement == dbp::kNonlinearFirst ? 1 : 0;
    kp.half_ends = p->arrangement == dbp::kSymmetric ? 1 : 0;
    kp.sidx_shift = 1;
  }
  kp.nc = p->nc;
  kp.fir_pad = (p->nc + 3) & ~3;
  kp.slice_floats = p->general ? 0 : dbp::slice_floats(p->N, kp.fir_pad, dispatch().shape[p->logn]().double_buffer);
  kp.precise_sincos = p->n_steps >= 3 ? 1 : 0;
  kp.tab_full = p->d_full;
  kp.tab_half = p->d_half ? p->d_half : p->d_full;
  kp.twiddle = p->d_tw;
  kp.wtw = p->d_wtw;
  kp.tab_nat = p->d_full_nat;
  kp.r2_full = p->d_r2_full;
  kp.r2_half = p->have_r2_half ? p->d_r2_half : nullptr;
  kp.r2_tw = p->d_r2_tw;
  kp.steps = p->d_steps;
  kp.coeff = p->d_coeff;
  std::memcpy(kp.c, p->c, sizeof(kp.c));
}

// The float64 multi-kernel path for block lengths outside [16, 8192]
// (dbp_general.cuh): the same KernelParams contract as the fused kernel.
int launch_general(const dbp_plan* cp, const dbp::KernelParams& kp, cudaStream_t s) {
  dbp_plan* p = const_cast<dbp_plan*>(cp);   // workspace grows lazily
  namespace dg = dbp_general;
  const long long n = p->N;
  // chunk of blocks whose workspace (2 x 2 N complex128 + N float64 per block) fits ~768 MB
  const long long per_block = 2 * 2 * n * (long long)sizeof(double2) + n * (long long)sizeof(double);
  static const long long budget = [] {   // DBP_GENERAL_WS_MB: workspace budget (tests force small chunks)
    const char* v = std::getenv("DBP_GENERAL_WS_MB");
    const long long mb = v && *v ? std::atoll(v) : 768;
    return (mb > 0 ? mb : 768) << 20;
  }();
  long long chunk = budget / per_block;
  if (chunk < 1) chunk = 1;
  if (chunk > kp.total_blocks) chunk = kp.total_blocks;
  if (p->ws_blocks < chunk) {
    cudaFree(p->d_ws);
    cudaFree(p->d_work);
    cudaFree(p->d_inten);
    p->d_ws = p->d_work = nullptr;
    p->d_inten = nullptr;
    p->ws_blocks = 0;
    if (cudaMalloc(&p->d_ws, chunk * 2 * n * sizeof(double2)) != cudaSuccess ||
        cudaMalloc(&p->d_work, chunk * 2 * n * sizeof(double2)) != cudaSuccess ||
        cudaMalloc(&p->d_inten, chunk * n * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return fail(DBP_ENOMEM, "workspace cudaMalloc failed for the general block-length path");
    }
    p->ws_blocks = chunk;
  }
  dg::Taps taps{};
  for (int i = 0; i <= p->nc && i < dg::kMaxTaps; ++i) taps.c[i] = p->c64[i];
  // one workspace per plan: calls on different streams (the two slots of the
  // host pipelines) take turns, each waiting for the previous call's kernels
  if (!p->ws_done) {
    DBP_CUDA(cudaEventCreateWithFlags(&p->ws_done, cudaEventDisableTiming), "cudaEventCreate");
  } else {
    DBP_CUDA(cudaStreamWaitEvent(s, p->ws_done, 0), "cudaStreamWaitEvent");
  }
  long long launches = 0;
  for (long long blk0 = 0; blk0 < kp.total_blocks; blk0 += chunk) {
    const long long nblk = std::min(chunk, kp.total_blocks - blk0);
    const long long rows = 2 * nblk;
    double2* cur = p->d_ws;
    double2* oth = p->d_work;
    dg::frame_kernel<<<dg::grid_for(rows * n), dg::kThreads, 0, s>>>(kp, blk0, nblk, n, cur);
    ++launches;
    for (int op = 0; op < kp.n_ops; ++op) {
      const bool is_conv = kp.conv_all || (op & 1) == kp.conv_parity;
      if (is_conv) {
        const bool half = kp.half_ends && (op == 0 || op == kp.n_ops - 1);
        const double2* tab = half && p->d_half64 ? p->d_half64 : p->d_full64;
        double2* r = dg::transform16(cur, oth, n, rows, false, s, &launches);
        if (!r) return cuda_fail(cudaGetLastError(), "general path forward FFT");
        if (r != cur) std::swap(cur, oth);
        dg::mul_kernel<<<dg::grid_for(rows * n), dg::kThreads, 0, s>>>(cur, tab, rows * n, n);
        ++launches;
        r = dg::transform16(cur, oth, n, rows, true, s, &launches);   // 1/N is in the table
        if (!r) return cuda_fail(cudaGetLastError(), "general path inverse FFT");
        if (r != cur) std::swap(cur, oth);
      } else {
        const int sidx = op >> kp.sidx_shift;
        if (sidx < 0 || sidx >= (int)p->steps64.size()) return fail(DBP_ESTATE, "step index outside the program");
        const int nc = kp.coeff_stride ? kp.nc : p->nc;
        dg::intensity_kernel<<<dg::grid_for(nblk * n), dg::kThreads, 0, s>>>(cur, p->d_inten, nblk, n);
        dg::rotate_kernel<<<dg::grid_for(nblk * n), dg::kThreads, 0, s>>>(
            cur, p->d_inten, nblk, n, kp, blk0, taps, nc, p->steps64[sidx].x, p->steps64[sidx].y);
        launches += 2;
      }
    }
    dg::store_kernel<<<dg::grid_for(rows * (long long)kp.step), dg::kThreads, 0, s>>>(cur, kp, blk0, nblk, n);
    ++launches;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "general block-length path launch");
  DBP_CUDA(cudaEventRecord(p->ws_done, s), "cudaEventRecord");
  g_launches.fetch_add(launches, std::memory_order_relaxed);
  return DBP_OK;
}

int launch(const dbp_plan* p, const dbp::KernelParams& kp, cudaStream_t s) {
  if (kp.total_blocks <= 0) return DBP_OK;
  if (p->general) return launch_general(p, kp, s);
  const Dispatch& d = dispatch();
  const dbp::LaunchShape sh = d.shape[p->logn]();
  const long long ctas = (kp.total_blocks + sh.slices - 1) / sh.slices;
  if (ctas > 0x7fffffffLL) return fail(DBP_EINVAL, "too many blocks for one launch");
#ifndef DBP_EXPERIMENT_MIN_SMEM
#define DBP_EXPERIMENT_MIN_SMEM 0   // timing experiment: pad the CTA's shared memory (bytes) to cap CTAs per SM
#endif
  size_t smem = (size_t)kp.slice_floats * sizeof(float) * sh.slices;
  if (smem < (size_t)DBP_EXPERIMENT_MIN_SMEM) smem = DBP_EXPERIMENT_MIN_SMEM;
  if (smem > 227 * 1024) return fail(DBP_EINVAL, "shared memory per CTA exceeds 227 KB for this block length");
  // Persistent grid (SMs x resident CTAs, each looping over block groups with
  // an L2 prefetch of the next): only N = 8192 (one 1024-thread CTA per SM)
  // gains, +3%; N <= 4096 loses ~10% against the hardware CTA scheduler
  // (tools/ab_persist.sh).  DBP_PERSISTENT=k overrides (0 = off).
  static const int env_persistent = [] {
    const char* v = std::getenv("DBP_PERSISTENT");
    return v ? std::atoi(v) : -1;
  }();
  // only the N = 8192 kernel loops; smaller N always get the full grid
  const int persistent = p->logn < DBP_PERSIST_MIN_LOGN ? 0 : env_persistent >= 0 ? env_persistent
                                                            : (p->logn >= 13 ? 1 : 0);
  long long grid = ctas;
  if (persistent > 0) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long resident = (long long)sms * sh.min_ctas * persistent;
    if (resident > 0 && resident < grid) grid = resident;
  }
  dbp::KernelParams k = kp;
  // item = blk / blocks_per_item by multiply-high (exact for 32-bit operands)
  k.bpi_magic = 0;
  if (kp.blocks_per_item > 1 && kp.blocks_per_item <= 0xffffffffLL && kp.total_blocks <= 0xffffffffLL)
    k.bpi_magic = ~0ULL / (unsigned long long)kp.blocks_per_item + 1;
  cudaError_t e = d.launch[p->logn](k, grid, smem, s);
  if (e != cudaSuccess) return cuda_fail(e, "dbp_block_kernel launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return DBP_OK;
}

int check_range(const dbp_plan* p, int64_t n_total, int batch, int64_t b0, int64_t b1) {
  if (n_total < 1) return fail(DBP_EINVAL, "signal must contain at least one sample");
  if (batch < 0) return fail(DBP_EINVAL, "batch must be >= 0");
  const int64_t nb = (n_total + p->step - 1) / p->step;
  if (b0 < 0 || b1 < b0 || b1 > nb)
    return fail(DBP_EINVAL, "block range outside [0, ceil(n_total / (N - M))]");
  return DBP_OK;
}

int ensure_staging(dbp_plan* p, size_t bytes) {
  if (p->stage_bytes >= bytes) return DBP_OK;
  for (int s = 0; s < 2; ++s)
    for (int k = 0; k < 2; ++k) {
      if (p->d_stage[s][k]) cudaFree(p->d_stage[s][k]);
      p->d_stage[s][k] = nullptr;
    }
  p->stage_bytes = 0;
  for (int s = 0; s < 2; ++s)
    for (int k = 0; k < 2; ++k) {
      cudaError_t e = cudaMalloc(&p->d_stage[s][k], bytes);
      if (e != cudaSuccess) return fail(DBP_ENOMEM, std::string("staging cudaMalloc: ") + cudaGetErrorString(e));
    }
  p->stage_bytes = bytes;
  for (int s = 0; s < 2; ++s)
    if (!p->streams[s]) DBP_CUDA(cudaStreamCreateWithFlags(&p->streams[s], cudaStreamNonBlocking), "cudaStreamCreate");
  return DBP_OK;
}

int ensure_pipeline(dbp_plan* p) {
  for (int s = 0; s < 3; ++s)
    if (!p->pipe[s]) DBP_CUDA(cudaStreamCreateWithFlags(&p->pipe[s], cudaStreamNonBlocking), "cudaStreamCreate");
  for (int s = 0; s < 2; ++s) {
    if (!p->ev_in[s]) DBP_CUDA(cudaEventCreateWithFlags(&p->ev_in[s], cudaEventDisableTiming), "cudaEventCreate");
    if (!p->ev_k[s]) DBP_CUDA(cudaEventCreateWithFlags(&p->ev_k[s], cudaEventDisableTiming), "cudaEventCreate");
    if (!p->ev_out[s]) DBP_CUDA(cudaEventCreateWithFlags(&p->ev_out[s], cudaEventDisableTiming), "cudaEventCreate");
  }
  return DBP_OK;
}

// bytes of one pipelined chunk of dbp_run_host (DBP_HOST_CHUNK_MB, default
// 64 MiB, capped by the staging budget / 4).  Measured on the configs[3]
// batch (profiles/r2/session4/ab_host_chunk.txt): 64 MiB reaches 0.93 of the
// bidirectional pinned-copy rate, 32 / 16 / 8 / 4 MiB 0.92 / 0.90 / 0.85 /
// 0.75 -- per-chunk costs outweigh the shorter pipeline fill and drain
size_t host_chunk_bytes() {
  static const size_t b = [] {
    const char* v = std::getenv("DBP_HOST_CHUNK_MB");
    const long long mb = v && *v ? std::atoll(v) : 64;
    return (size_t)(mb > 0 ? mb : 64) << 20;
  }();
  return b;
}

}  // namespace

extern "C" {

const char* dbp_last_error(void) { return g_last_error.c_str(); }

int dbp_version(void) { return 102; }

int64_t dbp_launch_count(void) { return g_launches.load(); }

int dbp_device_count(int* count) {
  if (!count) return fail(DBP_EINVAL, "null count");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    cudaGetLastError();
    return DBP_OK;
  }
  *count = n;
  return DBP_OK;
}

int dbp_plan_create(dbp_plan** out, int device, int block_len, int overlap) {
  if (!out) return fail(DBP_EINVAL, "null output pointer");
  *out = nullptr;
  const int logn = ilog2_exact(block_len);
  if (logn < 0) return fail(DBP_EINVAL, "block_len must be a power of two, got " + std::to_string(block_len));
  if (!(0 <= overlap && overlap < block_len)) return fail(DBP_EINVAL, "overlap must satisfy 0 <= overlap < block_len");
  if (logn > DBP_MAX_LOG2_BLOCK)
    return fail(DBP_EINVAL, "block_len " + std::to_string(block_len) + " above the supported 2^" +
                                std::to_string(DBP_MAX_LOG2_BLOCK));
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(DBP_ECUDA, "no CUDA device available");
  }
  if (device < 0 || device >= ndev) return fail(DBP_EINVAL, "device index out of range");
  DeviceGuard g(device);
  if (!g.ok) return fail(DBP_ECUDA, "cudaSetDevice failed");
  dbp_plan* p = new (std::nothrow) dbp_plan();
  if (!p) return fail(DBP_ENOMEM, "host allocation failed");
  p->device = device;
  p->N = block_len;
  p->M = overlap;
  p->logn = logn;
  p->step = block_len - overlap;
  p->lead = overlap / 2;
  p->general = logn < dbp::kMinLogN || logn > dbp::kMaxLogN;
  if (p->general) {   // the float64 path needs no block-FFT tables
    *out = p;
    return DBP_OK;
  }
  std::vector<float2> tw = dbp::make_twiddles(logn);
  int rc = upload(&p->d_tw, tw);
  if (rc == DBP_OK && dbp::warp_ffe_supported(logn)) rc = upload(&p->d_wtw, dbp::make_warp_twiddles(logn, &dbp::unit_float2));
  if (rc == DBP_OK && logn == 13) rc = upload(&p->d_r2_tw, dbp::make_twiddles(12));
  if (rc != DBP_OK) {
    dbp_plan_destroy(p);
    return rc;
  }
  *out = p;
  return DBP_OK;
}

int dbp_plan_destroy(dbp_plan* p) {
  if (!p) return DBP_OK;
  DeviceGuard g(p->device);
  for (int s = 0; s < 3; ++s)
    if (p->pipe[s]) {
      cudaStreamSynchronize(p->pipe[s]);
      cudaStreamDestroy(p->pipe[s]);
    }
  for (int s = 0; s < 2; ++s) {
    if (p->ev_in[s]) cudaEventDestroy(p->ev_in[s]);
    if (p->ev_k[s]) cudaEventDestroy(p->ev_k[s]);
    if (p->ev_out[s]) cudaEventDestroy(p->ev_out[s]);
  }
  for (int s = 0; s < 2; ++s) {
    if (p->streams[s]) cudaStreamSynchronize(p->streams[s]);
    for (int k = 0; k < 2; ++k)
      if (p->h_pin[s][k]) cudaFreeHost(p->h_pin[s][k]);
    if (p->done[s]) cudaEventDestroy(p->done[s]);
    for (int k = 0; k < 2; ++k)
      if (p->d_stage[s][k]) cudaFree(p->d_stage[s][k]);
    if (p->streams[s]) cudaStreamDestroy(p->streams[s]);
  }
  cudaFree(p->d_full);
  cudaFree(p->d_wtw);
  cudaFree(p->d_full_nat);
  cudaFree(p->d_r2_full);
  cudaFree(p->d_r2_half);
  cudaFree(p->d_r2_tw);
  cudaFree(p->d_half);
  cudaFree(p->d_tw);
  cudaFree(p->d_steps);
  cudaFree(p->d_coeff);
  cudaFree(p->d_coeff_batch);
  cudaFree(p->d_full64);
  cudaFree(p->d_half64);
  cudaFree(p->d_ws);
  cudaFree(p->d_work);
  cudaFree(p->d_inten);
  if (p->ws_done) cudaEventDestroy(p->ws_done);
  delete p;
  return DBP_OK;
}

int dbp_plan_set_staging(dbp_plan* p, size_t bytes) {
  if (!p) return fail(DBP_EINVAL, "null plan");
  if (bytes < (size_t(1) << 20)) return fail(DBP_EINVAL, "staging budget must be >= 1 MiB");
  p->staging_budget = bytes;
  return DBP_OK;
}

int dbp_plan_set_linear(dbp_plan* p, const double* kernel, const double* half_kernel) {
  if (!p) return fail(DBP_EINVAL, "null plan");
  if (!kernel) return fail(DBP_EINVAL, "null kernel");
  DeviceGuard g(p->device);
  const double inv_n = 1.0 / (double)p->N;
  if (p->general) {
    // natural bin order, float64, 1/N folded in (the inverse FFT is unscaled)
    auto convert64 = [&](const double* src, std::vector<double2>& h) {
      h.resize(p->N);
      for (int k = 0; k < p->N; ++k) {
        if (!std::isfinite(src[2 * k]) || !std::isfinite(src[2 * k + 1])) return false;
        h[k] = make_double2(src[2 * k] * inv_n, src[2 * k + 1] * inv_n);
      }
      return true;
    };
    std::vector<double2> h, hh;
    if (!convert64(kernel, h)) return fail(DBP_EINVAL, "kernel must be finite");
    if (half_kernel && !convert64(half_kernel, hh)) return fail(DBP_EINVAL, "half kernel must be finite");
    p->have_full = false;
    p->have_half = false;
    auto up = [&](double2** dst, const std::vector<double2>& src) -> int {
      if (!*dst) DBP_CUDA(cudaMalloc(dst, src.size() * sizeof(double2)), "cudaMalloc(table64)");
      DBP_CUDA(cudaMemcpy(*dst, src.data(), src.size() * sizeof(double2), cudaMemcpyHostToDevice),
               "cudaMemcpy(table64)");
      return DBP_OK;
    };
    int rc = up(&p->d_full64, h);
    if (rc != DBP_OK) return rc;
    if (half_kernel) {
      rc = up(&p->d_half64, hh);
      if (rc != DBP_OK) return rc;
    }
    p->have_full = true;
    p->have_half = half_kernel != nullptr;
    return DBP_OK;
  }
  const int T = p->N / 16;
  // stored in the kernel's register order: entry tab_index(t, e) holds the bin
  // that register e of thread t carries after the last forward FFT pass
  std::vector<int> bin(p->N);
  for (int t = 0; t < T; ++t)
    for (int e = 0; e < 16; ++e) bin[dbp::tab_index(p->logn, t, e)] = dbp::last_pass_bin(p->logn, t, e);
  // validate and convert both tables before touching the plan, so a failed
  // call leaves the previous (full, half) pair in place
  auto convert = [&](const double* src, std::vector<float2>& h) {
    h.resize(p->N);
    for (int j = 0; j < p->N; ++j) {
      const int k = bin[j];
      const double re = src[2 * k], im = src[2 * k + 1];
      if (!std::isfinite(re) || !std::isfinite(im)) return false;
      h[j] = make_float2((float)(re * inv_n), (float)(im * inv_n));
    }
    return true;
  };
  std::vector<float2> h, hh;
  if (!convert(kernel, h)) return fail(DBP_EINVAL, "kernel must be finite");
  if (half_kernel && !convert(half_kernel, hh)) return fail(DBP_EINVAL, "half kernel must be finite");
  // a failed upload leaves the tables undefined: drop both flags first
  p->have_full = false;
  p->have_half = false;
  int rc = upload(&p->d_full, h);
  if (rc != DBP_OK) return rc;
  if (dbp::warp_ffe_supported(p->logn)) {
    // the warp FFE kernel reads the full-step filter in natural bin order
    std::vector<float2> nat(p->N);
    for (int j = 0; j < p->N; ++j) nat[bin[j]] = h[j];
    rc = upload(&p->d_full_nat, nat);
    if (rc != DBP_OK) return rc;
  }
  if (half_kernel) {
    rc = upload(&p->d_half, hh);
    if (rc != DBP_OK) return rc;
  }
  if (p->logn == 13) {
    // the R2 kernel's step tables, from the float64 filters
    p->have_r2_half = false;
    rc = upload(&p->d_r2_full, dbp::make_r2_tables(kernel));
    if (rc != DBP_OK) return rc;
    if (half_kernel) {
      rc = upload(&p->d_r2_half, dbp::make_r2_tables(half_kernel));
      if (rc != DBP_OK) return rc;
      p->have_r2_half = true;
    }
  }
  p->have_full = true;
  p->have_half = half_kernel != nullptr;
  return DBP_OK;
}

int dbp_plan_set_steps(dbp_plan* p, int algorithm, int arrangement, int num_steps,
                       const double* weights, const double* gains, double gamma,
                       const double* coeffs, int n_coeffs) {
  if (!p) return fail(DBP_EINVAL, "null plan");
  if (algorithm < DBP_ALG_FFE || algorithm > DBP_ALG_IDENTITY)
    return fail(DBP_EINVAL, "unknown algorithm code " + std::to_string(algorithm));
  if (arrangement < DBP_ARR_SYMMETRIC || arrangement > DBP_ARR_NONLINEAR_FIRST)
    return fail(DBP_EINVAL, "unknown arrangement code " + std::to_string(arrangement));
  // validate everything into locals; the plan changes only once every check passed
  float c[dbp::kMaxSideCoeffs + 4] = {};
  c[0] = 1.0f;
  double c64[dbp::kMaxSideCoeffs + 1] = {};
  c64[0] = 1.0;
  int nc = 0;
  std::vector<float2> st;
  std::vector<double2> st64;
  const bool no_steps = algorithm == DBP_ALG_FFE || algorithm == DBP_ALG_IDENTITY;
  if (!no_steps) {
    if (num_steps < 1) return fail(DBP_EINVAL, "num_steps must be >= 1");
    if (!weights || !gains) return fail(DBP_EINVAL, "null weights or gains");
    if (!std::isfinite(gamma)) return fail(DBP_EINVAL, "gamma must be finite");
    if (algorithm == DBP_ALG_ESSFM || algorithm == DBP_ALG_ROTATE) {
      if (!coeffs) return fail(DBP_EINVAL, "essfm requires a coefficient set");
      if (n_coeffs < 0 || n_coeffs > DBP_MAX_SIDE_COEFFS)
        return fail(DBP_EINVAL, "n_coeffs must be in [0, " + std::to_string(DBP_MAX_SIDE_COEFFS) + "]");
      if (p->N <= 2 * n_coeffs) return fail(DBP_EINVAL, "block length too short for the coefficient memory");
      for (int i = 0; i <= n_coeffs; ++i)
        if (!std::isfinite(coeffs[i])) return fail(DBP_EINVAL, "coefficients must be finite");
      nc = n_coeffs;
      // trailing zero side taps contribute fma(0, s, acc) == acc: drop them (bit-identical)
      while (nc > 0 && (float)coeffs[nc] == 0.0f) --nc;
      for (int i = 0; i <= nc; ++i) c[i] = (float)coeffs[i];
      for (int i = 0; i <= nc; ++i) c64[i] = coeffs[i];
    }
    st.resize(num_steps);
    st64.resize(num_steps);
    for (int j = 0; j < num_steps; ++j) {
      if (!std::isfinite(weights[j]) || !std::isfinite(gains[j])) return fail(DBP_EINVAL, "schedule must be finite");
      // reference rotation exp(-j * gamma * w * F)  ==  exp(+j * a * F), a = -gamma * w
      st[j] = make_float2((float)(-gamma * weights[j]), (float)gains[j]);
      st64[j] = make_double2(-gamma * weights[j], gains[j]);
    }
  }
  DeviceGuard g(p->device);
  // from here on a failure leaves the plan without a step program (ESTATE on run)
  p->have_steps = false;
  if (!no_steps) {
    if (num_steps > p->steps_cap) {
      cudaFree(p->d_steps);
      p->d_steps = nullptr;
      p->steps_cap = 0;
      DBP_CUDA(cudaMalloc(&p->d_steps, num_steps * sizeof(float2)), "cudaMalloc(steps)");
      p->steps_cap = num_steps;
    }
    DBP_CUDA(cudaMemcpy(p->d_steps, st.data(), num_steps * sizeof(float2), cudaMemcpyHostToDevice),
             "cudaMemcpy(steps)");
    if (!p->d_coeff) DBP_CUDA(cudaMalloc(&p->d_coeff, sizeof(p->c)), "cudaMalloc(coeff)");
    DBP_CUDA(cudaMemcpy(p->d_coeff, c, sizeof(c), cudaMemcpyHostToDevice), "cudaMemcpy(coeff)");
  }
  p->program = algorithm;
  p->arrangement = arrangement;
  std::memcpy(p->c, c, sizeof(c));
  std::memcpy(p->c64, c64, sizeof(c64));
  p->steps64 = st64;
  p->nc = nc;
  p->n_steps = no_steps ? 0 : num_steps;
  p->have_steps = true;
  return DBP_OK;
}

int dbp_num_blocks(const dbp_plan* p, int64_t n_total, int64_t* out) {
  if (!p || !out) return fail(DBP_EINVAL, "null argument");
  if (n_total < 0) return fail(DBP_EINVAL, "n_total must be >= 0");
  *out = (n_total + p->step - 1) / p->step;
  return DBP_OK;
}

int dbp_run(dbp_plan* p, const void* d_in, void* d_out, int64_t n_total, int batch,
            int64_t block_begin, int64_t block_end, void* stream) {
  int rc = check_ready(p);
  if (rc) return rc;
  rc = check_range(p, n_total, batch, block_begin, block_end);
  if (rc) return rc;
  if (!d_in || !d_out) return fail(DBP_EINVAL, "null device buffer");
  DeviceGuard g(p->device);
  dbp::KernelParams kp;
  base_params(p, kp);
  kp.in = static_cast<const float2*>(d_in);
  kp.out = static_cast<float2*>(d_out);
  kp.n_total = n_total;
  kp.in_pol_stride = n_total;
  kp.in_item_stride = 2 * n_total;
  kp.out_pol_stride = n_total;
  kp.out_item_stride = 2 * n_total;
  kp.in_origin = 0;
  kp.out_origin = 0;
  kp.block_begin = block_begin;
  kp.blocks_per_item = block_end - block_begin;
  kp.total_blocks = kp.blocks_per_item * batch;
  kp.cyclic = 1;
  kp.step = p->step;
  kp.lead = p->lead;
  return launch(p, kp, static_cast<cudaStream_t>(stream));
}

int dbp_run_chunk(dbp_plan* p, const void* d_in, void* d_out, int64_t n_total, int batch,
                  int64_t block_begin, int64_t block_end, int64_t in_len, int64_t out_len,
                  void* stream) {
  int rc = check_ready(p);
  if (rc) return rc;
  rc = check_range(p, n_total, batch, block_begin, block_end);
  if (rc) return rc;
  if (!d_in || !d_out) return fail(DBP_EINVAL, "null device buffer");
  const int64_t need_in = (block_end - block_begin) * p->step + p->M;
  int64_t end = block_end * p->step;
  if (end > n_total) end = n_total;
  const int64_t need_out = end - block_begin * p->step;
  if (in_len < need_in) return fail(DBP_EINVAL, "in_len shorter than (blocks * step + M)");
  if (out_len < need_out) return fail(DBP_EINVAL, "out_len shorter than the kept samples");
  DeviceGuard g(p->device);
  dbp::KernelParams kp;
  base_params(p, kp);
  kp.in = static_cast<const float2*>(d_in);
  kp.out = static_cast<float2*>(d_out);
  kp.n_total = n_total;
  kp.in_pol_stride = in_len;
  kp.in_item_stride = 2 * in_len;
  kp.out_pol_stride = out_len;
  kp.out_item_stride = 2 * out_len;
  kp.in_origin = block_begin * p->step - p->lead;
  kp.out_origin = block_begin * p->step;
  kp.block_begin = block_begin;
  kp.blocks_per_item = block_end - block_begin;
  kp.total_blocks = kp.blocks_per_item * batch;
  kp.cyclic = 0;
  kp.step = p->step;
  kp.lead = p->lead;
  return launch(p, kp, static_cast<cudaStream_t>(stream));
}

int dbp_process_blocks(dbp_plan* p, const void* d_blocks, void* d_out, int64_t n_blocks, void* stream) {
  int rc = check_ready(p);
  if (rc) return rc;
  if (n_blocks < 0) return fail(DBP_EINVAL, "n_blocks must be >= 0");
  if (!d_blocks || !d_out) return fail(DBP_EINVAL, "null device buffer");
  DeviceGuard g(p->device);
  dbp::KernelParams kp;
  base_params(p, kp);
  kp.in = static_cast<const float2*>(d_blocks);
  kp.out = static_cast<float2*>(d_out);
  kp.n_total = p->N;
  kp.in_pol_stride = p->N;
  kp.in_item_stride = 2LL * p->N;
  kp.out_pol_stride = p->N;
  kp.out_item_stride = 2LL * p->N;
  kp.block_begin = 0;
  kp.blocks_per_item = 1;
  kp.total_blocks = n_blocks;
  kp.cyclic = 1;
  kp.step = p->N;
  kp.lead = 0;
  return launch(p, kp, static_cast<cudaStream_t>(stream));
}

int dbp_plan_synchronize(dbp_plan* p) {
  if (!p) return fail(DBP_EINVAL, "null plan");
  DeviceGuard g(p->device);
  for (int s = 0; s < 2; ++s)
    if (p->streams[s]) DBP_CUDA(cudaStreamSynchronize(p->streams[s]), "cudaStreamSynchronize");
  for (int s = 0; s < 3; ++s)
    if (p->pipe[s]) DBP_CUDA(cudaStreamSynchronize(p->pipe[s]), "cudaStreamSynchronize");
  return DBP_OK;
}

int dbp_run_host(dbp_plan* p, const void* h_in, void* h_out, int64_t n_total, int batch,
                 int64_t block_begin, int64_t block_end) {
  int rc = check_ready(p);
  if (rc) return rc;
  rc = check_range(p, n_total, batch, block_begin, block_end);
  if (rc) return rc;
  if (!h_in || !h_out) return fail(DBP_EINVAL, "null host buffer");
  if (batch == 0 || block_end == block_begin) return DBP_OK;
  DeviceGuard g(p->device);
  const size_t row = (size_t)n_total * sizeof(float2);    // one polarisation
  const size_t item = 2 * row;
  const size_t slot_budget = p->staging_budget / 4;       // per in/out buffer per slot
  const int64_t nb = (n_total + p->step - 1) / p->step;
  const bool full_range = block_begin == 0 && block_end == nb;
  const int64_t out_lo = block_begin * p->step;
  int64_t out_hi = block_end * p->step;
  if (out_hi > n_total) out_hi = n_total;
  const char* src = static_cast<const char*>(h_in);
  char* dst = static_cast<char*>(h_out);
  if (full_range) {   // pageable rows: through pinned staging on the host pool
    rc = dbp_capi_internal::run_host_staged(p, h_in, h_out, n_total, batch);
    if (rc != 1) return rc;
  }
  // copies that read / write the caller's host buffers may still be queued
  // when a later call fails: drain both staging streams before returning,
  // so the caller can free its buffers on any return code
  struct StreamDrain {
    dbp_plan* p;
    ~StreamDrain() {
      for (int s = 0; s < 2; ++s)
        if (p->streams[s]) cudaStreamSynchronize(p->streams[s]);
      for (int s = 0; s < 3; ++s)
        if (p->pipe[s]) cudaStreamSynchronize(p->pipe[s]);
    }
  } drain{p};

  // A block range (a multi-device shard of one waveform) stages only its
  // halo'd span [b0 step - M/2, b1 step - M/2 + N) through the chunk path,
  // so host-to-device traffic is shard + halo, not the whole waveform
  // (unless that span would wrap onto itself: a short waveform).
  const bool span_fits = (block_end - block_begin) * p->step + p->M <= n_total;
  if (item <= slot_budget && (full_range || !span_fits)) {
    // whole items per chunk, cyclic mode: copy-in / compute / copy-out
    // streams, two buffer slots, per-slot events guarding buffer reuse
    const size_t chunk = std::min(slot_budget, std::max(item, host_chunk_bytes()));
    const int per = (int)std::min<size_t>((size_t)batch, std::max<size_t>(1, chunk / item));
    rc = ensure_staging(p, per * item);
    if (rc) return rc;
    rc = ensure_pipeline(p);
    if (rc) return rc;
    cudaStream_t s_in = p->pipe[0], s_k = p->pipe[1], s_out = p->pipe[2];
    int k = 0;
    for (int i0 = 0; i0 < batch; i0 += per, ++k) {
      const int slot = k & 1;
      const int cnt = std::min(per, batch - i0);
      void* din = p->d_stage[slot][0];
      void* dout = p->d_stage[slot][1];
      // din[slot] was last read by the kernel of chunk k - 2
      if (k >= 2) DBP_CUDA(cudaStreamWaitEvent(s_in, p->ev_k[slot], 0), "cudaStreamWaitEvent");
      DBP_CUDA(cudaMemcpyAsync(din, src + (size_t)i0 * item, cnt * item, cudaMemcpyHostToDevice, s_in), "H2D");
      DBP_CUDA(cudaEventRecord(p->ev_in[slot], s_in), "cudaEventRecord");
      DBP_CUDA(cudaStreamWaitEvent(s_k, p->ev_in[slot], 0), "cudaStreamWaitEvent");
      // dout[slot] was last read by the copy-out of chunk k - 2
      if (k >= 2) DBP_CUDA(cudaStreamWaitEvent(s_k, p->ev_out[slot], 0), "cudaStreamWaitEvent");
      rc = dbp_run(p, din, dout, n_total, cnt, block_begin, block_end, s_k);
      if (rc) return rc;
      DBP_CUDA(cudaEventRecord(p->ev_k[slot], s_k), "cudaEventRecord");
      DBP_CUDA(cudaStreamWaitEvent(s_out, p->ev_k[slot], 0), "cudaStreamWaitEvent");
      if (full_range) {
        DBP_CUDA(cudaMemcpyAsync(dst + (size_t)i0 * item, dout, cnt * item, cudaMemcpyDeviceToHost, s_out), "D2H");
      } else {
        for (int it = 0; it < cnt; ++it)
          for (int pol = 0; pol < 2; ++pol) {
            const size_t off = (size_t)it * item + pol * row + out_lo * sizeof(float2);
            DBP_CUDA(cudaMemcpyAsync(dst + (size_t)i0 * item + off, static_cast<char*>(dout) + off,
                                     (out_hi - out_lo) * sizeof(float2), cudaMemcpyDeviceToHost, s_out), "D2H");
          }
      }
      DBP_CUDA(cudaEventRecord(p->ev_out[slot], s_out), "cudaEventRecord");
    }
    for (int s = 0; s < 3; ++s) DBP_CUDA(cudaStreamSynchronize(p->pipe[s]), "cudaStreamSynchronize");
  } else {
    // one item larger than a staging slot: block-range chunks with halos
    const int64_t span_budget = (int64_t)(slot_budget / (2 * sizeof(float2)));
    int64_t per_blocks = (span_budget - p->M) / p->step;
    if (per_blocks < 1) return fail(DBP_EINVAL, "staging budget too small for one block");
    rc = ensure_staging(p, slot_budget);
    if (rc) return rc;
    int slot = 0;
    for (int it = 0; it < batch; ++it) {
      for (int64_t b0 = block_begin; b0 < block_end; b0 += per_blocks, slot ^= 1) {
        const int64_t b1 = std::min(block_end, b0 + per_blocks);
        cudaStream_t s = p->streams[slot];
        char* din = static_cast<char*>(p->d_stage[slot][0]);
        char* dout = static_cast<char*>(p->d_stage[slot][1]);
        const int64_t span = (b1 - b0) * p->step + p->M;
        const int64_t g0 = b0 * p->step - p->lead;
        if (span > n_total) return fail(DBP_EINVAL, "chunk span exceeds the signal length");
        int64_t o1 = b1 * p->step;
        if (o1 > n_total) o1 = n_total;
        const int64_t olen = o1 - b0 * p->step;
        for (int pol = 0; pol < 2; ++pol) {
          const char* srow = src + (size_t)it * item + pol * row;
          char* drow = din + (size_t)pol * span * sizeof(float2);
          // pieces of [g0, g0 + span) modulo n_total (wraps at most once each side)
          int64_t done = 0;
          while (done < span) {
            int64_t gi = (g0 + done) % n_total;
            if (gi < 0) gi += n_total;
            const int64_t len = std::min(span - done, n_total - gi);
            DBP_CUDA(cudaMemcpyAsync(drow + done * sizeof(float2), srow + gi * sizeof(float2),
                                     len * sizeof(float2), cudaMemcpyHostToDevice, s), "H2D");
            done += len;
          }
        }
        rc = dbp_run_chunk(p, din, dout, n_total, 1, b0, b1, span, olen, s);
        if (rc) return rc;
        for (int pol = 0; pol < 2; ++pol)
          DBP_CUDA(cudaMemcpyAsync(dst + (size_t)it * item + pol * row + b0 * p->step * sizeof(float2),
                                   dout + (size_t)pol * olen * sizeof(float2), olen * sizeof(float2),
                                   cudaMemcpyDeviceToHost, s), "D2H");
      }
    }
  }
  for (int s = 0; s < 2; ++s) DBP_CUDA(cudaStreamSynchronize(p->streams[s]), "cudaStreamSynchronize");
  return DBP_OK;
}

extern "C++" {
namespace {

// one host conversion pool for the process (DBP_HOST_THREADS threads, default
// min(16, cores)), shared by every plan: idle threads are not multiplied by
// the number of cached plans
dbp::HostPool* shared_host_pool() {
  static dbp::HostPool pool([] {
    const char* v = std::getenv("DBP_HOST_THREADS");
    const int env = v ? std::atoi(v) : 0;
    const unsigned hc = std::thread::hardware_concurrency();
    return env > 0 ? env : (int)std::min(16u, hc ? hc : 1u);
  }());
  return &pool;
}

int ensure_pinned(dbp_plan* p, size_t bytes) {
  if (p->pin_bytes >= bytes) return DBP_OK;
  for (int s = 0; s < 2; ++s)
    for (int k = 0; k < 2; ++k) {
      if (p->h_pin[s][k]) cudaFreeHost(p->h_pin[s][k]);
      p->h_pin[s][k] = nullptr;
    }
  p->pin_bytes = 0;
  for (int s = 0; s < 2; ++s)
    for (int k = 0; k < 2; ++k)
      if (cudaHostAlloc(&p->h_pin[s][k], bytes, cudaHostAllocPortable) != cudaSuccess)
        return fail(DBP_ENOMEM, "pinned staging allocation failed");
  p->pin_bytes = bytes;
  for (int s = 0; s < 2; ++s)
    if (!p->done[s]) DBP_CUDA(cudaEventCreateWithFlags(&p->done[s], cudaEventDisableTiming), "cudaEventCreate");
  if (!p->pool) p->pool = shared_host_pool();
  return DBP_OK;
}

// Host casts of the complex128 drop-in path.  Rows of 2^18 samples and more
// are written with SSE2 streaming stores: the pinned staging is read next by
// the copy engine and a result row of that size does not stay in cache, so
// write-allocating those lines only adds a third to the casts' memory traffic
// (cvtpd2ps / cvtps2pd round exactly like the scalar casts).
long long stream_min_len() {   // DBP_HOST_STREAM_MIN: shortest row (samples) cast with streaming stores
  static const long long v = [] {
    const char* e = std::getenv("DBP_HOST_STREAM_MIN");
    return e && *e ? std::atoll(e) : (1LL << 18);
  }();
  return v;
}

inline void narrow_run(const double2* s, float2* d, long long run, bool stream) {
  long long k = 0;
#if defined(__SSE2__)
  if (stream) {
    for (; k < run && (reinterpret_cast<uintptr_t>(d + k) & 15); ++k) d[k] = make_float2((float)s[k].x, (float)s[k].y);
    for (; k + 2 <= run; k += 2) {
      const __m128 a = _mm_cvtpd_ps(_mm_loadu_pd(reinterpret_cast<const double*>(s + k)));
      const __m128 b = _mm_cvtpd_ps(_mm_loadu_pd(reinterpret_cast<const double*>(s + k + 1)));
      _mm_stream_ps(reinterpret_cast<float*>(d + k), _mm_movelh_ps(a, b));
    }
  }
#endif
  for (; k < run; ++k) d[k] = make_float2((float)s[k].x, (float)s[k].y);
}

inline void widen_run(const float2* s, double2* d, long long lo, long long hi, bool stream) {
  long long k = lo;
#if defined(__SSE2__)
  if (stream && (reinterpret_cast<uintptr_t>(d) & 15) == 0) {
    for (; k < hi; ++k) {
      const __m128 v = _mm_castpd_ps(_mm_load_sd(reinterpret_cast<const double*>(s + k)));
      _mm_stream_pd(reinterpret_cast<double*>(d + k), _mm_cvtps_pd(v));
    }
  }
#endif
  for (; k < hi; ++k) d[k] = make_double2((double)s[k].x, (double)s[k].y);
}

// complex64 rows (a caller's pageable buffers staged through pinned memory): plain copies
inline void copy_run(const float2* s, float2* d, long long run, bool stream) {
  long long k = 0;
#if defined(__SSE2__)
  if (stream) {
    for (; k < run && (reinterpret_cast<uintptr_t>(d + k) & 15); ++k) d[k] = s[k];
    for (; k + 8 <= run; k += 8) {
      const __m128 a = _mm_loadu_ps(reinterpret_cast<const float*>(s + k));
      const __m128 b = _mm_loadu_ps(reinterpret_cast<const float*>(s + k + 2));
      const __m128 c = _mm_loadu_ps(reinterpret_cast<const float*>(s + k + 4));
      const __m128 e = _mm_loadu_ps(reinterpret_cast<const float*>(s + k + 6));
      _mm_stream_ps(reinterpret_cast<float*>(d + k), a);
      _mm_stream_ps(reinterpret_cast<float*>(d + k + 2), b);
      _mm_stream_ps(reinterpret_cast<float*>(d + k + 4), c);
      _mm_stream_ps(reinterpret_cast<float*>(d + k + 6), e);
    }
  }
#endif
  std::memcpy(d + k, s + k, (size_t)(run - k) * sizeof(float2));
}
inline void narrow_run(const float2* s, float2* d, long long run, bool stream) { copy_run(s, d, run, stream); }
inline void widen_run(const float2* s, float2* d, long long lo, long long hi, bool stream) {
  copy_run(s + lo, d + lo, hi - lo, stream);
}

// dst[pol][i] = (float2) src[pol][(g0 + i) mod n] for i < len (rows of pitch len), both
// polarisations in one pass over the host pool
template <typename Elem>
void narrow_span(dbp::HostPool* pool, const Elem* const src[2], int64_t n, int64_t g0, int64_t len, float2* dst) {
  const bool stream = len >= stream_min_len();
  pool->parallel_for(len, [&](long long lo, long long hi) {
    for (int pol = 0; pol < 2; ++pol) {
      long long i = lo;
      while (i < hi) {
        int64_t g = (g0 + i) % n;
        if (g < 0) g += n;
        const long long run = std::min<long long>(hi - i, n - g);
        narrow_run(src[pol] + g, dst + pol * len + i, run, stream);
        i += run;
      }
    }
#if defined(__SSE2__)
    if (stream) _mm_sfence();
#endif
  });
}

// dst[pol][k] = (Elem) src[pol][k] for k < len (src rows of pitch len)
template <typename Elem>
void widen(dbp::HostPool* pool, const float2* src, int64_t len, Elem* const dst[2]) {
  const bool stream = len >= stream_min_len();
  pool->parallel_for(len, [&](long long lo, long long hi) {
    for (int pol = 0; pol < 2; ++pol) widen_run(src + pol * len, dst[pol], lo, hi, stream);
#if defined(__SSE2__)
    if (stream) _mm_sfence();
#endif
  });
}

// samples per polarisation and chunk of the staged host pipeline: a quarter
// of the signal, so that even one configs[0] waveform overlaps its casts with
// its copies, within [2^16, 2^21]; a batch of four items and more fills the
// pipeline with its other items and takes whole items up to 2^21 samples
// (DBP_C128_CHUNK overrides)
int64_t c128_chunk_samples(int64_t n_total, int batch) {
  static const int64_t forced = [] {
    const char* v = std::getenv("DBP_C128_CHUNK");
    return v && *v ? std::atoll(v) : 0LL;
  }();
  if (forced > 0) return forced;
  const int64_t want = batch >= 4 ? n_total : n_total / 4;
  return std::min<int64_t>(int64_t(1) << 21, std::max<int64_t>(int64_t(1) << 16, want));
}

// Host rows staged through pinned memory, for `batch` items of two rows each
// (Elem = double2: the reference's complex128 rows, cast on the host pool;
// float2: a caller's pageable complex64 rows, copied).  The chunks -- whole
// items, or block ranges with halos of one item -- run as one pipeline over
// all items: host copy-in, H2D, kernel, D2H on the chunk's stream (two slots),
// host copy-out two chunks later.
template <typename Elem, typename InRow, typename OutRow>
int staged_pipeline(dbp_plan* p, InRow in_row, OutRow out_row, int64_t n_total, int batch) {
  const int64_t nb = (n_total + p->step - 1) / p->step;
  // chunk: a block range whose halo'd span is c128_chunk_samples() per polarisation
  // (balanced: the nearest whole number of equal chunks)
  const int64_t per0 = std::max<int64_t>(1, (c128_chunk_samples(n_total, batch) - p->M) / p->step);
  const int64_t want_chunks = std::max<int64_t>(1, (nb + per0 / 2) / per0);
  const int64_t per_blocks = (nb + want_chunks - 1) / want_chunks;
  const bool single = nb <= per_blocks || per_blocks * p->step + p->M > n_total;
  const int64_t span_cap = single ? n_total : per_blocks * p->step + p->M;
  const int64_t out_cap = single ? n_total : per_blocks * p->step;
  const size_t in_bytes = (size_t)2 * span_cap * sizeof(float2), out_bytes = (size_t)2 * out_cap * sizeof(float2);
  int rc = ensure_staging(p, std::max(in_bytes, out_bytes));
  if (rc) return rc;
  rc = ensure_pinned(p, std::max(in_bytes, out_bytes));
  if (rc) return rc;
  struct StreamDrain {
    dbp_plan* p;
    ~StreamDrain() {
      for (int s = 0; s < 2; ++s)
        if (p->streams[s]) cudaStreamSynchronize(p->streams[s]);
    }
  } drain{p};
  const int64_t per_item = single ? 1 : (nb + per_blocks - 1) / per_blocks;
  const int64_t n_chunks = per_item * batch;
  // output of chunk k (chunk k % per_item of item k / per_item): [olo, ohi) per polarisation
  auto out_range = [&](int64_t k, int64_t& olo, int64_t& ohi) {
    if (single) {
      olo = 0;
      ohi = n_total;
      return;
    }
    const int64_t b0 = (k % per_item) * per_blocks, b1 = std::min(nb, b0 + per_blocks);
    olo = b0 * p->step;
    ohi = std::min<int64_t>(n_total, b1 * p->step);
  };
  auto finish = [&](int64_t k) -> int {
    const int slot = (int)(k & 1);
    DBP_CUDA(cudaEventSynchronize(p->done[slot]), "cudaEventSynchronize");
    int64_t olo, ohi;
    out_range(k, olo, ohi);
    const float2* pin = static_cast<const float2*>(p->h_pin[slot][1]);
    const int item = (int)(k / per_item);
    Elem* const dst[2] = {out_row(item, 0) + olo, out_row(item, 1) + olo};
    widen<Elem>(p->pool, pin, ohi - olo, dst);
    return DBP_OK;
  };
  for (int64_t k = 0; k < n_chunks; ++k) {
    const int slot = (int)(k & 1);
    if (k >= 2 && (rc = finish(k - 2))) return rc;
    cudaStream_t s = p->streams[slot];
    float2* pin_in = static_cast<float2*>(p->h_pin[slot][0]);
    float2* pin_out = static_cast<float2*>(p->h_pin[slot][1]);
    char* din = static_cast<char*>(p->d_stage[slot][0]);
    char* dout = static_cast<char*>(p->d_stage[slot][1]);
    const int item = (int)(k / per_item);
    const Elem* const in[2] = {in_row(item, 0), in_row(item, 1)};
    int64_t olo, ohi;
    out_range(k, olo, ohi);
    if (single) {
      narrow_span<Elem>(p->pool, in, n_total, 0, n_total, pin_in);
      DBP_CUDA(cudaMemcpyAsync(din, pin_in, 2 * n_total * sizeof(float2), cudaMemcpyHostToDevice, s), "H2D");
      rc = dbp_run(p, din, dout, n_total, 1, 0, nb, s);
      if (rc) return rc;
    } else {
      const int64_t b0 = (k % per_item) * per_blocks, b1 = std::min(nb, b0 + per_blocks);
      const int64_t span = (b1 - b0) * p->step + p->M, g0 = b0 * p->step - p->lead;
      narrow_span<Elem>(p->pool, in, n_total, g0, span, pin_in);
      DBP_CUDA(cudaMemcpyAsync(din, pin_in, 2 * span * sizeof(float2), cudaMemcpyHostToDevice, s), "H2D");
      rc = dbp_run_chunk(p, din, dout, n_total, 1, b0, b1, span, ohi - olo, s);
      if (rc) return rc;
    }
    DBP_CUDA(cudaMemcpyAsync(pin_out, dout, 2 * (ohi - olo) * sizeof(float2), cudaMemcpyDeviceToHost, s), "D2H");
    DBP_CUDA(cudaEventRecord(p->done[slot], s), "cudaEventRecord");
  }
  for (int64_t k = std::max<int64_t>(0, n_chunks - 2); k < n_chunks; ++k)
    if ((rc = finish(k))) return rc;
  return DBP_OK;
}

// true when a host pointer is ordinary pageable memory (not cudaHostAlloc / cudaHostRegister)
bool is_pageable(const void* ptr) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

}  // namespace

namespace dbp_capi_internal {
// dbp_run_host on pageable complex64 buffers (whole items of 2^16 samples and
// more): cudaMemcpyAsync from pageable memory is a synchronous driver-staged
// copy, so the rows go through the plan's pinned staging on the host pool
// instead (DBP_STAGE_PAGEABLE=0: the plain copies).  Returns 1 when the call
// was not taken.
int run_host_staged(dbp_plan* p, const void* h_in, void* h_out, int64_t n_total, int batch) {
  static const bool enabled = [] {
    const char* v = std::getenv("DBP_STAGE_PAGEABLE");
    return !(v && *v == '0');
  }();
  if (!enabled || n_total < (int64_t(1) << 16)) return 1;
  if (!is_pageable(h_in) && !is_pageable(h_out)) return 1;
  // in place (or overlapping) buffers keep the plain path, which uploads a whole item before
  // it writes any of its output: here a later chunk's halo would read rows already rewritten
  const char* a0 = static_cast<const char*>(h_in);
  const char* b0 = static_cast<const char*>(h_out);
  const size_t bytes = (size_t)batch * 2 * n_total * sizeof(float2);
  if (a0 < b0 + bytes && b0 < a0 + bytes) return 1;
  const float2* src = static_cast<const float2*>(h_in);
  float2* dst = static_cast<float2*>(h_out);
  return staged_pipeline<float2>(
      p, [&](int item, int pol) { return src + ((int64_t)2 * item + pol) * n_total; },
      [&](int item, int pol) { return dst + ((int64_t)2 * item + pol) * n_total; }, n_total, batch);
}
}  // namespace dbp_capi_internal

}  // extern "C++"

int dbp_backpropagate_c128(dbp_plan* p, const void* h_x, const void* h_y, void* h_out_x, void* h_out_y,
                           int64_t n_total) {
  int rc = check_ready(p);
  if (rc) return rc;
  if (!h_x || !h_y || !h_out_x || !h_out_y) return fail(DBP_EINVAL, "null host buffer");
  if (n_total < 1) return fail(DBP_EINVAL, "signal must contain at least one sample");
  DeviceGuard g(p->device);
  const double2* in[2] = {static_cast<const double2*>(h_x), static_cast<const double2*>(h_y)};
  double2* out[2] = {static_cast<double2*>(h_out_x), static_cast<double2*>(h_out_y)};
  // the reference never mutates its input (spectral.py:129): a chunk's halo is read after
  // earlier chunks' results are written, so the result rows must be separate from the input rows
  for (int i = 0; i < 2; ++i)
    for (int o = 0; o < 2; ++o)
      if (in[i] < out[o] + n_total && out[o] < in[i] + n_total)
        return fail(DBP_EINVAL, "result rows must not overlap the input rows");
  if (out[0] < out[1] + n_total && out[1] < out[0] + n_total)
    return fail(DBP_EINVAL, "result rows must not overlap each other");
  return staged_pipeline<double2>(
      p, [&](int, int pol) { return in[pol]; }, [&](int, int pol) { return out[pol]; }, n_total, 1);
}

int dbp_plan_set_coeff_batch(dbp_plan* p, const double* coeffs, int n_sets, int n_coeffs) {
  if (!p) return fail(DBP_EINVAL, "null plan");
  if (!coeffs || n_sets < 1) return fail(DBP_EINVAL, "need at least one coefficient set");
  if (n_coeffs < 0 || n_coeffs > DBP_MAX_SIDE_COEFFS)
    return fail(DBP_EINVAL, "n_coeffs must be in [0, " + std::to_string(DBP_MAX_SIDE_COEFFS) + "]");
  if (p->N <= 2 * n_coeffs) return fail(DBP_EINVAL, "block length too short for the coefficient memory");
  DeviceGuard g(p->device);
  const int stride = (n_coeffs + 1 + 3 + 3) & ~3;  // c_0..c_nc + 4-tap chunk padding
  std::vector<float> h((size_t)n_sets * stride, 0.0f);
  for (int s = 0; s < n_sets; ++s)
    for (int i = 0; i <= n_coeffs; ++i) {
      const double v = coeffs[(size_t)s * (n_coeffs + 1) + i];
      if (!std::isfinite(v)) return fail(DBP_EINVAL, "coefficients must be finite");
      h[(size_t)s * stride + i] = (float)v;
    }
  const size_t bytes = h.size() * sizeof(float);
  if (bytes > p->batch_cap) {
    cudaFree(p->d_coeff_batch);
    p->d_coeff_batch = nullptr;
    DBP_CUDA(cudaMalloc(&p->d_coeff_batch, bytes), "cudaMalloc(coeff batch)");
    p->batch_cap = bytes;
  }
  DBP_CUDA(cudaMemcpy(p->d_coeff_batch, h.data(), bytes, cudaMemcpyHostToDevice), "cudaMemcpy(coeff batch)");
  p->batch_sets = n_sets;
  p->batch_nc = n_coeffs;
  p->batch_stride = stride;
  return DBP_OK;
}

int dbp_run_coeff_batch(dbp_plan* p, const void* d_in, void* d_out, int64_t n_total,
                        int64_t block_begin, int64_t block_end, void* stream) {
  int rc = check_ready(p);
  if (rc) return rc;
  if (p->batch_sets < 1) return fail(DBP_ESTATE, "dbp_plan_set_coeff_batch has not been called");
  if (p->program != dbp::kESSFM && p->program != dbp::kRotateOnly)
    return fail(DBP_EINVAL, "coefficient batches need an essfm (or rotation) program");
  rc = check_range(p, n_total, p->batch_sets, block_begin, block_end);
  if (rc) return rc;
  if (!d_in || !d_out) return fail(DBP_EINVAL, "null device buffer");
  DeviceGuard g(p->device);
  dbp::KernelParams kp;
  base_params(p, kp);
  kp.nc = p->batch_nc;
  kp.fir_pad = (p->batch_nc + 3) & ~3;
  kp.slice_floats = p->general ? 0 : dbp::slice_floats(p->N, kp.fir_pad, dispatch().shape[p->logn]().double_buffer);
  kp.coeff = p->d_coeff_batch;
  kp.coeff_stride = p->batch_stride;
  kp.in = static_cast<const float2*>(d_in);
  kp.out = static_cast<float2*>(d_out);
  kp.n_total = n_total;
  kp.in_pol_stride = n_total;
  kp.in_item_stride = 0;  // every coefficient set reads the same waveform
  kp.out_pol_stride = n_total;
  kp.out_item_stride = 2 * n_total;
  kp.block_begin = block_begin;
  kp.blocks_per_item = block_end - block_begin;
  kp.total_blocks = kp.blocks_per_item * p->batch_sets;
  kp.cyclic = 1;
  kp.step = p->step;
  kp.lead = p->lead;
  return launch(p, kp, static_cast<cudaStream_t>(stream));
}

int dbp_run_host_coeff_batch(dbp_plan* p, const void* h_in, void* h_out, int64_t n_total) {
  int rc = check_ready(p);
  if (rc) return rc;
  if (p->batch_sets < 1) return fail(DBP_ESTATE, "dbp_plan_set_coeff_batch has not been called");
  if (!h_in || !h_out) return fail(DBP_EINVAL, "null host buffer");
  if (n_total < 1) return fail(DBP_EINVAL, "signal must contain at least one sample");
  DeviceGuard g(p->device);
  const size_t in_bytes = (size_t)n_total * 2 * sizeof(float2);
  const size_t out_bytes = in_bytes * p->batch_sets;
  rc = ensure_staging(p, out_bytes > in_bytes ? out_bytes : in_bytes);
  if (rc) return rc;
  cudaStream_t s = p->streams[0];
  DBP_CUDA(cudaMemcpyAsync(p->d_stage[0][0], h_in, in_bytes, cudaMemcpyHostToDevice, s), "H2D");
  const int64_t nb = (n_total + p->step - 1) / p->step;
  rc = dbp_run_coeff_batch(p, p->d_stage[0][0], p->d_stage[0][1], n_total, 0, nb, s);
  if (rc) return rc;
  DBP_CUDA(cudaMemcpyAsync(h_out, p->d_stage[0][1], out_bytes, cudaMemcpyDeviceToHost, s), "D2H");
  DBP_CUDA(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  return DBP_OK;
}

int dbp_host_alloc(void** ptr, size_t bytes) {
  if (!ptr) return fail(DBP_EINVAL, "null pointer");
  *ptr = nullptr;
  cudaError_t e = cudaHostAlloc(ptr, bytes, cudaHostAllocPortable);
  if (e != cudaSuccess) return fail(DBP_ENOMEM, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
  return DBP_OK;
}

int dbp_host_free(void* ptr) {
  if (!ptr) return DBP_OK;
  DBP_CUDA(cudaFreeHost(ptr), "cudaFreeHost");
  return DBP_OK;
}

}  // extern "C"
