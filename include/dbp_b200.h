/*
 * dbp_b200.h -- C ABI of the B200-native overlap-save digital-backpropagation
 * library (libdbp_b200.so).
 *
 * This is the drop-in boundary for the reference's DBP hot path
 * (pkg/src/fiberdbp/dbp.py:160 ``backpropagate`` driving
 * pkg/src/fiberdbp/spectral.py:87 ``overlap_save_run``).  Plain pointers and
 * sizes only; no torch, numpy or C++ types cross it.  Every function returns
 * DBP_OK (0) or a negative error code and never throws; the message of the
 * last failure on the calling thread is available from dbp_last_error().
 *
 * Sample layout everywhere: complex64 (interleaved float re, im), batch-major
 * rows ``[item][polarisation x|y][sample]``, i.e. each item is the reference's
 * DualPolSignal.stack() (sigkit.py:73-75) in single precision.
 *
 * Threading: a plan belongs to one device; calls on one plan must be
 * serialised by the caller.  Plans on different devices may be driven
 * concurrently from different threads.
 */
#ifndef DBP_B200_H
#define DBP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DBP_OK 0
#define DBP_EINVAL (-1)   /* invalid argument  (reference: ValueError)  */
#define DBP_ECUDA (-2)    /* CUDA runtime failure / no device           */
#define DBP_ENOMEM (-3)   /* device or pinned-host allocation failed   */
#define DBP_ESTATE (-4)   /* plan not configured (set_linear/set_steps) */

/* algorithms: dbp.py:25 ALGORITHMS = ("ffe", "ssfm", "essfm"); 3 = rotation
 * only (the nonlinear sub-step alone, dbp.py:49 / channel.py:61); 4 = no
 * operator at all: the overlap-save framing alone, i.e. overlap_save_run
 * with the identity block processor (spectral.py:87-145, the reference's
 * `lambda b: b` in test_spectral.py:72-76 and 119-125).  An FFE program whose
 * kernel is any caller-supplied filter H is the block processor
 * `ifft(fft(b) * H)` (test_spectral.py:78-97).                              */
#define DBP_ALG_FFE 0
#define DBP_ALG_SSFM 1
#define DBP_ALG_ESSFM 2
#define DBP_ALG_ROTATE 3
#define DBP_ALG_IDENTITY 4

/* arrangements: dbp.py:32 ARRANGEMENTS                                      */
#define DBP_ARR_SYMMETRIC 0
#define DBP_ARR_LINEAR_FIRST 1
#define DBP_ARR_NONLINEAR_FIRST 2

#define DBP_MAX_SIDE_COEFFS 64   /* EssfmCoefficients.n_coeffs supported   */
/* OverlapPlan.block_len: any power of two up to 2^DBP_MAX_LOG2_BLOCK (the
 * reference accepts any power of two, spectral.py:72-76).  Lengths in
 * [DBP_MIN_BLOCK_LEN, DBP_MAX_BLOCK_LEN] run the fused block kernel; shorter
 * and longer blocks the float64 multi-kernel path (dbp_general.cuh), with
 * the same entry points and results within the same tolerance.             */
#define DBP_MIN_BLOCK_LEN 16
#define DBP_MAX_BLOCK_LEN 8192
#define DBP_MAX_LOG2_BLOCK 22

typedef struct dbp_plan dbp_plan;

/* Message of the last failure on this thread ("" if none). */
const char* dbp_last_error(void);

/* ABI version (major * 100 + minor): 102 adds the general block-length path. */
int dbp_version(void);

/* Number of visible CUDA devices (0 when none). */
int dbp_device_count(int* count);

/* Plan for OverlapPlan(block_len, overlap) on ``device``
 * (replaces the geometry checks of spectral.py:63-81).                      */
int dbp_plan_create(dbp_plan** out, int device, int block_len, int overlap);
int dbp_plan_destroy(dbp_plan* plan);

/* Linear sub-step filters, natural FFT bin order, interleaved (re, im)
 * float64, length 2*block_len each, exactly as the reference builds them
 * (dbp.py:186 for FFE; dbp.py:196-197 ``kernel`` / ``half_kernel``).  The
 * library folds numpy's 1/N inverse normalisation in and rounds to
 * complex64.  ``half_kernel`` may be NULL unless the symmetric arrangement
 * of a split-step program is used.                                          */
int dbp_plan_set_linear(dbp_plan* plan, const double* kernel, const double* half_kernel);

/* Step program (dbp.py:193-233).  ``weights``/``gains`` hold the reverse
 * schedule's per-step nonlinear weight and amplitude gain in processing
 * order (dbp.py:112-157), ``gamma`` the value the reference passes to the
 * sub-step (i.e. -link.gamma, dbp.py:203/207); each rotation is
 * exp(-j * gamma * weight_j * F).  ``coeffs`` = c_0..c_{n_coeffs} for
 * ESSFM (sigkit.py:152-183), ignored otherwise.  FFE ignores everything
 * but ``algorithm``.                                                         */
int dbp_plan_set_steps(dbp_plan* plan, int algorithm, int arrangement, int num_steps,
                       const double* weights, const double* gains, double gamma,
                       const double* coeffs, int n_coeffs);

/* Number of overlap-save blocks ceil(n_total / (N - M)) (spectral.py:126). */
int dbp_num_blocks(const dbp_plan* plan, int64_t n_total, int64_t* out);

/* Whole-signal run on device buffers (the GPU replacement of
 * overlap_save_run(sig, plan, process), spectral.py:87-145): ``d_in`` and
 * ``d_out`` are [batch][2][n_total] complex64; blocks
 * [block_begin, block_end) of every item are processed with the circular
 * extension of the whole signal and their kept centres written to the
 * matching output samples.  Asynchronous on ``stream`` (cudaStream_t, NULL =
 * legacy default stream).                                                    */
int dbp_run(dbp_plan* plan, const void* d_in, void* d_out, int64_t n_total, int batch,
            int64_t block_begin, int64_t block_end, void* stream);

/* Chunk run for sharding a long stream: ``d_in`` is [batch][2][in_len]
 * holding global samples [block_begin*step - M/2, ...) already extended
 * cyclically by the caller (in_len >= (block_end-block_begin)*step + M);
 * ``d_out`` is [batch][2][out_len] receiving global samples
 * [block_begin*step, min(block_end*step, n_total)).                          */
int dbp_run_chunk(dbp_plan* plan, const void* d_in, void* d_out, int64_t n_total, int batch,
                  int64_t block_begin, int64_t block_end, int64_t in_len, int64_t out_len,
                  void* stream);

/* Host-buffer run: h_in/h_out are [batch][2][n_total] complex64 in host
 * memory (pinned for full PCIe speed; pageable rows of whole waveforms of
 * 2^16 samples and more are staged through the plan's pinned buffers by
 * host threads, same bits).  Copies in, processes blocks [block_begin,
 * block_end) and copies the kept samples out, pipelined over two streams;
 * returns after completion (the reference's synchronous semantics).          */
int dbp_run_host(dbp_plan* plan, const void* h_in, void* h_out, int64_t n_total, int batch,
                 int64_t block_begin, int64_t block_end);

/* The drop-in call itself: backpropagate(sig, cfg) (dbp.py:160) on the
 * reference's complex128 rows -- h_x, h_y: n_total complex128 samples of
 * each polarisation (DualPolSignal.x / .y, sigkit.py:56-68), h_out_x,
 * h_out_y: complex128 results of the same length.  The whole signal, cyclic
 * framing (spectral.py:122-145).  The complex128 -> complex64 casts (numpy's
 * astype rounding) and back run on host threads (DBP_HOST_THREADS, default
 * min(16, cores)) into pinned staging, pipelined over block-range chunks
 * (a quarter of the signal within [2^16, 2^21] samples) with halos against
 * the H2D copy, the kernel and the D2H copy.  The result rows must not
 * overlap the input rows or each other (DBP_EINVAL): like the reference
 * (spectral.py:129) the call never mutates its input.  Synchronous; bitwise
 * equal to dbp_run_host on the complex64 cast.                               */
int dbp_backpropagate_c128(dbp_plan* plan, const void* h_x, const void* h_y, void* h_out_x, void* h_out_y,
                           int64_t n_total);

/* The nonlinear sub-step alone on one (2, n) block of ANY length n > 2 N_c
 * (dbp.py:49-75 nonlinear_substep_essfm; channel.py:61-71 is N_c = 0, c = 1):
 * float64 like the reference, cyclic FIR indices inside the block,
 * h_out = h_block * exp(-j gamma dz_eff F).  Host complex128 (2, n) buffers;
 * coeffs = c_0 .. c_{n_coeffs}.  Synchronous.                                */
int dbp_nonlinear_substep_c128(int device, const void* h_block, void* h_out, int64_t n, double gamma,
                               double dz_eff, const double* coeffs, int n_coeffs);

/* Device staging budget (bytes) used by dbp_run_host (default 256 MiB: 32   
 * pipelined chunks for the configs[3] batch, so the un-overlapped first    
 * H2D and last D2H stay short).                                             */
int dbp_plan_set_staging(dbp_plan* plan, size_t bytes);

/* Unit seam: apply the configured per-block operator (the reference's
 * ``process`` closure, dbp.py:212-233) to n_blocks full (2, N) blocks,
 * [n_blocks][2][N] complex64 -> same shape, every sample kept.              */
int dbp_process_blocks(dbp_plan* plan, const void* d_blocks, void* d_out, int64_t n_blocks,
                       void* stream);

/* Overlap-save framing alone, for block processors the fused kernel cannot
 * run (spectral.py:84-92 accepts any callable; replaces the cyclic extension
 * and block cut of overlap_save_run, spectral.py:122-131, and its keep-centre
 * assembly, spectral.py:138-145).  Pure data movement, bit-exact for either
 * element width: elem_bytes 8 (complex64) or 16 (complex128).
 *   dbp_frame_blocks:   d_sig [batch][2][n_total] -> d_blocks
 *                       [batch][block_end-block_begin][2][block_len], block b
 *                       holding samples (b step - overlap/2 + j) mod n_total.
 *   dbp_unframe_blocks: d_blocks (same layout) -> d_out [batch][2][n_total],
 *                       writing samples [block_begin step, min(n_total,
 *                       block_end step)) from each block's centre
 *                       [overlap/2, overlap/2 + step).
 * Asynchronous on ``stream``; block_len a power of two, 0 <= overlap <
 * block_len (spectral.py:72-76).                                             */
int dbp_frame_blocks(const void* d_sig, void* d_blocks, int64_t n_total, int batch, int block_len,
                     int overlap, int64_t block_begin, int64_t block_end, int elem_bytes, void* stream);
int dbp_unframe_blocks(const void* d_blocks, void* d_out, int64_t n_total, int batch, int block_len,
                       int overlap, int64_t block_begin, int64_t block_end, int elem_bytes, void* stream);

/* Per-item coefficient sets for ESSFM training batches (the reference's
 * finite-difference Jacobian evaluates N_c+1 perturbed sets on one
 * waveform, train.py:153-158): ``coeffs`` is [n_sets][n_coeffs + 1]
 * float64.  Used only by the *_coeff_batch entry points.                   */
int dbp_plan_set_coeff_batch(dbp_plan* plan, const double* coeffs, int n_sets, int n_coeffs);

/* One waveform d_in [2][n_total], every coefficient set: d_out is
 * [n_sets][2][n_total], item i processed with set i (blocks
 * [block_begin, block_end)).  Asynchronous on ``stream``.                   */
int dbp_run_coeff_batch(dbp_plan* plan, const void* d_in, void* d_out, int64_t n_total,
                        int64_t block_begin, int64_t block_end, void* stream);

/* Host-buffer form of dbp_run_coeff_batch (synchronous): h_in [2][n_total],
 * h_out [n_sets][2][n_total] complex64.                                     */
int dbp_run_host_coeff_batch(dbp_plan* plan, const void* h_in, void* h_out, int64_t n_total);

/* Wait for all work the plan queued on its internal streams. */
int dbp_plan_synchronize(dbp_plan* plan);

/* Pinned host memory helpers (cudaHostAlloc / cudaFreeHost). */
int dbp_host_alloc(void** ptr, size_t bytes);
int dbp_host_free(void* ptr);

/* Kernel launches issued by this process so far (evidence counter). */
int64_t dbp_launch_count(void);

/* Measurement utility (not on the DBP path): FP32 FFMA throughput of
 * ``device`` in TFLOP/s from an 8-accumulator FFMA kernel over all SMs,
 * ``iters`` x 16 x 8 FMAs per thread; ``ms`` receives the kernel time.
 * bench.py uses it as the FP32 roofline denominator.                        */
int dbp_probe_fp32_peak(int device, int iters, double* tflops, double* ms);
/* The same with sm_100a's packed FFMA2 (fma.rn.f32x2: two float32 FMAs per
 * lane per instruction); the FP32 roofline uses the larger of the two.      */
int dbp_probe_fp32x2_peak(int device, int iters, double* tflops, double* ms);
/* Packed and scalar FMAs interleaved (8 FFMA2 + scalar_chains FFMA chains per
 * step, scalar_chains in {2, 4, 8, 16}): whether the scalar FMA pipe adds
 * throughput beside FFMA2 (roofline denominator check).                     */
int dbp_probe_fp32_mixed_peak(int device, int iters, int scalar_chains, double* tflops, double* ms);

/* ------------------------------------------------------------------------
 * Whole-waveform split-step link simulator: the reference's
 * propagate_span / amplify_with_ase / apply_jones_matrix
 * (pkg/src/fiberdbp/channel.py:74-153) for a batch of circular waveforms of
 * n = 2^log2_n samples (n in [2^8, 2^26]).  The simulator owns the device
 * waveform buffer [item][pol][n] complex64; all calls are synchronous.
 * ------------------------------------------------------------------------ */
typedef struct dbp_sim dbp_sim;

int dbp_sim_create(dbp_sim** out, int device, int log2_n, int max_batch);
int dbp_sim_destroy(dbp_sim* sim);
int dbp_sim_length(const dbp_sim* sim, int64_t* n);
int dbp_sim_upload(dbp_sim* sim, const void* h_in, int batch);     /* [batch][2][n] complex64 */
int dbp_sim_download(dbp_sim* sim, void* h_out, int batch);

/* ``steps`` SSFM steps of one span (channel.py:74-94): per step
 * x <- ifft(fft(x) exp(-j 2 pi^2 beta2 1e-24 f^2 dz)), then (nonlinear != 0)
 * x <- x exp(-j gamma dz_eff (|x|^2 + |y|^2)), then x <- x * loss.          */
int dbp_sim_span(dbp_sim* sim, int batch, double sample_rate, double beta2, double gamma, double dz,
                 double dz_eff, double loss, int steps, int nonlinear);

/* Span-end amplifier (channel.py:97-153): x <- J (g_amp x + noise) with
 * ``h_noise`` a host [batch][2][n] complex64 noise realisation (NULL: none)
 * and ``jones`` one row-major 2x2 complex matrix per waveform, [batch][2][2]
 * complex as 8 * batch doubles (NULL: no rotation).                         */
int dbp_sim_amplify(dbp_sim* sim, int batch, double g_amp, const void* h_noise, const double* jones);

/* ------------------------------------------------------------------------
 * Post-DBP receiver DSP: pkg/src/fiberdbp/modem.py
 * butterfly_equalize (:207-271), carrier_recover (:283-351), qpsk_decide
 * (:116-125) and the counting core of measure_ber (:358-413), in float64,
 * for a batch of waveforms of 2 n_symbols samples (2 samples/symbol).
 * Buffers are host memory; every call is synchronous.
 * ------------------------------------------------------------------------ */
typedef struct dbp_rx dbp_rx;

int dbp_rx_create(dbp_rx** out, int device, int64_t n_symbols, int max_batch);
int dbp_rx_destroy(dbp_rx* rx);

/* CMA 2x2 butterfly, T/2 spaced, centre-spike start, ``passes`` circular
 * sweeps with the collapse re-initialisation of modem.py:259-266.
 * h_in [batch][2][2 n_symbols] complex128 -> h_out [batch][2][n_symbols]
 * complex128; reinits[batch] and h_taps [batch][4][taps] (hxx, hxy, hyx,
 * hyy) complex128 may be NULL.  taps odd, <= 64.                           */
int dbp_rx_equalize(dbp_rx* rx, const void* h_in, int batch, int taps, double step_size, int passes,
                    void* h_out, int* reinits, void* h_taps);

/* 4th-power frequency-offset removal, sliding-window phase tracking and (with
 * h_ref [2][n_symbols] complex128, else NULL) the 90-degree rotation search.
 * h_sym -> h_out [batch][2][n_symbols] complex128; f_off[batch] (may be NULL);
 * status[batch] = 1 where the offset sits at the aliasing edge (the
 * reference's FrequencyOffsetError), else 0.                                */
int dbp_rx_carrier_recover(dbp_rx* rx, const void* h_sym, int batch, double symbol_rate, const void* h_ref,
                           int window, void* h_out, double* f_off, int* status);

/* Hard decisions: h_bits [batch][2][2 n_symbols], I and Q bits interleaved. */
int dbp_rx_decide(dbp_rx* rx, const void* h_sym, int batch, uint8_t* h_bits);

/* Bit errors at the best circular alignment and polarisation pairing:
 * h_dec [batch][2][2 n_symbols], h_ref [2][2 n_symbols]; errors[batch];
 * *counted = 2 (n_symbols - ceil(skip_bits / 2)) (BER = errors / (2 counted)). */
int dbp_rx_count_errors(dbp_rx* rx, const uint8_t* h_dec, int batch, const uint8_t* h_ref, int64_t skip_bits,
                        int64_t* errors, int64_t* counted);

/* The whole receiver of cli.py:677-685 device-resident: h_in [batch][2][2
 * n_symbols] complex64 (in_is_c64) or complex128, h_ref_sym [2][n_symbols]
 * complex128.  metrics[batch][6] = (ber, errors, bits counted, evm %,
 * frequency offset Hz, re-initialisations); status[batch] = 0 ok, 1
 * frequency offset at the aliasing edge, 2 no alignment below BER 0.4.     */
int dbp_rx_chain(dbp_rx* rx, const void* h_in, int in_is_c64, int batch, int taps, double step_size, int passes,
                 double symbol_rate, const void* h_ref_sym, int window, int64_t skip_bits, double* metrics,
                 int* status);

/* ------------------------------------------------------------------------
 * Device-side residual algebra of the coefficient fit (train.py:130-178).
 * d_out: [sets][2][n_total] complex64 DBP outputs of coefficient sets,
 * d_target / d_base: [2][n_total] complex64 (fine-step target, output of the
 * current coefficients); residuals are (out - target) * scale on samples
 * [w0, w1) of both polarisations, real and imaginary parts, in float64.
 * Synchronous on ``stream``; results are host arrays.
 * ------------------------------------------------------------------------ */
/* h_sums[s] = || r_s ||^2 (line search). */
int dbp_fit_sumsq(const void* d_out, int n_sets, int64_t n_total, const void* d_target, int64_t w0, int64_t w1,
                  double scale, double* h_sums, void* stream);
/* Gauss-Newton normal equations with central differences: sets i and
 * n_params + i hold c + h e_i and c - h e_i; J_i = (r_{+i} - r_{-i}) / (2 h);
 * h_ata [n_params][n_params] = J^T J, h_atr [n_params] = J^T r(base).       */
int dbp_fit_normal(const void* d_out, int n_params, int64_t n_total, const void* d_target, const void* d_base,
                   int64_t w0, int64_t w1, double scale, double fd_step, double* h_ata, double* h_atr,
                   void* stream);

/* Float64 DFT along the last axis of a [batch][n] complex128 host array
 * (spectral.py:37-48: forward unnormalised, inverse x 1/n; n a power of two),
 * the library's own float64 Stockham FFT (csrc/fft64.cuh) -- API
 * completeness, not the DBP path.                                           */
int dbp_fft_c2c(int device, const void* h_in, void* h_out, int64_t n, int64_t batch, int inverse);

/* Laser phase noise (channel.py:156-171): out = in exp(j cumsum(incr)) for a
 * [2][n] complex128 waveform; ``incr`` are the host-drawn Wiener increments
 * (the reference's seeded normal draws), so a seeded run is reproduced.      */
int dbp_phase_noise(int device, const void* h_in, const double* h_incr, void* h_out, int64_t n);

#ifdef __cplusplus
}
#endif

#endif /* DBP_B200_H */
