/* greentherm_b200.h — batched / device-resident extension of greentherm.h.
 *
 * The reference C ABI cannot take a caller-supplied variation map per sample
 * (refresh_random, reference greens.cpp:448-454, is not exported) and runs one
 * sample per thread (reference solver.cpp:376-387). These entry points keep
 * the reference conventions (gt_status return, thread-local last error,
 * caller-owned out objects, borrowed inputs) and add:
 *   - a prepared, device-resident GreensSet (reference PreparedGreens,
 *     solver.cpp:113-121, built once instead of on every call);
 *   - the Monte-Carlo steady composition of the reference run_one
 *     (solver.cpp:353-374) over a batch of (power map, variation map) pairs,
 *     from host buffers (end-to-end) or device buffers (resident).
 *
 * Per-sample semantics (mode A, reference closed forms):
 *   p_leak0 = leak_frac * p_dyn * var            (leakage_baseline with
 *                                                 d_length = ln(var)/beta_L)
 *   mu      = mean(p_leak0), p_var = p_leak0 - mu
 *   T       = max(0, conv(F_det, p_dyn + p_leak0) + f_rand o p_var * sum * rand_scale)
 * with F_det / f_rand from the closed forms at mu_used = mu (mu_per_sample=1)
 * or the GreensSet mu (mu_per_sample=0, the reference monte_carlo choice).
 */
#ifndef GREENTHERM_B200_H
#define GREENTHERM_B200_H

#include <stddef.h>

#include "greentherm.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { GT_FP32 = 0, GT_FP64 = 1 };

/* Per-sample status bits reported by the batch solves. */
enum {
    GT_SAMPLE_BAD_POWER = 1,
    GT_SAMPLE_BAD_VAR = 2,
    GT_SAMPLE_RUNAWAY_DET = 4,
    GT_SAMPLE_RUNAWAY_RAND = 8,
    GT_SAMPLE_NONFINITE = 16,
    GT_SAMPLE_NOCONVERGE = 32,
    GT_SAMPLE_KIRCHHOFF = 64,
    GT_SAMPLE_ILLCOND = 128
};

/* Build a GreensSet from arrays (n x n row-major doubles) instead of a
 * calibration directory; g_sp0 may be NULL (then f_sp0 + f_sp0(c,c) - kappa_inf,
 * reference greens.cpp:170-175). f_det/f_rand/p_var may be NULL (zero maps). */
gt_status gt_greens_from_arrays(int n, double pitch, const double* f_sp0, const double* g_sp0,
                                double phi, double kappa_inf, double alpha, double beta,
                                double mu, double capacitance, double rand_scale,
                                const double* f_det, const double* f_rand, const double* p_var,
                                gt_greens** out);

typedef struct gt_device_greens gt_device_greens;

/* Prepare the device tables (baseline kernel spectrum, alpha multiplier, ...)
 * for `precision` (GT_FP32 / GT_FP64) on CUDA device `device`. */
gt_status gt_greens_to_device(const gt_greens* g, int precision, int device,
                              gt_device_greens** out);
void gt_device_greens_free(gt_device_greens* d);
int gt_device_greens_precision(const gt_device_greens* d);

typedef struct gt_batch_opts {
    double leak_frac;    /* p_leak0 = leak_frac * p_dyn * var (0.3 for the benchmark) */
    int mu_per_sample;   /* 1: sample mean leakage in the closed forms; 0: GreensSet mu */
    int with_rand;       /* 0 omits the shift-variant term                       */
    int chunk;           /* samples in flight per pass (0 = automatic)          */
    double exponent_cap; /* |ln var| guard, 0 = reference default 6.0            */
    double fp64_check;   /* GT_FP32 handles: pairs whose max 1/|den2|^2 (random_greens
                            denominator) exceeds this are re-solved in fp64 on the
                            device (0 = default 1e4; < 0 = off). Re-solved pairs
                            report a negative gt_sample_stats.max_rden2; pairs beyond
                            the re-solve capacity (batch/16) get GT_SAMPLE_ILLCOND. */
} gt_batch_opts;

void gt_batch_opts_default(gt_batch_opts* o);

/* Per-sample results (device layout of gt_mc_batch_device's `stats`). */
typedef struct gt_sample_stats {
    double sum_leak, sum_applied, sum_rise, max_rise, mean_rise, mu;
    unsigned long long max_bits;
    int status;
    float max_rden2;  /* max over frequencies of 1/|den2|^2 (random_greens denominator): fp32 conditioning */
} gt_sample_stats;

/* End-to-end batch from host memory: p_dyn, var are batch x n x n in the
 * device precision (float* for GT_FP32, double* for GT_FP64; pinned memory is
 * fastest). t_out (same type, may be NULL) receives the rise maps; max_out /
 * mean_out / status_out (may be NULL) receive per-sample results. Copies are
 * overlapped with compute in chunks. online_ms = wall time of the call. */
gt_status gt_mc_batch(const gt_device_greens* d, const void* p_dyn, const void* var, int batch,
                      const gt_batch_opts* opts, void* t_out, double* max_out, double* mean_out,
                      int* status_out, double* online_ms);

/* Device-resident batch: all pointers are device memory on the greens'
 * device; stats is batch x gt_sample_stats. Enqueued on `stream` (a
 * cudaStream_t; NULL = the library's own stream, pass cudaStreamLegacy for the
 * legacy default stream); returns without synchronising. Calls on one handle
 * share its scratch, so each call's stream first waits for the previous
 * call's work on the handle (whatever stream that used): calls on different
 * streams are ordered, never overlapped. The same holds for every *_device
 * entry point below. */
gt_status gt_mc_batch_device(const gt_device_greens* d, const void* p_dyn, const void* var,
                             int batch, const gt_batch_opts* opts, void* t_out,
                             gt_sample_stats* stats, void* stream);

/* ---- mode B: the north-star leakage fixed point ----
 * Per sample, the outer loop of the reference FDM oracle (fdm.cpp:167-205)
 * with the linear solve replaced by the Green convolution of the baseline
 * kernel spectrum on the mirror-padded torus:
 *   theta_{k+1} - T0 = crop(IFFT(fk . FFT(mirror(P + L0 f(T_k)))))
 *   L0 = leak_frac * p_dyn * var, f(dT) = exp(beta dT) (law 1) or 1 + beta dT (law 0)
 *   T = Kirchhoff inverse of theta for k = k_ref (T/T0)^-eta (kirchhoff = 1)
 * Stops when max|T_{k+1} - T_k| < tol after iteration 1; max_iters ->
 * GT_SAMPLE_NOCONVERGE (ConvergenceError); non-finite / Kirchhoff-invalid
 * temperatures (thermal runaway) -> GT_SAMPLE_NONFINITE / GT_SAMPLE_KIRCHHOFF. */
typedef struct gt_fp_opts {
    double leak_frac;
    int law;
    int kirchhoff;
    double beta, t_ambient, eta, tol;
    int max_iters;
    int chunk;
    double fp32_stage_tol; /* GT_FP32 handles (BASELINE config 1: "fp32 with fp64 residual
                              check"): the fp32 iteration stops at this tolerance, then
                              fp64 iterations warm-started from it finish to `tol`
                              (0 = default: 5e-4, or 1e-2 with accel < 0 whose history the
                              fp64 stage continues; < 0 = fp32 only). Iteration counts add up. */
    int with_rand;         /* 1: combined config 2 -- every iteration adds the reference's
                              shift-variant term h * sum(applied), h = f_rand o p_var *
                              rand_scale with f_rand = random_greens at the GreensSet mu
                              from the sample's leakage baseline (greens.cpp:225-251,
                              solver.cpp:169-174), before the Kirchhoff inverse. */
    int accel;             /* 0: plain Picard iteration (the reference outer loop,
                              fdm.cpp:167-205: iteration counts match it); k0 > 0:
                              Chebyshev semi-iteration from iteration k0 on, with the
                              contraction rate estimated per sample from the residual
                              ratio there; same stop rule on max|G(T) - T|.
                              -m (m = 1..4): Anderson(m) mixing on the 16 x 16 lowest cosine
                              modes of the die field between the column and row passes
                              (fixed_point.cu fp_lowmode; slab.py on the large-grid path):
                              the same fixed point, stop rule on max|T_{k+1} - T_k|. */
    int warm_start;        /* 1: the t_out map holds the initial temperature rise T_0 on
                              entry (device entry; e.g. the mode-A closed-form solution of
                              the same pair), 0: T_0 = 0 as the reference loop starts. */
} gt_fp_opts;

void gt_fp_opts_default(gt_fp_opts* o);

/* Host arrays (device precision); t_out / iters_out / status_out / max_out may be NULL. */
gt_status gt_fp_batch(const gt_device_greens* d, const void* p_dyn, const void* var, int batch,
                      const gt_fp_opts* opts, void* t_out, int* iters_out, int* status_out, double* max_out,
                      double* online_ms);
/* Device arrays; t_out (batch x n x n, required) holds the state and the result. */
gt_status gt_fp_batch_device(const gt_device_greens* d, const void* p_dyn, const void* var, int batch,
                             const gt_fp_opts* opts, void* t_out, int* iters_out, int* status_out,
                             double* max_out, double* mean_out, void* stream);
size_t gt_fp_scratch_bytes(int n, int precision);

/* ---- Batched transient traces with the leakage update every step (config 3).
 * Per trace b (north-star; oracle: the reference's time_varying_profile,
 * solver.cpp:212-287, driven one step at a time):
 *   P_n = P_dyn,n + L0 o f(T_{n-1}),  T_0 = 0,  f = 1 + beta dT (law 0, variation.cpp:213-222) or exp
 *   T_n = max(0, windowed superposition over window k of P_1..P_n)   (with_rand off)
 * P_dyn,n is piecewise constant over blocks: P_dyn,n(x,y) = sched[b][n-1][blk[b][x][y]]
 * (per-cell watts). blk / leak0 with stride 0 are shared by all traces.
 * T_n is stored for n = out_stride, 2 out_stride, ... into t_out[b][frame][n][n];
 * max_out[b][frame] is its maximum. Spectra r = exp(-dt/tau), r^(k+1) and F_det
 * come from the GreensSet (alpha, beta, mu, capacitance) exactly as for
 * gt_solve_trace; a non-positive Re tau or a runaway F_det is GT_ERR_SOLVER. */
typedef struct gt_trace_opts {
    double dt;       /* seconds per step */
    int steps;
    int window;      /* k; <= 0 selects ceil(5 ms / dt) (solver.cpp:224-226); clipped to steps */
    int law;         /* 0 linear, 1 exp */
    double beta;     /* leakage temperature coefficient, 1/K */
    int out_stride;  /* store every out_stride-th step (steps % out_stride frames) */
    int chunk;       /* traces per in-flight chunk; 0 = auto */
} gt_trace_opts;

void gt_trace_opts_default(gt_trace_opts* o);
/* Device arrays in the device precision (blk: int32). */
gt_status gt_trace_batch_device(const gt_device_greens* d, const int* blk, long long blk_stride, const void* sched,
                                int nblk, const void* leak0, long long leak_stride, int batch,
                                const gt_trace_opts* opts, void* t_out, double* max_out, void* stream);
/* Device scratch bytes per in-flight trace (power ring of window + 2 maps, spectral state). */
size_t gt_trace_scratch_bytes(int n, int precision, int window);

/* ---- Large single grid (config 4), fp64, one slab of a multi-GPU solve per call.
 * The mode-B fixed point of gt_fp_batch on ONE map of side n (m = 2n = M1 * M2,
 * four-step transforms), split into three phases so a driver can place an
 * all-to-all transpose between the row and the column phases
 * (paper_2307_12119_b200/slab.py). All pointers are device pointers; the
 * device GreensSet must be GT_FP64.
 *   rows_fwd : applied rows [2 pairs][n] -> Z [pairs][m] (spectra of the
 *              mirrored rows, two rows per line); s1 = pairs x m complex scratch
 *   cols     : Z of ALL pairs (compact = 0: [n/2][m]; 1: [n/2][2 hc] columns
 *              c0.. and their mirrors m - c0 - c) -> y [n][hc] = rows [0, n) of
 *              IFFT_col(fk . FFT_col(.)) for half-spectrum columns [c0, c0+hc);
 *              c1, c2 = m x hc complex scratch
 *   rows_inv : y [2 pairs][hy] (columns 0..n) -> theta -> T (t, [2 pairs][n], in
 *              place: old T in, new T out) -> next applied rows P + L0 f(T);
 *              max |T_new - T_old| is atomically max-ed into res_bits (double
 *              bits), sample status bits OR-ed into *status. */
/* f_sp0 alone (the reference impulse_response, 1 W at (c, c), fdm.cpp:288-296) by the
 * device modal solution of the stack file's network, for power-of-two n up to 16384
 * (the full gt_calibrate is limited to n <= 1024). Call with f_sp0_out = NULL to read n. */
gt_status gt_modal_kernel(const char* stack_path, int* n_out, double* f_sp0_out);
gt_status gt_large_geometry(const gt_device_greens* d, int* m1, int* m2);
/* Layout of rows_fwd's output `z` (and of what cols / cols_peer read from it):
 * dct_rows = 1 (n <= 8192): the rows' real DCT-II coefficients [2 pairs][n + 1] doubles
 *   (the mirrored row's half spectrum is conj(exp(-i pi v / m)) C[v]); a compact cols input is
 *   then [n][hc] doubles (columns c0.. of every die row, rank-major);
 * dct_rows = 0 (larger n): packed row-pair spectra [pairs][m] complex, compact [n/2][2 hc]. */
gt_status gt_large_row_layout(const gt_device_greens* d, int* dct_rows);

/* Low-mode Anderson mixing of gt_fp_opts.accel = -m on the large-grid path (slab.py drives it
 * between gt_large_cols* and gt_large_rows_inv): `y` is this rank's part [rows][hy] (complex
 * fp64) of the row buffer, holding die rows row0 .. row0 + rows - 1.
 *   project: coef[256] = the slab's share of the 16 x 16 lowest cosine coefficients of G(x_k)
 *            (partial: scratch of gt_large_lowmode_partial_blocks(rows) x 256 doubles); a
 *            multi-GPU driver all-reduces coef over the ranks (sum);
 *   mix:     one Anderson(depth <= 4) step on the summed coefficients (state:
 *            gt_large_lowmode_state_bytes() bytes, initialised by gt_large_lowmode_init;
 *            res_prev: the residual of the previous iteration) -> corr[256];
 *   apply:   the correction's row spectra added to columns [0, 16) of y.
 * All device pointers; no host synchronisation. */
size_t gt_large_lowmode_state_bytes(void);
int gt_large_lowmode_partial_blocks(int rows);
gt_status gt_large_lowmode_init(void* state, void* stream);
gt_status gt_large_lowmode_project(const gt_device_greens* d, const void* y, int hy, int rows, int row0,
                                   double* partial, double* coef, void* stream);
gt_status gt_large_lowmode_mix(void* state, const double* coef, int depth, double res_prev, double* corr,
                               void* stream);
gt_status gt_large_lowmode_apply(const gt_device_greens* d, void* y, int hy, int rows, int row0, const double* corr,
                                 void* stream);
gt_status gt_large_rows_fwd(const gt_device_greens* d, const double* app, int pairs, void* s1, void* z,
                            void* stream);
gt_status gt_large_cols(const gt_device_greens* d, const void* z, int compact, int c0, int hc, void* c1, void* c2,
                        void* y, void* stream);
gt_status gt_large_rows_inv(const gt_device_greens* d, const void* y, int hy, int pairs, void* s1, double* t,
                            double* app, const double* p, const double* l0, const gt_fp_opts* opts,
                            unsigned long long* res_bits, int* status, void* stream);
/* cols over peer memory: the multi-GPU column phase without all-to-all copies.
 * z_ranks / y_ranks are DEVICE arrays of `world` pointers, each mapped into this
 * process (gt_ipc_open for other GPUs): z_ranks[r] = rank r's rows_fwd output
 * [pairs_per_rank][m], y_ranks[r] = rank r's row buffer [2 pairs_per_rank][hy]
 * (hy >= n + 1). The columns [c0, c0 + hc) are read from every rank's spectra in
 * place (peer loads overlapped with the FFT work) and rows [0, n) of the result are
 * stored straight into their owners' row buffers at columns c0.. (peer stores). The
 * caller orders the phases across ranks (a barrier after rows_fwd and after cols). */
gt_status gt_large_cols_peer(const gt_device_greens* d, const void* z_ranks, int world, int pairs_per_rank, int c0,
                             int hc, void* c1, void* c2, const void* y_ranks, int hy, void* stream);
/* CUDA IPC helpers for the peer exchange: gt_ipc_alloc returns a device buffer and its
 * 64-byte handle; gt_ipc_open maps another process's handle (peer access enabled). */
gt_status gt_ipc_alloc(size_t bytes, void** ptr, void* handle64);
gt_status gt_ipc_open(const void* handle64, void** ptr);
gt_status gt_ipc_close(void* ptr);
gt_status gt_ipc_free(void* ptr);
/* rows_inv with the Chebyshev semi-iteration of gt_fp_opts.accel (slab.py drives omega /
 * gamma from the residual history): x_prev [2 pairs][n] holds x_{k-1} on entry and x_k on
 * exit, g_out (may be NULL) receives G(x_k); omega > 0 stores x_{k+1} =
 * omega (gamma G(x_k) + (1 - gamma) x_k - x_{k-1}) + x_{k-1} in t (and the next applied
 * rows from it); omega <= 0 is the plain Picard step. The residual is max|G(x_k) - x_k|. */
gt_status gt_large_rows_inv_accel(const gt_device_greens* d, const void* y, int hy, int pairs, void* s1, double* t,
                                  double* app, const double* p, const double* l0, const gt_fp_opts* opts,
                                  unsigned long long* res_bits, int* status, double* x_prev, double* g_out,
                                  double omega, double gamma, void* stream);

/* ---- Seeded variation maps generated on the device (n = 64, 128, 256).
 * The config-1 variation model: var = 1 + sigma_over_mu * z, z a unit-variance
 * Gaussian random field with the reference's spherical correlogram
 * (variation.cpp:75-79) of range range_frac x die width, by circulant embedding
 * on the 2n torus (gen_systematic_map, variation.cpp:87-132), drawn from
 * counter-based Philox noise: a sample depends only on its 64-bit seed, not on
 * the batch it is generated in. Same distribution as the reference generator,
 * not the same samples (gt_monte_carlo keeps the reference's own RNG stream).
 *   gt_var_model       : prepare sqrt(lambda) on the device set (once)
 *   gt_var_generate_device : device seeds -> device maps [batch][n][n]
 *   gt_mc_batch_seeded : gt_mc_batch with var generated on the device from host
 *                        seeds (the reference monte_carlo takes seeds, not maps):
 *                        only the power maps cross PCIe */
gt_status gt_var_model(gt_device_greens* d, double sigma_over_mu, double range_frac);
gt_status gt_var_generate_device(const gt_device_greens* d, const unsigned long long* seeds, int batch, void* var_out,
                                 void* stream);
gt_status gt_mc_batch_seeded(const gt_device_greens* d, const void* p_dyn, const unsigned long long* seeds, int batch,
                             const gt_batch_opts* opts, void* t_out, double* max_out, double* mean_out,
                             int* status_out, double* online_ms);

/* Bytes of device scratch a device-resident batch uses per in-flight sample,
 * and the number of kernels it launches for (batch, chunk). */
size_t gt_mc_scratch_bytes(int n, int precision);
int gt_mc_kernel_launches(int batch, int chunk);

/* Per-pass profiling of device batches: between begin and end every batch
 * call records CUDA events on its stream around the three fused passes;
 * end() synchronises and returns the summed milliseconds per pass
 * (pass_ms[0..2] = row / column / row pass, pass_ms[3] = their sum), the
 * kernels launched and the batch calls made since begin. */
gt_status gt_profile_begin(gt_device_greens* d);
/* mode 0: as gt_profile_begin; mode 1: events around the column pass only (the
 * dominant kernel; two events per chunk instead of four keep a timed region's
 * launch stream lighter), pass_ms[0] = pass_ms[2] = 0. */
gt_status gt_profile_begin_mode(gt_device_greens* d, int mode);
gt_status gt_profile_end(gt_device_greens* d, double* pass_ms, long long* kernels, long long* calls);
/* Kernels launched by this prepared set since the last gt_profile_begin. */
long long gt_kernel_launches(const gt_device_greens* d);

/* Device count visible to the library (0 without a GPU). */
int gt_device_count(void);

#ifdef __cplusplus
}
#endif

#endif /* GREENTHERM_B200_H */
