// gt_device.h — internal thin C ABI between the C++ host layer (capi.cpp) and
// the sm_100a kernels. Plain POD structs, device pointers, dims and a stream;
// no torch or C++ types cross this boundary.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Per-sample scalars accumulated by the fused passes (fp64 accumulation of
 * the compensated sums of the reference, field.cpp:45-57). */
typedef struct gtd_sample_stats {
    double sum_leak;     /* sum of p_leak0 over the die (-> mu)      */
    double sum_applied;  /* sum of p_dyn + p_leak0 (-> Hadamard scale) */
    double sum_rise;     /* sum of the clamped rise map             */
    double max_rise;     /* written by finalize                     */
    double mean_rise;    /* written by finalize                     */
    double mu;           /* mean leakage used for p_var             */
    unsigned long long max_bits; /* double bits of max rise (rise >= 0) */
    int status;          /* bit flags, GTD_ST_*                      */
    float max_rden2;     /* max_(u,v) 1/|den2|^2 of random_greens (conditioning of the fp32 path) */
} gtd_sample_stats;

enum {
    GTD_ST_BAD_POWER = 1,     /* p_dyn < 0 or non-finite  -> ConfigError   */
    GTD_ST_BAD_VAR = 2,       /* var <= 0 / non-finite / |ln var|>cap      */
    GTD_ST_RUNAWAY_DET = 4,   /* |den| < 1e-6 in deterministic_spectrum    */
    GTD_ST_RUNAWAY_RAND = 8,  /* |den| < 1e-6 in random_greens             */
    GTD_ST_NONFINITE = 16,    /* non-finite rise                           */
    GTD_ST_NOCONVERGE = 32,   /* fixed point hit max_iters                 */
    GTD_ST_KIRCHHOFF = 64,    /* Kirchhoff inverse left its validity range */
    GTD_ST_ILLCOND = 128      /* fp32 pair above the conditioning threshold that the
                                 fp64 re-solve could not take (capacity exceeded)    */
};

/* Device-resident prepared GreensSet (reference PreparedGreens,
 * solver.cpp:113-121, plus the per-frequency tables the fused kernels read). */
typedef struct gtd_greens {
    int n, m, h, hp;      /* grid, padded grid 2n, R2C width n+1, padded pitch */
    int fp64;             /* 1: tables are double, 0: float                    */
    void* fk;             /* [m][hp] complex: baseline kernel spectrum (C7)    */
    void* gtab;           /* [(n+1)][hp] real: alpha multiplier g(du,dv) (C6)   */
    void* k1;             /* [m] complex: 1-D spectrum of the centred die box  */
    void* tw;             /* [m] complex: exp(-2 pi i t/m)                     */
    void* hs;             /* [m] complex: exp(-i pi t/m) (half-step twiddles)    */
    void* fg;             /* [m][hp] {fk.re, fk.im, alpha g(du,v), D(u)D(v)}: one vector load per frequency */
    double alpha, beta, rand_scale, mu_fixed;
    void* fgm;            /* [m][hp][4] fixed-mu table {F_det, fk} (k_fgm)                     */
    int det_flags;        /* GTD_ST_RUNAWAY_DET if den1 at mu_fixed fails check_denominator  */
} gtd_greens;

/* Inputs of a Monte-Carlo batch: p_leak0 = nom_scale * N * V, applied = P + p_leak0.
 * Sample strides are in elements (0 broadcasts one map to every sample). */
typedef struct gtd_mc_in {
    const void* P;
    const void* N;
    const void* V;
    long long sP, sN, sV;
    double nom_scale;
} gtd_mc_in;

/* fp64 re-solve of ill-conditioned fp32 pairs ("fp32 with fp64 residual check"):
 * after the fp32 passes, pairs whose max 1/|den2|^2 (random_greens denominator,
 * greens.cpp:243-247) exceeds `thr` are gathered (up to `cap`), solved again by
 * the fp64 passes with a device-side count, and their maps / stats replace the
 * fp32 ones. All buffers are device memory owned by the caller. */
typedef struct gtd_mc_resolve {
    const struct gtd_greens* g64; /* fp64 tables of the same GreensSet          */
    void* in64;                   /* [cap][3][n][n] double: P, N, V              */
    void* out64;                  /* [cap][n][n] double                          */
    gtd_sample_stats* stats64;    /* [cap]                                       */
    void* scratch64;              /* cap * gtd_mc_scratch_bytes_per_sample(n, 1) */
    int* sel;                     /* [1 + cap]: count, then sample indices       */
    int cap;
    float thr;
} gtd_mc_resolve;

/* Options of the Monte-Carlo batch (mode A = reference run_one semantics). */
typedef struct gtd_mc_opts {
    int mu_per_sample;  /* 1: closed forms use the sample mean leakage; 0: gs.mu */
    int with_rand;      /* 0 drops the shift-variant term (ablation); 2 outputs the
                           shift-variant map f_rand o p_var * rand_scale alone (no
                           deterministic part, no clamp: the config-2 fixed point's term) */
    double exponent_cap;/* |ln var| guard (variation.cpp:173-178)               */
    const gtd_mc_resolve* resolve; /* fp32 only: NULL = no fp64 re-solve        */
} gtd_mc_opts;

/* Optional profiling hook: called on the host between launches with the
 * point index (0 before pass 1, 1 after pass 1, 2 after pass 2, 3 after pass 3)
 * so the caller can record CUDA events on the same stream. */
typedef void (*gtd_mark_fn)(void* ctx, int point, cudaStream_t st);

/* Scratch bytes needed per in-flight sample by gtd_mc_batch. */
size_t gtd_mc_scratch_bytes_per_sample(int n, int fp64);

/* Mode-A batch. Maps are [B][n][n] (float or double per g->fp64).
 * out: [B][n][n] rise maps or NULL. stats: [B] device array. scratch holds
 * `chunk` samples (gtd_mc_scratch_bytes_per_sample each). Returns a CUDA
 * error code (0 = launched). */
int gtd_mc_batch(const gtd_greens* g, const gtd_mc_in* in, int batch,
                 const gtd_mc_opts* opts, void* out, gtd_sample_stats* stats, void* scratch,
                 int chunk, cudaStream_t stream, gtd_mark_fn mark, void* ctx);

/* Number of kernel launches gtd_mc_batch issues for a given batch/chunk
 * (resolve: 1 if the fp64 re-solve is attached). */
int gtd_mc_launch_count(int batch, int chunk);
int gtd_mc_resolve_launch_count(void);

#ifdef __cplusplus
}
#endif

#ifdef __cplusplus
extern "C" {
#endif
/* Padded R2C width of the fused passes (n+1 rounded to the column tile). */
int gtd_padded_width(int n, int fp64);
/* Batched in-place 2-D complex FFT of [batch][m][m] (sign -1 forward,
 * +1 inverse without 1/m^2); tw = m complex twiddles of the same precision. */
int gtd_fft2d(void* data, int m, int batch, int sign, int fp64, const void* tw, cudaStream_t st);
/* Fixed-mu column-pass table from the full fp64 fk in work_d (after gtd_greens_tables);
 * mub = mu * beta; *flag_d = 1 if den1 fails the runaway check. */
int gtd_greens_fgm(const void* work_d, const double* g_sp0_d, int n, int hp, int fp64, double alpha, double mub,
                   void* fgm_out, int* flag_d, cudaStream_t st);
/* GreensSet device tables from fp64 f_sp0 / g_sp0 (device n x n maps). */
int gtd_greens_tables(const double* f_sp0_d, const double* g_sp0_d, double phi, int n, int hp,
                      int fp64, const void* tw64_d, void* work_d, void* fk_out, void* gtab_out, void* fg_out,
                      double alpha, cudaStream_t st);
#ifdef __cplusplus
}
#endif

/* ---- fp64 full-spectrum kernels of the reference-API solves (ops.cu) ---- */
#ifdef __cplusplus
extern "C" {
#endif
int gtd_mirror_pad(const double* a, const double* b, int n, void* X, cudaStream_t st);
int gtd_fdet_full(const void* fk, const double* gtab, int n, int hp, double alpha, double beta, double mu,
                  void* Fd, int* flag, cudaStream_t st);
int gtd_transient(const void* fk, const double* gtab, const void* Fd, int n, int hp, double alpha, double cap,
                  double fk_floor, double t, void* out, double dt, int kwin, void* r, void* rk, int* flag,
                  cudaStream_t st);
int gtd_spec_mul(void* X, const void* S, size_t count, cudaStream_t st);
int gtd_crop(const void* X, int n, double scale, double* out, cudaStream_t st);
int gtd_trace_step(const void* dlt, const void* dk, const void* r, const void* rk, const void* F, void* E,
                   void* Pacc, void* X, size_t count, cudaStream_t st);
int gtd_saturation(const void* F, const void* r, size_t count, int k, double re_sum_F, double* part, int blocks,
                   double* sat, cudaStream_t st);
int gtd_trace_scale(const double* totals, const double* sat, int steps, int k, double* scale, cudaStream_t st);
int gtd_add_rand(double* T, const double* a, const double* b, const double* scale, double scale_mul, size_t nn,
                 int maps, cudaStream_t st);
int gtd_reduce(const double* x, size_t count, double* out3, cudaStream_t st);   /* sum, min, max */
int gtd_creduce(const void* x, size_t count, double* out3, cudaStream_t st);   /* Re sum, Im sum, max|.| */
int gtd_clamp(double* x, size_t count, unsigned long long* neg, cudaStream_t st);
#ifdef __cplusplus
}
#endif

/* ---- mode B: leakage fixed point with the Kirchhoff transform (fixed_point.cu) ---- */
#ifdef __cplusplus
extern "C" {
#endif
typedef struct gtd_fp_opts {
    int law;          /* 1: exp(beta dT) (north star), 0: 1 + beta dT (reference leakage_at_temperature) */
    int kirchhoff;    /* 1: T(theta) inverse for k = k_ref (T/T0)^-eta */
    double beta, t_ambient, eta, tol;
    int max_iters;
    int poll;         /* host convergence poll interval in iterations (0 = 4) */
    int warm_start;   /* 1: t_state holds T_0 on entry (else T_0 = 0)                 */
    const void* H;    /* optional [B][n][n] shift-variant maps h = f_rand o p_var * rand_scale:
                         theta += h * sum(applied) each iteration (combined config 2)      */
    long long sH;     /* sample stride of H in elements                                    */
    int accel;        /* 0: Picard (reference outer loop); k0 > 0: Chebyshev semi-iteration
                         from iteration k0 on, rho from the residual ratio there              */
    void* Tprev;      /* [B][n][n] x_{k-1} state of the acceleration (required if accel)   */
    void* Yout;       /* [B][n][n] G(x_k) of the last iteration: the result (required if accel) */
    void* lm_state;   /* accel = -m < 0: Anderson(m <= 4) mixing on the 16 x 16 lowest cosine modes
                         (fp_lowmode); [B] x gtd_fp_lowmode_bytes() of state, and lm_cos a
                         [16][n] double table cos(pi p (x + 1/2) / n) (gtd_fp_lowmode_cos)      */
    const double* lm_cos;
    int lm_keep;      /* 1: lm_state continues a previous stage's history (no re-initialisation) */
    int min_iters;    /* the stop rule may fire from this iteration on (0 = 2: the reference
                         loop tests convergence after iteration 1, fdm.cpp:190-200); 1 for the
                         fp64 stage that continues an fp32 iteration: its first evaluation is
                         the fp64 residual check of the fp32 iterate                           */
} gtd_fp_opts;
size_t gtd_fp_lowmode_bytes(void);
int gtd_fp_lowmode_cos(int n, double* table, cudaStream_t st);
/* fp32 <-> fp64 copies of device maps (fp64 finish stage of an fp32 fixed point). */
int gtd_widen(const float* src, double* dst, size_t count, cudaStream_t st);
int gtd_narrow(const double* src, float* dst, size_t count, cudaStream_t st);
/* iters = it32 + it64, status = st64 | NOCONVERGE if it32 + it64 > max_iters (both [batch]). */
int gtd_fp_combine(int* iters, int* status, const int* it64, const int* st64, int batch, int max_iters,
                   cudaStream_t st);
/* status[i] |= stats[i].status (mode-A status of the shift-variant maps). */
int gtd_fp_or_status(int* status, const gtd_sample_stats* stats, int batch, cudaStream_t st);
size_t gtd_fp_scratch_bytes_per_sample(int n, int fp64);

/* ---- config 4: large-grid mode B by four-step passes (large.cu), fp64.
 * m = M1 * M2 (gtd_lg_split); rows phase on `pairs` die-row pairs of a slab,
 * columns phase on half-spectrum columns [c0, c0 + hc) of all rows. */
typedef struct gtd_lg {
    int n, m, M1, M2;
    const void* tw; /* [m] double2 exp(-2 pi i t / m) */
    const void* fk; /* [m][fkp] double2 baseline kernel half spectrum */
    int fkp;
    const void* hs; /* [m] double2 exp(-i pi t / m) (half steps; NULL: four-step row passes) */
} gtd_lg;
int gtd_lg_split(int m, int* M1, int* M2);
/* row-phase output layout: 1 = real DCT rows At [rows][n + 1] (n <= 8192, one-pass row kernels;
 * the column phase reads columns c0.. of every row), 0 = packed row-pair spectra Z [pairs][m] */
int gtd_lg_row_layout(const gtd_lg* g);
/* Low-mode Anderson mixing on this rank's rows [rows][hy] of the row buffer (die rows row0 ..):
 * project -> coef[256] (partial: [gtd_lg_lowmode_partial_blocks(rows)][256] scratch), all-reduce
 * coef over the ranks, mix (state: gtd_lg_lowmode_state_bytes(), depth <= 4) -> corr[256], apply. */
size_t gtd_lg_lowmode_state_bytes(void);
int gtd_lg_lowmode_partial_blocks(int rows);
int gtd_lg_lowmode_init(void* state, cudaStream_t st);
int gtd_lg_lowmode_project(const gtd_lg* g, const void* y, int hy, int rows, int row0, double* partial, double* coef,
                           cudaStream_t st);
int gtd_lg_lowmode_mix(void* state, const double* coef, int depth, double res_prev, double* corr, cudaStream_t st);
int gtd_lg_lowmode_apply(const gtd_lg* g, void* y, int hy, int rows, int row0, const double* corr, cudaStream_t st);

/* applied rows [2 pairs][n] -> Z [pairs][m] (mirrored rows' spectra, two rows per line) */
int gtd_lg_rows_fwd(const gtd_lg* g, const double* app, int pairs, void* S1, void* Z, cudaStream_t st);
/* Z (all pairs) -> Y [n][hc] = rows [0,n) of IFFT_col(fk . FFT_col(mirror(A))) for columns c0..c0+hc.
 * compact = 0: Z is [n/2][m]; 1: Z is [n/2][2 hc] = (Z_p[c0 + c], Z_p[(m - c0 - c) mod m]) per column c. */
int gtd_lg_cols(const gtd_lg* g, const void* Z, int compact, int c0, int hc, void* C1, void* C2, void* Y,
                cudaStream_t st);
/* The column phase over peer memory (multi-GPU without all-to-all copies): Zr / Yr are DEVICE
 * arrays of one mapped pointer per rank (Zr[r]: rank r's [P][m] row spectra, Yr[r]: its
 * [2P][hy] row buffer); the columns [c0, c0+hc) are read from every rank's Z in place and the
 * results stored into every rank's Y rows directly. */
int gtd_lg_cols_peer(const gtd_lg* g, const void* const* Zr, int pairs_per_rank, int c0, int hc, void* C1, void* C2,
                     void* const* Yr, int hy, cudaStream_t st);
/* Y [2 pairs][hy] (all columns 0..n of the slab's rows) -> theta -> T (Tst), residual (max bits),
 * status bits, next applied rows. Q / G (may be NULL): x_{k-1} in / x_k out, G(x_k) out; omega > 0
 * stores the Chebyshev step x_{k+1} = omega (gamma G + (1 - gamma) x_k - x_{k-1}) + x_{k-1}. */
int gtd_lg_rows_inv(const gtd_lg* g, const void* Y, int hy, int pairs, void* S1, double* Tst, double* app,
                    const double* P, const double* L0, const gtd_fp_opts* o, unsigned long long* res_bits,
                    int* status, double* Q, double* G, double omega, double gamma, cudaStream_t st);

/* fk = FFT2(center_kernel(f_sp0 - phi)) + phi m^2/4 at DC, [m][fkp] (g->fk unused);
 * S1, Z: (n/2) x m complex scratch; C1: m x fkp complex scratch. */
int gtd_lg_kernel_spectrum(const gtd_lg* g, const double* f_sp0, double phi, void* S1, void* Z, void* C1,
                           void* fk_out, cudaStream_t st);

/* ---- FDM network oracle (fdm.cu): the reference 3-layer network, Jacobi-PCG. fp64. */
typedef struct gtd_fdm {
    int n;
    double pitch, t_die, t_tim, t_spr, k_tim, k_spr;
    double c_die, c_tim, c_spr; /* node heat capacities (J/K) */
    double g_sink;              /* per spreader cell (W/K) */
    double inv_dt;              /* 1/dt for backward Euler, 0 steady */
    const double* kd;           /* [n*n] effective die conductivity */
} gtd_fdm;
int gtd_fdm_kcell(const double* k_map, const double* rise, double c, int n, double* kd, int* flag, cudaStream_t st);
int gtd_fdm_diag(const gtd_fdm* f, double* diag, cudaStream_t st);
int gtd_fdm_spmv(const gtd_fdm* f, const double* diag, const double* x, double* y, const double* w, double* dot,
                 cudaStream_t st);
/* CG scalars sc[8]: 0 r.z, 1 r.r, 2 b.b, 3 p.Ap, 4 r.r (new), 5 r.z (new) */
int gtd_cg_init(int N, const double* b, const double* ax, const double* diag, double* r, double* z, double* p,
                double* sc, cudaStream_t st);
int gtd_cg_step(const gtd_fdm* f, const double* diag, double* x, double* r, double* z, double* p, double* q,
                double* sc, cudaStream_t st);
int gtd_cg_direction(int N, const double* z, double* p, double* sc, cudaStream_t st);
int gtd_fdm_rhs(const double* p_dyn, const double* leak, int temp_dep, double beta, const double* x, double c_die,
                double c_tim, double c_spr, double inv_dt, int nn, double* b, cudaStream_t st);
int gtd_absdiff(const double* a, const double* b, size_t count, double* out, cudaStream_t st);

/* ---- seeded variation maps on the device (vargen.cu), m = 128 / 256 / 512 */
int gtd_var_pitch(int n);
size_t gtd_var_scratch_bytes_per_sample(int n, int fp64);
/* sqrt(lambda) [m][var_pitch] (device precision) of the spherical correlogram with `range`
 * (same length unit as pitch), normalised to unit variance. work_d: m*m double2,
 * lam_d: m*m double, red_d: 3 doubles. */
int gtd_var_model(const gtd_greens* g, const void* tw64, double pitch, double range, void* work_d, double* lam_d,
                  double* red_d, void* sqlam_out, cudaStream_t st);
/* var[b] = 1 + sigma z_b, z_b the field of seeds[b] (device array); scratch per sample as above */
int gtd_var_generate(const gtd_greens* g, const void* sqlam, const unsigned long long* seeds, int batch,
                     double sigma, void* var, void* scratch, int chunk, cudaStream_t st);

/* ---- config-3 batched transient traces (trace_batch.cu) */
typedef struct gtd_trace_in {
    const int* blk;
    long long blk_stride; /* elements between traces' block maps (0: shared) */
    const void* sched;    /* [B][steps][nblk] per-cell watts, device precision */
    int nblk, steps;
    const void* leak0;    /* [B][n*n] leakage base L0 (device precision) */
    long long leak_stride;
} gtd_trace_in;
typedef struct gtd_trace_opts {
    int window; /* k >= 1 */
    int law;
    double beta;
    int out_stride;
} gtd_trace_opts;
int gtd_trace_pitch(int n, int fp64);
size_t gtd_trace_bytes_per_trace(int n, int fp64, int window);
size_t gtd_trace_table_bytes(int n, int fp64);
/* tab = {(1 - r) F, r, r^(k+1) F} half width, from fp64 full (m x m) F_det, r, r^(k+1). */
int gtd_trace_tables(const gtd_greens* g, const void* Fd, const void* r, const void* rk, void* tab, cudaStream_t st);
int gtd_trace_batch(const gtd_greens* g, const void* tab, const gtd_trace_in* in, int batch, const gtd_trace_opts* o,
                    void* t_out, double* max_out, void* scratch, int chunk, cudaStream_t st, long long* launches);
size_t gtd_fp_state_bytes(void);
/* t_state: [B][n][n] rise maps (state and result); iters/status: [B] device ints;
 * max_out/mean_out: [B] device doubles (may be NULL); state: B * gtd_fp_state_bytes();
 * counter_d: device int; counter_h: pinned host int. Synchronises the stream every
 * `poll` iterations to stop when every sample of a chunk is done. */
int gtd_fp_batch(const gtd_greens* g, const gtd_mc_in* in, int batch, const gtd_fp_opts* opts, void* t_state,
                 int* iters, int* status, double* max_out, double* mean_out, void* scratch, void* state,
                 int* counter_d, int* counter_h, int chunk, cudaStream_t stream, long long* launches);
#ifdef __cplusplus
}
#endif

/* ---- calibration: modal kernel producer and variation / closed-form maps (calib.cu, variation.cu) ---- */
#ifdef __cplusplus
extern "C" {
#endif
typedef struct gtd_stack {  /* reference ChipStack (stack.hpp:17-26) */
    int n;
    double die_edge, t_die, k_die, c_die, t_tim, k_tim, c_tim, t_spr, k_spr, c_spr, ambient, sink_resistance;
} gtd_stack;
/* f_sp0 (n x n fp64, device) of a uniform-k die by the modal DCT-II solution; work: 3 n^2 doubles. */
int gtd_modal_impulse(const gtd_stack* s, double k_die, double* work, double* out, cudaStream_t st);
/* centre values f_sp0(c,c) for up to 64 die conductivities; d_nets: count * gtd_modal_net_bytes(). */
int gtd_modal_center(const gtd_stack* s, const double* k_values, int count, double* d_nets, double* out,
                     cudaStream_t st);
size_t gtd_modal_net_bytes(void);
/* backward-Euler centre-cell step response after steps_d[i] (cumulative) steps of dt. */
int gtd_modal_transient(const gtd_stack* s, double k_die, double dt, const int* steps_d, int ntimes,
                        double* part, int blocks, double* out, cudaStream_t st);
/* fit_capacitance centre-cell model for capacitance `cap` (<= 16 times). */
int gtd_cap_model(const void* fk_full, size_t count, double floor_abs, double cap, const double* times_d,
                  int ntimes, double inv_m2, double* part, int blocks, double* out, cudaStream_t st);

/* variation.cu */
/* sqrt(lambda * fix) of the spherical-correlogram circulant embedding (variation.cpp:87-132). */
int gtd_var_eigs(int n, double pitch, double range, int fp64_twiddles_dummy, const void* tw64, void* work_cplx,
                 double* sqrt_lam, double* red3, cudaStream_t st);
/* out[n][n] = sigma * Re(IFFT(sqrt_lam . FFT(noise)))[top-left]; noise: m*m doubles; work: m*m double2. */
int gtd_var_shape(const double* noise, const double* sqrt_lam, int n, double sigma, const void* tw64, void* work,
                  double* out, cudaStream_t st);
/* expo = bl * dl + bt * dt; flag |= 1 if |expo| > cap; out = nominal * exp(expo) (or exp only if nominal NULL). */
int gtd_leak_exp(const double* nominal, const double* dl, const double* dt, double bl, double bt, double cap, int n,
                 double* out, int* flag, cudaStream_t st);
int gtd_add_maps(const double* a, const double* b, size_t count, double* out, cudaStream_t st);
int gtd_sub_scalar(const double* a, double s, size_t count, double* out, cudaStream_t st);
/* K = centre_kernel(f - phi) (spectral.cpp:126-141) as complex; out: m*m double2. */
int gtd_center_kernel(const double* f, double phi, int n, void* K, cudaStream_t st);
/* kernel_to_die (spectral.cpp:150-165) with scale: out[x][y] = scale * Re K[(x-c) mod m][(y-c) mod m]. */
int gtd_kernel_to_die(const void* K, int n, double scale, double* out, cudaStream_t st);
/* q(du, dv) = 1/4 sum f(clamp(c+-du), clamp(c+-dv)) + shift, table [(n+1)][n+1] (symmetric_multiplier). */
int gtd_sym_table(const double* f, int n, double shift, double* tab, cudaStream_t st);
/* random_greens spectral algebra (greens.cpp:225-251) over the full m x m spectrum, in place on Fp (= F(p_var)):
 * Fp <- F_det (beta fk q + alpha Fp g) / (1 - alpha (1 + F(mu) + Fp) g - mu beta fk - beta fk q). */
int gtd_rand_spectrum(const void* Fd, const void* fk, const double* gtab, int hp, const double* qtab, int n,
                      double alpha, double beta, double mu, void* Fp, int* flag, cudaStream_t st);
#ifdef __cplusplus
}
#endif
