/* oracle/restate.h — TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py's
 * cpu_baseline / --impl reference legs). Never linked into the product.
 *
 * extern "C" entry points over the UNCHANGED reference core (compiled from
 * /root/reference/proj/src/core by oracle/Makefile) for the batch shapes the
 * reference C ABI cannot express, plus fp64 CPU restatements of the
 * north-star parts the reference lacks. Each function cites the reference
 * code it drives or restates.
 */
#ifndef GT_ORACLE_RESTATE_H
#define GT_ORACLE_RESTATE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ref_greens {
    int n;
    double pitch, phi, kappa_inf, alpha, beta, mu, capacitance, rand_scale;
    const double* f_sp0; /* n*n */
    const double* g_sp0; /* n*n */
    const double* f_det; /* n*n or NULL */
    const double* f_rand;
    const double* p_var;
} ref_greens;

/* Mode A: the reference monte_carlo run_one (solver.cpp:353-374) per
 * (p_dyn, var) pair, with p_leak0 from leakage_baseline(leak_frac*p_dyn,
 * d_length = ln(var)/beta_L, d_tox = 0) (variation.cpp:162-195).
 * mu_per_sample = 1 evaluates deterministic_spectrum / random_greens at the
 * sample's mean leakage, 0 at g->mu (the reference monte_carlo choice).
 * Runs a std::thread pool of `jobs` workers like solver.cpp:376-387.
 * status_out[i]: 0 ok, else the gt_status class of the reference exception.
 * Returns wall seconds. */
double ref_mc_batch(const ref_greens* g, const double* p_dyn, const double* var, int batch,
                    double leak_frac, int mu_per_sample, double beta_l, int with_rand, int jobs,
                    double* t_out, double* max_out, double* mean_out, int* status_out);

/* Writes a GreensSet directory with the reference's own save_greens
 * (greens.cpp:464-517); f_det/f_rand/p_var default to zero maps. */
int ref_greens_save_dir(const ref_greens* g, const char* dir);

/* Reference impulse_response (fdm.cpp:288-296) for the default stack with the
 * given n / die_edge and uniform die conductivity k_die: n*n K/W map. */
int ref_impulse_response(int n, double die_edge, double k_die, double* out);

/* The reference's own calibrate() (greens.cpp:346-446) on the default stack
 * with n / die_edge overridden, a uniform nominal leakage of leak_total W, the
 * variation defaults except beta and dopant_spread (0 -> uniform die k, the
 * case the modal kernel reproduces exactly). out->f_* must point at n*n
 * buffers; scalars are filled in. fit_transient / fit_rand_scale as in
 * CalibrateOptions (greens.hpp:138-145). */
int ref_calibrate(int n, double die_edge, double beta, double dopant_spread, double leak_total,
                  int fit_rand_scale, int fit_transient, ref_greens* out);

/* Mode B restatement (north star (4)): per sample the FDM outer loop of
 * fdm.cpp:167-205 with the CG solve replaced by the Green convolution of the
 * baseline kernel spectrum (greens.cpp:194-201) on the mirror-padded torus:
 *   theta_{k+1} - T0 = crop(IFFT(fk . FFT(mirror(P + P_leak(T_k)))))
 *   P_leak(T) = leak_frac*P*var * (law==0 ? 1 + beta dT : exp(beta dT))
 *   T(theta) = Kirchhoff inverse for k = k0 (T/300)^-eta when kirchhoff != 0
 * stop when max|T_{k+1} - T_k| < tol after iteration 1 (fdm.cpp:190-195);
 * max_iters -> status 3 (ConvergenceError). iters_out receives K_ref. */
double ref_fixed_point_batch(const ref_greens* g, const double* p_dyn, const double* var, int batch,
                             double leak_frac, double beta, int law, int kirchhoff, double t_ambient,
                             double eta, double tol, int max_iters, int jobs, double* t_out,
                             int* iters_out, int* status_out);

/* Combined config 2 (north star (3) + (4)): ref_fixed_point_batch with the
 * reference's shift-variant term in every iteration,
 *   theta = conv(fk, applied) + hadamard(f_rand, p_var) * sum(applied) * rand_scale,
 * f_rand = random_greens at gs.mu from the sample's leakage baseline (once per sample). */
double ref_fixed_point_rand_batch(const ref_greens* g, const double* p_dyn, const double* var, int batch,
                                  double leak_frac, double beta, int law, int kirchhoff, double t_ambient,
                                  double eta, double tol, int max_iters, int jobs, double* t_out,
                                  int* iters_out, int* status_out);

/* Config 3 (north star (5) + (4)): batched power traces with the leakage
 * update every step, driven through the reference's own windowed superposition
 * time_varying_profile (solver.cpp:212-287, with_rand off), one step at a time:
 *   P_n = P_dyn,n + leak0 o f(T_{n-1}), T_0 = 0, f = 1 + beta dT (law 0,
 *   leakage_at_temperature, variation.cpp:213-222) or exp(beta dT) (law 1);
 *   T_n = last map of time_varying_profile(P_1..P_n, window)  (clamped >= 0)
 * P_dyn,n(x,y) = sched[b][n-1][blk[b][x][y]]; blk/leak0 stride 0 = shared.
 * T_n is stored every out_stride steps into t_out[b][frame]. Returns seconds. */
double ref_trace_leak_batch(const ref_greens* g, const int* blk, long long blk_stride, const double* sched,
                            int nblk, const double* leak0, long long leak_stride, int batch, double dt, int steps,
                            int window, int law, double beta, int out_stride, int jobs, double* t_out,
                            int* status_out);

#ifdef __cplusplus
}
#endif

#endif
