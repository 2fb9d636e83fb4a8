// oracle/restate.cpp — TEST INFRASTRUCTURE ONLY (see restate.h).
//
// Batch drivers over the UNCHANGED reference core (mode A) and the fp64 CPU
// restatement of the north-star fixed point (mode B), built by oracle/Makefile
// into oracle/_ref/libgt_restate.so. Only tests/, __graft_entry__.smoke() and
// bench.py's CPU legs load this library.
#include "restate.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <thread>
#include <vector>

#include "errors.hpp"
#include "fdm.hpp"
#include "field.hpp"
#include "greens.hpp"
#include "solver.hpp"
#include "spectral.hpp"
#include "stack.hpp"
#include "variation.hpp"

using namespace gtherm;

namespace {

int status_class(const Error& e) {
    if (dynamic_cast<const ConfigError*>(&e)) return 2;
    if (dynamic_cast<const ValidationError*>(&e)) return 4;
    if (dynamic_cast<const ConvergenceError*>(&e) || dynamic_cast<const RunawayError*>(&e) ||
        dynamic_cast<const CalibrationError*>(&e))
        return 3;
    return 5;
}

FieldMap to_field(const double* src, int n, double pitch, Unit u) {
    FieldMap f(n, pitch, u);
    if (src) std::copy(src, src + static_cast<size_t>(n) * n, f.values().begin());
    return f;
}

GreensSet to_greens(const ref_greens* g) {
    GreensSet gs;
    gs.n = g->n;
    gs.pitch = g->pitch;
    gs.f_sp0 = to_field(g->f_sp0, g->n, g->pitch, Unit::KelvinPerWatt);
    gs.g_sp0 = to_field(g->g_sp0, g->n, g->pitch, Unit::KelvinPerWatt);
    gs.f_det = to_field(g->f_det, g->n, g->pitch, Unit::KelvinPerWatt);
    gs.f_rand = to_field(g->f_rand, g->n, g->pitch, Unit::KelvinPerWatt);
    gs.p_var = to_field(g->p_var, g->n, g->pitch, Unit::Watts);
    gs.phi = g->phi;
    gs.kappa_inf = g->kappa_inf;
    gs.alpha = g->alpha;
    gs.beta = g->beta;
    gs.mu = g->mu;
    gs.capacitance = g->capacitance;
    gs.rand_scale = g->rand_scale;
    return gs;
}

template <typename Fn>
void pool(int count, int jobs, Fn&& fn) {
    jobs = std::max(1, jobs);
    if (jobs == 1) {
        for (int i = 0; i < count; ++i) fn(i);
        return;
    }
    std::atomic<int> next{0};
    std::vector<std::thread> th;
    for (int w = 0; w < jobs; ++w)
        th.emplace_back([&] {
            for (int i = next.fetch_add(1); i < count; i = next.fetch_add(1)) fn(i);
        });
    for (auto& t : th) t.join();
}

// crop(IFFT(spec . FFT(mirror_pad(p)))) — PreparedGreens::convolve_det
// (solver.cpp:123-127) with an explicit spectrum.
FieldMap convolve_with(const std::vector<cplx>& spec, const FieldMap& p) {
    const int n = p.n(), m = 2 * n;
    FieldMap padded = mirror_pad(p);
    std::vector<cplx> buf(padded.values().begin(), padded.values().end());
    buf = fft2(buf, m);
    for (size_t k = 0; k < buf.size(); ++k) buf[k] *= spec[k];
    std::vector<cplx> sp = ifft2(buf, m);
    FieldMap out(n, p.pitch(), Unit::Kelvin);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) out(i, j) = sp[static_cast<size_t>(i) * m + j].real();
    return out;
}

}  // namespace

extern "C" {

double ref_mc_batch(const ref_greens* g, const double* p_dyn, const double* var, int batch, double leak_frac,
                    int mu_per_sample, double beta_l, int with_rand, int jobs, double* t_out, double* max_out,
                    double* mean_out, int* status_out) {
    const auto t0 = std::chrono::steady_clock::now();
    const GreensSet gs = to_greens(g);
    const int n = gs.n;
    const size_t nn = static_cast<size_t>(n) * n;
    // Seed-invariant spectrum, as monte_carlo hoists it (solver.cpp:350-351).
    std::vector<cplx> fdet_fixed;
    if (!mu_per_sample) {
        try {
            fdet_fixed = deterministic_spectrum(gs.f_sp0, gs.phi, gs.g_sp0, gs.alpha, gs.beta, gs.mu);
        } catch (const Error& e) {  // the whole reference call fails (solver.cpp:350-351)
            for (int i = 0; i < batch; ++i)
                if (status_out) status_out[i] = status_class(e);
            return 0.0;
        }
    }
    const FieldMap zero(n, gs.pitch, Unit::Dimensionless);
    pool(batch, jobs, [&](int i) {
        int st = 0;
        try {
            const FieldMap P = to_field(p_dyn + i * nn, n, gs.pitch, Unit::Watts);
            FieldMap nominal = P;
            for (double& x : nominal.values()) x *= leak_frac;
            FieldMap dl(n, gs.pitch, Unit::Dimensionless);
            for (size_t k = 0; k < nn; ++k) dl.values()[k] = std::log(var[i * nn + k]) / beta_l;
            // d_tox = 0: p_leak0 = nominal * exp(beta_L * ln(var)/beta_L) = nominal * var.
            LeakageBaseline leak = leakage_baseline(nominal, dl, zero, beta_l, -5.0, gs.beta);
            const double mu = mu_per_sample ? leak.mu : gs.mu;
            std::vector<cplx> fdet = mu_per_sample
                                         ? deterministic_spectrum(gs.f_sp0, gs.phi, gs.g_sp0, gs.alpha, gs.beta, mu)
                                         : fdet_fixed;
            FieldMap applied = P + leak.p_leak0;
            FieldMap t_map = convolve_with(fdet, applied);
            if (with_rand) {
                FieldMap f_rand = random_greens(fdet, gs.f_sp0, gs.phi, gs.g_sp0, leak.p_var, gs.alpha, gs.beta, mu);
                t_map += hadamard(f_rand, leak.p_var) * (applied.sum() * gs.rand_scale);
            }
            for (double& x : t_map.values()) x = std::max(x, 0.0);
            if (t_out) std::copy(t_map.values().begin(), t_map.values().end(), t_out + i * nn);
            if (max_out) max_out[i] = t_map.max();
            if (mean_out) mean_out[i] = t_map.mean();
        } catch (const Error& e) {
            st = status_class(e);
        } catch (const std::exception&) {
            st = 5;
        }
        if (status_out) status_out[i] = st;
    });
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int ref_greens_save_dir(const ref_greens* g, const char* dir) {
    try {
        GreensSet gs = to_greens(g);
        save_greens(gs, CalibrationReport{}, dir);
        return 0;
    } catch (const Error& e) {
        return status_class(e);
    } catch (const std::exception&) {
        return 5;
    }
}

int ref_impulse_response(int n, double die_edge, double k_die, double* out) {
    try {
        ChipStack s;
        s.n = n;
        s.die_edge = die_edge;
        s.layers[0].conductivity = k_die;
        VariationParams v;
        v.dopant_spread = 0.0;
        ConductivityMap km = conductivity_map(k_die, v, n, s.pitch());
        FieldMap f = impulse_response(s, km);
        std::copy(f.values().begin(), f.values().end(), out);
        return 0;
    } catch (const Error& e) {
        return status_class(e);
    }
}

int ref_calibrate(int n, double die_edge, double beta, double dopant_spread, double leak_total,
                  int fit_rand_scale, int fit_transient, ref_greens* out) {
    try {
        ChipStack s;
        s.n = n;
        s.die_edge = die_edge;
        VariationParams v;
        v.beta = beta;
        v.dopant_spread = dopant_spread;
        FieldMap leak(n, s.pitch(), Unit::Watts, leak_total / (static_cast<double>(n) * n));
        CalibrateOptions o;
        o.fit_rand_scale = fit_rand_scale != 0;
        o.fit_transient = fit_transient != 0;
        Calibration cal = calibrate(s, v, leak, o);
        const GreensSet& gs = cal.gs;
        const size_t nn = static_cast<size_t>(n) * n;
        auto put = [&](const FieldMap& f, const double* dst) {
            std::copy(f.values().begin(), f.values().begin() + nn, const_cast<double*>(dst));
        };
        put(gs.f_sp0, out->f_sp0);
        put(gs.g_sp0, out->g_sp0);
        put(gs.f_det, out->f_det);
        put(gs.f_rand, out->f_rand);
        put(gs.p_var, out->p_var);
        out->n = n;
        out->pitch = gs.pitch;
        out->phi = gs.phi;
        out->kappa_inf = gs.kappa_inf;
        out->alpha = gs.alpha;
        out->beta = gs.beta;
        out->mu = gs.mu;
        out->capacitance = gs.capacitance;
        out->rand_scale = gs.rand_scale;
        return 0;
    } catch (const Error& e) {
        return status_class(e);
    }
}

// with_rand: the combined config-2 loop -- each iteration adds the reference's
// shift-variant Hadamard term hadamard(f_rand, p_var) * (sum(applied) * rand_scale)
// (solver.cpp:169-174, 364-365) to the convolution before the Kirchhoff inverse, with
// f_rand = random_greens at gs.mu (greens.cpp:225-251; F_det hoisted as monte_carlo,
// solver.cpp:350-351) from the sample's own leakage baseline (variation.cpp:162-195;
// p_leak0 = leak_frac P var as ref_mc_batch builds it), computed once per sample.
static double fixed_point_impl(const ref_greens* g, const double* p_dyn, const double* var, int batch,
                               double leak_frac, double beta, int law, int kirchhoff, double t_ambient, double eta,
                               double tol, int max_iters, int jobs, double* t_out, int* iters_out, int* status_out,
                               int with_rand) {
    const auto t0 = std::chrono::steady_clock::now();
    const GreensSet gs = to_greens(g);
    const int n = gs.n;
    const size_t nn = static_cast<size_t>(n) * n;
    const std::vector<cplx> fk = baseline_kernel_spectrum(gs.f_sp0, gs.phi);
    std::vector<cplx> fdet;
    if (with_rand) {
        try {
            fdet = deterministic_spectrum(gs.f_sp0, gs.phi, gs.g_sp0, gs.alpha, gs.beta, gs.mu);
        } catch (const Error& e) {
            for (int i = 0; i < batch; ++i)
                if (status_out) status_out[i] = status_class(e);
            return 0.0;
        }
    }
    const FieldMap zero(n, gs.pitch, Unit::Dimensionless);
    const double beta_l = -10.0;
    // Kirchhoff inverse for k = k_ref (T/T0)^-eta (k normalised at ambient):
    // T = [T0^(1-eta) + (1-eta)(theta-T0) T0^-eta]^(1/(1-eta)).
    const double a = std::pow(t_ambient, 1.0 - eta), b = (1.0 - eta) * std::pow(t_ambient, -eta);
    pool(batch, jobs, [&](int i) {
        int st = 0, it_done = 0;
        FieldMap rise(n, gs.pitch, Unit::Kelvin);
        try {
            const FieldMap P = to_field(p_dyn + i * nn, n, gs.pitch, Unit::Watts);
            FieldMap l0 = P;
            FieldMap hmap;  // hadamard(f_rand, p_var) when with_rand
            if (with_rand) {
                FieldMap nominal = P;
                for (double& x : nominal.values()) x *= leak_frac;
                FieldMap dl(n, gs.pitch, Unit::Dimensionless);
                for (size_t k = 0; k < nn; ++k) dl.values()[k] = std::log(var[i * nn + k]) / beta_l;
                LeakageBaseline leak = leakage_baseline(nominal, dl, zero, beta_l, -5.0, gs.beta);
                l0 = leak.p_leak0;
                FieldMap f_rand = random_greens(fdet, gs.f_sp0, gs.phi, gs.g_sp0, leak.p_var, gs.alpha, gs.beta, gs.mu);
                hmap = hadamard(f_rand, leak.p_var);
            } else {
                for (size_t k = 0; k < nn; ++k) l0.values()[k] *= leak_frac * var[i * nn + k];
            }
            for (int it = 1; it <= max_iters; ++it) {
                FieldMap applied = P;
                for (size_t k = 0; k < nn; ++k) {
                    const double dt = rise.values()[k];
                    const double f = law == 0 ? 1.0 + beta * dt : std::exp(beta * dt);
                    applied.values()[k] += l0.values()[k] * f;
                }
                FieldMap theta = convolve_with(fk, applied);
                if (with_rand) theta += hmap * (applied.sum() * gs.rand_scale);
                double delta = 0.0;
                for (size_t k = 0; k < nn; ++k) {
                    double t = theta.values()[k];
                    if (kirchhoff) {
                        const double br = a + b * t;
                        if (!(br > 0.0)) throw ValidationError("oracle", "Kirchhoff inverse outside validity");
                        t = std::pow(br, 1.0 / (1.0 - eta)) - t_ambient;
                    }
                    if (!std::isfinite(t)) throw ValidationError("oracle", "non-finite temperature (runaway)");
                    delta = std::max(delta, std::abs(t - rise.values()[k]));
                    theta.values()[k] = t;
                }
                rise = theta;
                it_done = it;
                if (it > 1 && delta < tol) break;
                if (it == max_iters) throw ConvergenceError("oracle", "fixed-point loop hit max_iters");
            }
        } catch (const Error& e) {
            st = status_class(e);
        }
        if (t_out) std::copy(rise.values().begin(), rise.values().end(), t_out + i * nn);
        if (iters_out) iters_out[i] = it_done;
        if (status_out) status_out[i] = st;
    });
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

double ref_fixed_point_batch(const ref_greens* g, const double* p_dyn, const double* var, int batch,
                             double leak_frac, double beta, int law, int kirchhoff, double t_ambient, double eta,
                             double tol, int max_iters, int jobs, double* t_out, int* iters_out, int* status_out) {
    return fixed_point_impl(g, p_dyn, var, batch, leak_frac, beta, law, kirchhoff, t_ambient, eta, tol, max_iters,
                            jobs, t_out, iters_out, status_out, 0);
}

double ref_fixed_point_rand_batch(const ref_greens* g, const double* p_dyn, const double* var, int batch,
                                  double leak_frac, double beta, int law, int kirchhoff, double t_ambient, double eta,
                                  double tol, int max_iters, int jobs, double* t_out, int* iters_out,
                                  int* status_out) {
    return fixed_point_impl(g, p_dyn, var, batch, leak_frac, beta, law, kirchhoff, t_ambient, eta, tol, max_iters,
                            jobs, t_out, iters_out, status_out, 1);
}

double ref_trace_leak_batch(const ref_greens* g, const int* blk, long long blk_stride, const double* sched,
                            int nblk, const double* leak0, long long leak_stride, int batch, double dt, int steps,
                            int window, int law, double beta, int out_stride, int jobs, double* t_out,
                            int* status_out) {
    const auto t0 = std::chrono::steady_clock::now();
    const GreensSet gs = to_greens(g);
    const int n = gs.n;
    const size_t nn = static_cast<size_t>(n) * n;
    const int frames = steps / out_stride;
    pool(batch, jobs, [&](int b) {
        int st = 0;
        try {
            const PreparedGreens pg(gs);
            const int* bm = blk + b * blk_stride;
            const double* l0 = leak0 + b * leak_stride;
            PowerTrace tr;
            tr.dt = dt;
            std::vector<double> rise(nn, 0.0);
            const FieldMap no_var;  // p_var of another shape: shift-variant term off
            ProfileOptions opt;
            opt.with_rand = false;
            for (int s = 1; s <= steps; ++s) {
                FieldMap P(n, gs.pitch, Unit::Watts);
                const double* sc = sched + (static_cast<size_t>(b) * steps + (s - 1)) * nblk;
                for (size_t k = 0; k < nn; ++k) {
                    const double f = law == 0 ? 1.0 + beta * rise[k] : std::exp(beta * rise[k]);
                    P.values()[k] = sc[bm[k]] + l0[k] * f;
                }
                tr.frames.push_back(std::move(P));
                const ThermalResult res = time_varying_profile(pg, tr, window, no_var, opt);
                const FieldMap& last = res.rise.back();
                std::copy(last.values().begin(), last.values().end(), rise.begin());
                if (s % out_stride == 0 && t_out)
                    std::copy(rise.begin(), rise.end(), t_out + (static_cast<size_t>(b) * frames + s / out_stride - 1) * nn);
            }
        } catch (const Error& e) {
            st = status_class(e);
        }
        if (status_out) status_out[b] = st;
    });
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // extern "C"
