// gt_ops.cpp — host orchestration of the reference-API solves on the device.
//
// gt_solve_steady  -> steady_profile   (reference solver.cpp:158-179)
// gt_solve_step    -> step_response    (solver.cpp:181-210)
// gt_solve_trace   -> time_varying_profile (solver.cpp:212-287), with the
//                     O(steps * k * m^2) window sum replaced by the exact
//                     per-mode recursion of SURVEY §8a D10.
// All arithmetic runs in fp64 kernels (ops.cu, fft2d.cu); the host validates
// inputs, sequences launches and reads back results and scalars.
#include "gt_ops.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>

#include "devctx.hpp"

using namespace gth;

namespace {

using wall = std::chrono::steady_clock;
double ms_since(wall::time_point t0) { return std::chrono::duration<double, std::milli>(wall::now() - t0).count(); }

int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

// check_power (solver.cpp:63-70)
void check_power(const Field& p, int n, const char* what) {
    if (p.n != n) fail(ST_CONFIG, "solver", std::string(what) + ": power map does not match the GreensSet grid");
    p.check_finite(what);
    if (p.min() < 0.0) fail(ST_CONFIG, "solver", std::string(what) + ": powers must be >= 0");
}

// Device working set of one reference-API solve (fp64, full m x m spectra).
struct Solve {
    std::unique_ptr<gt_device_greens> d;
    int n, m;
    size_t mm, nn;
    cudaStream_t st;
    DBuf Fd, X, flag, red, fr, pv, rnd_scale, cnt, P, T, P0, Sp;  // the last four: per-call working maps
    double fk_max = 0.0, re_sum_F = 0.0;
    bool rand_uploaded = false;  // f_rand / p_var of the (immutable) GreensSet are on the device

    explicit Solve(const Greens& g) {
        g.validate();
        d = prepare_device(g, GT_FP64, current_device());
        n = g.n;
        m = 2 * n;
        mm = static_cast<size_t>(m) * m;
        nn = static_cast<size_t>(n) * n;
        st = d->stream;
        Fd.ensure(mm * 16);
        X.ensure(mm * 16);
        flag.ensure(sizeof(int) * 4);
        red.ensure(sizeof(double) * 8);
        cuda_ok(cudaMemsetAsync(flag.p, 0, sizeof(int) * 4, st), "memset");
        // PreparedGreens: F_det at the GreensSet mu (solver.cpp:113-121)
        cuda_ok(gtd_fdet_full(d->fk_full.p, d->gtab.as<double>(), n, d->d.hp, g.alpha, g.beta, g.mu, Fd.p,
                              flag.as<int>(), st),
                "fdet");
        if (read_flag() & GTD_ST_RUNAWAY_DET)
            fail(ST_SOLVER, "greens",
                 "deterministic_greens: spectral denominator collapsed below 1e-6 (leakage feedback gain reached unity)");
        double r3[3];
        creduce(d->fk_full.p, mm, r3);
        fk_max = r3[2];
        creduce(Fd.p, mm, r3);
        re_sum_F = r3[0];
    }

    int read_flag() {
        int f = 0;
        cuda_ok(cudaMemcpyAsync(&f, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st), "d2h");
        cuda_ok(cudaStreamSynchronize(st), "sync");
        cuda_ok(cudaMemsetAsync(flag.p, 0, sizeof(int), st), "memset");
        return f;
    }
    void reduce(const double* x, size_t count, double* out3) {
        cuda_ok(gtd_reduce(x, count, red.as<double>(), st), "reduce");
        cuda_ok(cudaMemcpyAsync(out3, red.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, st), "d2h");
        cuda_ok(cudaStreamSynchronize(st), "sync");
    }
    void creduce(const void* x, size_t count, double* out3) {
        cuda_ok(gtd_creduce(x, count, red.as<double>(), st), "creduce");
        cuda_ok(cudaMemcpyAsync(out3, red.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, st), "d2h");
        cuda_ok(cudaStreamSynchronize(st), "sync");
    }
    // X = FFT(mirror_pad(a - b)) on the given buffer
    void padded_fft(const double* a, const double* b, void* out) {
        cuda_ok(gtd_mirror_pad(a, b, n, out, st), "mirror");
        cuda_ok(gtd_fft2d(out, m, 1, -1, 1, d->tw64.p, st), "fft");
    }
    // out = crop(IFFT(in)) / m^2   (destroys in)
    void inverse_crop(void* in, double* out) {
        cuda_ok(gtd_fft2d(in, m, 1, +1, 1, d->tw64.p, st), "ifft");
        cuda_ok(gtd_crop(in, n, 1.0 / (double(m) * double(m)), out, st), "crop");
    }
    void upload_rand(const Greens& g) {
        if (rand_uploaded) return;
        upload(fr, g.f_rand.v.data(), nn * 8, st);
        upload(pv, g.p_var.v.data(), nn * 8, st);
        rand_uploaded = true;
    }
    // clamp_negatives over `maps` maps with one shared peak (solver.cpp:33-46)
    void clamp(double* T, size_t count, double peak, double tol, double vmin) {
        const double floor = -tol * std::max(peak, 0.0);
        if (vmin < floor) {
            char b[96];
            std::snprintf(b, sizeof b, "%f", vmin);
            fail(ST_VALIDATION, "solver", std::string("negative temperature rise beyond tolerance: ") + b + " K");
        }
        cnt.ensure(8);
        cuda_ok(cudaMemsetAsync(cnt.p, 0, 8, st), "memset");
        cuda_ok(gtd_clamp(T, count, static_cast<unsigned long long*>(cnt.p), st), "clamp");
    }
};

Field download(const double* src, int n, double pitch, cudaStream_t st) {
    Field f(n, pitch, Unit::Kelvin);
    cuda_ok(cudaMemcpyAsync(f.v.data(), src, f.v.size() * 8, cudaMemcpyDeviceToHost, st), "d2h");
    cuda_ok(cudaStreamSynchronize(st), "sync");
    return f;
}

}  // namespace

struct GtSolveCache {
    int device;
    Solve s;
    GtSolveCache(const Greens& g, int dev) : device(dev), s(g) {}
};

namespace {
// The handle's prepared set on the current device (built on first use; rebuilt if the
// caller moved to another device). The caller holds slot.mu.
Solve& prepared(const Greens& g, GtSolveSlot& slot) {
    const int dev = current_device();
    if (!slot.cache || slot.cache->device != dev) {
        slot.cache.reset();
        slot.cache = std::make_shared<GtSolveCache>(g, dev);
    }
    return slot.cache->s;
}
}  // namespace

void gt_ops_check_trace(double dt, const std::vector<Field>& frames) {
    // reference solver.cpp:74-83
    if (frames.empty()) fail(ST_CONFIG, "solver", "power trace is empty");
    if (!(dt > 0.0)) fail(ST_CONFIG, "solver", "power trace dt must be positive");
    for (const Field& f : frames) {
        if (!f.same_shape(frames.front())) fail(ST_CONFIG, "solver", "power trace frames differ in shape");
        f.check_finite("trace frame");
        if (f.min() < 0.0) fail(ST_CONFIG, "solver", "trace powers must be >= 0");
    }
}

Field gt_ops_steady(const Greens& g, GtSolveSlot& slot, const Field& p_dyn, bool with_rand, double* online_ms) {
    need_device();
    std::lock_guard<std::mutex> lk(slot.mu);
    Solve& S = prepared(g, slot);
    auto t0 = wall::now();
    check_power(p_dyn, g.n, "steady_profile");
    DBuf& P = S.P;
    DBuf& T = S.T;
    upload(P, p_dyn.v.data(), S.nn * 8, S.st);
    T.ensure(S.nn * 8);
    S.padded_fft(P.as<double>(), nullptr, S.X.p);
    cuda_ok(gtd_spec_mul(S.X.p, S.Fd.p, S.mm, S.st), "mul");
    S.inverse_crop(S.X.p, T.as<double>());
    double tol = 1e-9;
    if (with_rand) {
        double r3[3];
        S.reduce(P.as<double>(), S.nn, r3);  // sum p_dyn (field.cpp:45-57)
        S.upload_rand(g);
        S.rnd_scale.ensure(8);
        const double sc = r3[0] * g.rand_scale;
        cuda_ok(cudaMemcpyAsync(S.rnd_scale.p, &sc, 8, cudaMemcpyHostToDevice, S.st), "h2d");
        cuda_ok(gtd_add_rand(T.as<double>(), S.fr.as<double>(), S.pv.as<double>(), S.rnd_scale.as<double>(), 1.0,
                             S.nn, 1, S.st),
                "rand");
        tol = 0.02;
    }
    double r3[3];
    S.reduce(T.as<double>(), S.nn, r3);
    S.clamp(T.as<double>(), S.nn, r3[2], tol, r3[1]);
    Field out = download(T.as<double>(), g.n, g.pitch, S.st);
    if (online_ms) *online_ms = ms_since(t0);
    return out;
}

std::vector<Field> gt_ops_step(const Greens& g, GtSolveSlot& slot, const Field& p_dyn,
                               const std::vector<double>& times, bool with_rand, double* online_ms) {
    need_device();
    std::lock_guard<std::mutex> lk(slot.mu);
    Solve& S = prepared(g, slot);
    auto t0 = wall::now();
    check_power(p_dyn, g.n, "step_response");
    for (double t : times)
        if (t < 0.0) fail(ST_CONFIG, "solver", "step_response: negative time");
    DBuf &P = S.P, &P0 = S.P0, &Sp = S.Sp, &T = S.T;
    upload(P, p_dyn.v.data(), S.nn * 8, S.st);
    P0.ensure(S.mm * 16);
    Sp.ensure(S.mm * 16);
    T.ensure(S.nn * 8);
    S.padded_fft(P.as<double>(), nullptr, P0.p);
    double r3[3];
    S.reduce(P.as<double>(), S.nn, r3);
    const double total = r3[0];
    if (with_rand) S.upload_rand(g);
    S.rnd_scale.ensure(8);
    std::vector<Field> out;
    for (double t : times) {
        if (t > 0.0 && !(g.capacitance > 0.0)) fail(ST_SOLVER, "solver", "GreensSet has no fitted capacitance");
        // transient_spectrum(t) (solver.cpp:129-149)
        cuda_ok(gtd_transient(S.d->fk_full.p, S.d->gtab.as<double>(), S.Fd.p, g.n, S.d->d.hp, g.alpha, g.capacitance,
                              1e-6 * S.fk_max, t, Sp.p, 0.0, 0, nullptr, nullptr, S.flag.as<int>(), S.st),
                "transient");
        if (t > 0.0 && (S.read_flag() & 1))
            fail(ST_SOLVER, "solver", "non-positive transient time constant");
        cuda_ok(cudaMemcpyAsync(S.X.p, P0.p, S.mm * 16, cudaMemcpyDeviceToDevice, S.st), "copy");
        cuda_ok(gtd_spec_mul(S.X.p, Sp.p, S.mm, S.st), "mul");
        S.inverse_crop(S.X.p, T.as<double>());
        double tol = 0.01;
        if (with_rand && t > 0.0) {
            double c3[3];
            S.creduce(Sp.p, S.mm, c3);
            const double sat = c3[0] / S.re_sum_F;  // saturation (solver.cpp:151-156)
            const double sc = total * g.rand_scale * sat;
            cuda_ok(cudaMemcpyAsync(S.rnd_scale.p, &sc, 8, cudaMemcpyHostToDevice, S.st), "h2d");
            cuda_ok(gtd_add_rand(T.as<double>(), S.fr.as<double>(), S.pv.as<double>(), S.rnd_scale.as<double>(), 1.0,
                                 S.nn, 1, S.st),
                    "rand");
            tol = 0.02;
        }
        S.reduce(T.as<double>(), S.nn, r3);
        S.clamp(T.as<double>(), S.nn, r3[2], tol, r3[1]);
        out.push_back(download(T.as<double>(), g.n, g.pitch, S.st));
    }
    if (online_ms) *online_ms = ms_since(t0);
    return out;
}

std::vector<Field> gt_ops_trace(const Greens& g, GtSolveSlot& slot, double dt, const std::vector<Field>& frames,
                                int window, bool with_rand, std::vector<double>* times, double* online_ms) {
    need_device();
    std::lock_guard<std::mutex> lk(slot.mu);
    Solve& S = prepared(g, slot);
    auto t0 = wall::now();
    gt_ops_check_trace(dt, frames);
    if (frames.front().n != g.n) fail(ST_CONFIG, "solver", "trace frames do not match the GreensSet grid");
    int k = window > 0 ? window : static_cast<int>(std::ceil(0.005 / dt));
    k = std::max(1, k);
    const int steps = static_cast<int>(frames.size());
    k = std::min(k, steps);
    if (!(g.capacitance > 0.0)) fail(ST_SOLVER, "solver", "GreensSet has no fitted capacitance");

    // per-mode r = exp(-dt/tau), r^(k+1); saturation fractions sat_i, i = 1..k
    DBuf r, rk, E, Pacc, dl, dk, part, sat, F, tot, scl, raw;
    r.ensure(S.mm * 16);
    rk.ensure(S.mm * 16);
    cuda_ok(gtd_transient(S.d->fk_full.p, S.d->gtab.as<double>(), S.Fd.p, g.n, S.d->d.hp, g.alpha, g.capacitance,
                          1e-6 * S.fk_max, 0.0, nullptr, dt, k, r.p, rk.p, S.flag.as<int>(), S.st),
            "transient");
    if (S.read_flag() & 1) fail(ST_SOLVER, "solver", "non-positive transient time constant");
    const int blocks = 148;
    part.ensure(sizeof(double) * blocks * k);
    sat.ensure(sizeof(double) * k);
    cuda_ok(gtd_saturation(S.Fd.p, r.p, S.mm, k, S.re_sum_F, part.as<double>(), blocks, sat.as<double>(), S.st),
            "saturation");

    // frames on the device, totals (compensated sums, field.cpp:45-57)
    F.ensure(S.nn * 8 * steps);
    std::vector<double> totals(steps);
    for (int j = 0; j < steps; ++j) {
        cuda_ok(cudaMemcpyAsync(F.as<double>() + j * S.nn, frames[j].v.data(), S.nn * 8, cudaMemcpyHostToDevice, S.st),
                "h2d");
        double r3[3];
        S.reduce(F.as<double>() + j * S.nn, S.nn, r3);
        totals[j] = r3[0];
    }
    upload(tot, totals.data(), totals.size() * 8, S.st);
    scl.ensure(sizeof(double) * steps);
    cuda_ok(gtd_trace_scale(tot.as<double>(), sat.as<double>(), steps, k, scl.as<double>(), S.st), "scale");

    E.ensure(S.mm * 16);
    Pacc.ensure(S.mm * 16);
    dl.ensure(S.mm * 16);
    dk.ensure(S.mm * 16);
    raw.ensure(S.nn * 8 * steps);
    cuda_ok(cudaMemsetAsync(E.p, 0, S.mm * 16, S.st), "memset");
    cuda_ok(cudaMemsetAsync(Pacc.p, 0, S.mm * 16, S.st), "memset");
    const double* fr = F.as<double>();
    for (int nstep = 1; nstep <= steps; ++nstep) {
        // Delta_n = FFT(mirror(P_n - P_{n-1})) (linearity of the padded transform)
        const double* cur = fr + (nstep - 1) * S.nn;
        const double* prev = nstep >= 2 ? fr + (nstep - 2) * S.nn : nullptr;
        S.padded_fft(cur, prev, dl.p);
        const void* dkp = nullptr;
        if (nstep > k) {
            const int j = nstep - k;  // Delta_{n-k}
            S.padded_fft(fr + (j - 1) * S.nn, j >= 2 ? fr + (j - 2) * S.nn : nullptr, dk.p);
            dkp = dk.p;
        }
        cuda_ok(gtd_trace_step(dl.p, dkp, r.p, rk.p, S.Fd.p, E.p, Pacc.p, S.X.p, S.mm, S.st), "recursion");
        S.inverse_crop(S.X.p, raw.as<double>() + (nstep - 1) * S.nn);
    }
    if (with_rand) {
        S.upload_rand(g);
        cuda_ok(gtd_add_rand(raw.as<double>(), S.fr.as<double>(), S.pv.as<double>(), scl.as<double>(), g.rand_scale,
                             S.nn, steps, S.st),
                "rand");
    }
    double r3[3];
    S.reduce(raw.as<double>(), S.nn * steps, r3);
    S.clamp(raw.as<double>(), S.nn * steps, r3[2], 0.02, r3[1]);
    std::vector<Field> out;
    out.reserve(steps);
    times->clear();
    for (int j = 0; j < steps; ++j) {
        out.push_back(download(raw.as<double>() + j * S.nn, g.n, g.pitch, S.st));
        times->push_back((j + 1) * dt);
    }
    if (online_ms) *online_ms = ms_since(t0);
    return out;
}
