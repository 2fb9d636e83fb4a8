// calib_host.cpp — host orchestration of device calibration (gt_calibrate)
// and of the reference-API Monte Carlo (gt_monte_carlo).
//
// Random numbers: the reference draws its variation noise with std::mt19937_64
// and std::normal_distribution<double> (variation.cpp:87-147). Both are drawn
// here on the host with the same library calls and seeds (derived_seed,
// variation.cpp:68-85), so the device consumes bit-identical noise; every
// transform, exponent, reduction and closed form on that noise runs in fp64
// device kernels (variation.cu, calib.cu, fft2d.cu, mc_modeA.cu).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <random>
#include <thread>
#include <atomic>
#include <mutex>
#include <utility>

#include "devctx.hpp"
#include "gt_ops.h"

using namespace gth;

namespace {

using wall = std::chrono::steady_clock;

uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
// reference FieldPurpose (variation.hpp:33-39)
enum : uint64_t { GL_SYS = 0x11, GL_RAND = 0x12, OX_SYS = 0x21, OX_RAND = 0x22 };
uint64_t derived_seed(uint64_t base, uint64_t purpose, uint64_t run) {
    return splitmix64(base ^ (purpose << 32) ^ (run * 0x51ed2701ULL));
}

// Draw `count` normals exactly as the reference loops do.
void draw_normals(uint64_t seed, double sigma, size_t count, double* out) {
    std::mt19937_64 eng(seed);
    std::normal_distribution<double> gauss(0.0, sigma);
    for (size_t i = 0; i < count; ++i) out[i] = gauss(eng);
}

// Host noise of one leakage realisation (make_leakage_baseline, variation.cpp:197-211):
// systematic m^2 N(0,1) draws (x2) and random n^2 N(0, sigma_rand) draws (x2).
struct LeakNoise {
    std::vector<double> sys_l, rnd_l, sys_t, rnd_t;
};
LeakNoise leak_noise(const VarParams& v, int n, uint64_t base_seed, uint64_t run) {
    const size_t mm = static_cast<size_t>(2 * n) * (2 * n), nn = static_cast<size_t>(n) * n;
    LeakNoise z;
    if (v.sigma_sys != 0.0) {
        z.sys_l.resize(mm);
        z.sys_t.resize(mm);
        draw_normals(derived_seed(base_seed, GL_SYS, run), 1.0, mm, z.sys_l.data());
        draw_normals(derived_seed(base_seed, OX_SYS, run), 1.0, mm, z.sys_t.data());
    }
    if (v.sigma_rand != 0.0) {
        z.rnd_l.resize(nn);
        z.rnd_t.resize(nn);
        draw_normals(derived_seed(base_seed, GL_RAND, run), v.sigma_rand, nn, z.rnd_l.data());
        draw_normals(derived_seed(base_seed, OX_RAND, run), v.sigma_rand, nn, z.rnd_t.data());
    }
    return z;
}

// Device builder of d_length / d_tox maps from host noise.
struct VarDevice {
    int n, m;
    size_t nn, mm;
    double pitch;
    const void* tw64;
    cudaStream_t stream;
    DBuf sqrt_lam, work, noise, sys, red;
    VarDevice(gt_device_greens* dd, const VarParams& v, double pitch_)
        : VarDevice(dd->d.n, dd->tw64.p, dd->stream, v, pitch_) {}
    VarDevice(int n_, const void* tw64_, cudaStream_t st_, const VarParams& v, double pitch_)
        : n(n_), pitch(pitch_), tw64(tw64_), stream(st_) {
        m = 2 * n;
        nn = static_cast<size_t>(n) * n;
        mm = static_cast<size_t>(m) * m;
        work.ensure(mm * 16);
        red.ensure(64);
        if (v.sigma_sys != 0.0) {
            sqrt_lam.ensure(mm * 8);
            cuda_ok(gtd_var_eigs(n, pitch, v.corr_range * (n * pitch), 1, tw64, work.p, sqrt_lam.as<double>(),
                                 red.as<double>(), stream),
                    "variation eigenvalues");
        }
        noise.ensure(mm * 8);
        sys.ensure(nn * 8);
    }
    // out = sigma_sys * shaped(sys_noise) + rnd_noise (either part may be absent). With
    // sync = false the host noise buffers must stay alive until the stream reaches this work.
    void field(const VarParams& v, const std::vector<double>& sysn, const std::vector<double>& rndn, double* out,
               bool sync = true) {
        field(v, sysn.empty() ? nullptr : sysn.data(), rndn.empty() ? nullptr : rndn.data(), out, sync);
    }
    void field(const VarParams& v, const double* sysn, const double* rndn, double* out, bool sync) {
        cudaStream_t st = stream;
        cuda_ok(cudaMemsetAsync(out, 0, nn * 8, st), "memset");
        if (sysn) {
            cuda_ok(cudaMemcpyAsync(noise.p, sysn, mm * 8, cudaMemcpyHostToDevice, st), "h2d");
            cuda_ok(gtd_var_shape(noise.as<double>(), sqrt_lam.as<double>(), n, v.sigma_sys, tw64, work.p, out, st),
                    "shape");
        }
        if (rndn) {
            cuda_ok(cudaMemcpyAsync(sys.p, rndn, nn * 8, cudaMemcpyHostToDevice, st), "h2d");
            cuda_ok(gtd_add_maps(out, sys.as<double>(), nn, out, st), "add");
        }
        if (sync) cuda_ok(cudaStreamSynchronize(st), "sync");  // host noise buffers are reused by the caller
    }
};

// Pinned host slab for the Monte-Carlo noise ring (kept for the life of the process: a
// second gt_monte_carlo call does not pay the page-locking again).
struct PinnedSlab {
    double* p = nullptr;
    size_t cap = 0;
    void ensure(size_t doubles) {
        if (doubles <= cap) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        cuda_ok(cudaMallocHost(reinterpret_cast<void**>(&p), doubles * 8), "cudaMallocHost (noise ring)");
        cap = doubles;
    }
    ~PinnedSlab() {
        if (p) cudaFreeHost(p);
    }
};

// linearize_conductivity (variation.cpp:240-265): LSQ of k0 (T/300)^-eta on 313.15..373.15 K.
void linearize(double k0_300, double eta, double t_amb, double* k0_prime, double* c) {
    double sx = 0, sy = 0, sxx = 0, sxy = 0;
    int cnt = 0;
    for (double t = 313.15; t <= 373.15 + 1e-9; t += 1.0) {
        const double x = t - t_amb, y = k0_300 * std::pow(t / 300.0, -eta);
        sx += x;
        sy += y;
        sxx += x * x;
        sxy += x * y;
        ++cnt;
    }
    const double b = (cnt * sxy - sx * sy) / (cnt * sxx - sx * sx);
    const double a = (sy - b * sx) / cnt;
    *k0_prime = a;
    *c = -b / a;
}

gtd_stack to_dev(const Stack& s) {
    gtd_stack d{};
    d.n = s.n;
    d.die_edge = s.die_edge;
    d.t_die = s.die.thickness;
    d.k_die = s.die.conductivity;
    d.c_die = s.die.heat_capacity;
    d.t_tim = s.tim.thickness;
    d.k_tim = s.tim.conductivity;
    d.c_tim = s.tim.heat_capacity;
    d.t_spr = s.spreader.thickness;
    d.k_spr = s.spreader.conductivity;
    d.c_spr = s.spreader.heat_capacity;
    d.ambient = s.ambient;
    d.sink_resistance = s.sink_resistance;
    return d;
}

std::pair<int, int> farthest_corner(int n) {  // greens.cpp:41-54
    const int c = n / 2;
    std::pair<int, int> best{0, 0};
    double bd = -1.0;
    for (int i : {0, n - 1})
        for (int j : {0, n - 1}) {
            const double d = std::hypot(double(i - c), double(j - c));
            if (d > bd) {
                bd = d;
                best = {i, j};
            }
        }
    return best;
}

void d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    cuda_ok(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), "d2h");
    cuda_ok(cudaStreamSynchronize(st), "sync");
}

}  // namespace

// ============================================================ FDM oracle (fdm.cu)
// The reference's ThermalNetwork (fdm.cpp:22-296) on the device: per-cell die
// conductivity, Jacobi-preconditioned CG with Eigen's stopping rule
// (|r|^2 < tol^2 |b|^2, 40000 iterations), the steady outer fixed point and
// backward-Euler stepping with leakage refreshed every sub-step.
namespace {

enum : uint64_t { COND_PURPOSE = 0x31 };

std::vector<double> host_twiddles(int m) {
    std::vector<double> t(2 * static_cast<size_t>(m));
    for (int k = 0; k < m; ++k) {
        const double a = -2.0 * M_PI * static_cast<double>(k) / m;
        t[2 * k] = std::cos(a);
        t[2 * k + 1] = std::sin(a);
    }
    return t;
}

// conductivity_map (variation.cpp:224-238): i.i.d. clamped dopant spread per cell
std::vector<double> conductivity_map(double k_nominal, const VarParams& v, int n) {
    std::vector<double> k(static_cast<size_t>(n) * n, k_nominal);
    if (v.dopant_spread == 0.0) return k;
    std::mt19937_64 eng(derived_seed(v.seed, COND_PURPOSE, 0));
    std::normal_distribution<double> gauss(0.0, v.dopant_spread);
    for (double& x : k) x = k_nominal * (1.0 + std::clamp(gauss(eng), -v.cond_clamp, v.cond_clamp));
    return k;
}

struct FdmNet {
    Stack s;
    int n;
    size_t nn, N;
    cudaStream_t st = nullptr;
    DBuf kmap, kd, diag, x, xo, b, r, z, p, q, ax, sc, flag, red, tmp;
    double g_sink, c_die, c_tim, c_spr;

    FdmNet(const Stack& s_, const std::vector<double>& k_host) : s(s_), n(s_.n) {
        s.validate();
        nn = static_cast<size_t>(n) * n;
        N = 3 * nn;
        for (double k : k_host)
            if (!(k > 0.0)) fail(ST_CONFIG, "oracle", "non-positive die conductivity");
        cuda_ok(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
        upload(kmap, k_host.data(), nn * 8, st);
        for (DBuf* bu : {&kd}) bu->ensure(nn * 8);
        for (DBuf* bu : {&diag, &x, &xo, &b, &r, &z, &p, &q, &ax, &tmp}) bu->ensure(N * 8);
        sc.ensure(8 * 8);
        flag.ensure(8);
        red.ensure(64);
        const double area = s.pitch() * s.pitch();
        c_die = s.die.heat_capacity * area * s.die.thickness;
        c_tim = s.tim.heat_capacity * area * s.tim.thickness;
        c_spr = s.spreader.heat_capacity * area * s.spreader.thickness;
        // spreader half-thickness plus the cell's share of the lumped sink (fdm.cpp:38-42)
        const double r_half = s.spreader.thickness / (2.0 * s.spreader.conductivity * area);
        g_sink = 1.0 / (r_half + static_cast<double>(n) * n * s.sink_resistance);
        cuda_ok(cudaMemsetAsync(x.p, 0, N * 8, st), "memset");
    }
    ~FdmNet() {
        if (st) cudaStreamDestroy(st);
    }
    gtd_fdm net(double inv_dt) const {
        gtd_fdm f{};
        f.n = n;
        f.pitch = s.pitch();
        f.t_die = s.die.thickness;
        f.t_tim = s.tim.thickness;
        f.t_spr = s.spreader.thickness;
        f.k_tim = s.tim.conductivity;
        f.k_spr = s.spreader.conductivity;
        f.c_die = c_die;
        f.c_tim = c_tim;
        f.c_spr = c_spr;
        f.g_sink = g_sink;
        f.inv_dt = inv_dt;
        f.kd = kd.as<double>();
        return f;
    }
    // effective conductivity at the die rise (nullptr: k_map) and the operator diagonal
    void prepare(const double* rise, double cond_c, double inv_dt) {
        cuda_ok(cudaMemsetAsync(flag.p, 0, 8, st), "memset");
        cuda_ok(gtd_fdm_kcell(kmap.as<double>(), rise, cond_c, n, kd.as<double>(), flag.as<int>(), st), "kcell");
        int fl = 0;
        d2h(&fl, flag.p, 4, st);
        if (fl)
            fail(ST_VALIDATION, "oracle",
                 "die conductivity went non-positive; outside linearization validity");
        const gtd_fdm f = net(inv_dt);
        cuda_ok(gtd_fdm_diag(&f, diag.as<double>(), st), "diag");
    }
    // Eigen ConjugateGradient<..., DiagonalPreconditioner> on A x = b (fdm.cpp:120-146);
    // x holds the guess (zero when !guess) and the solution.
    void solve(double inv_dt, bool guess, double tol) {
        if (!guess) cuda_ok(cudaMemsetAsync(x.p, 0, N * 8, st), "memset");
        const gtd_fdm f = net(inv_dt);
        cuda_ok(gtd_fdm_spmv(&f, diag.as<double>(), x.as<double>(), ax.as<double>(), nullptr, nullptr, st), "spmv");
        cuda_ok(gtd_cg_init(static_cast<int>(N), b.as<double>(), ax.as<double>(), diag.as<double>(), r.as<double>(),
                            z.as<double>(), p.as<double>(), sc.as<double>(), st),
                "cg init");
        double h[8];
        d2h(h, sc.p, 64, st);
        const double rhs2 = h[2];
        if (rhs2 == 0.0) {
            cuda_ok(cudaMemsetAsync(x.p, 0, N * 8, st), "memset");
            return;
        }
        const double threshold = std::max(tol * tol * rhs2, std::numeric_limits<double>::min());
        if (h[1] < threshold) return;
        const int max_iters = 40000;
        int i = 0;
        double rr = h[1];
        for (; i < max_iters; ++i) {
            cuda_ok(gtd_cg_step(&f, diag.as<double>(), x.as<double>(), r.as<double>(), z.as<double>(), p.as<double>(),
                                q.as<double>(), sc.as<double>(), st),
                    "cg step");
            d2h(&rr, sc.as<double>() + 4, 8, st);
            if (rr < threshold) break;
            cuda_ok(gtd_cg_direction(static_cast<int>(N), z.as<double>(), p.as<double>(), sc.as<double>(), st),
                    "cg direction");
        }
        if (i == max_iters)
            fail(ST_SOLVER, "oracle", "conjugate gradient stalled, residual " + std::to_string(std::sqrt(rr / rhs2)));
    }
};

struct OracleSetup {
    Stack stack;
    VarParams var;
    std::vector<double> k_map;
    bool have_leak = false, temp_dep_leakage = false, temp_dep_cond = false;
    double cond_c = 0.0;
    std::vector<double> p_leak0;  // host copy
};

// oracle_setup (reference capi.cpp:265-284)
OracleSetup oracle_setup(const Stack& st, const VarParams* vp, const Field* nominal_leak, int tdl, int tdc) {
    OracleSetup s;
    s.stack = st;
    s.stack.validate();
    s.var = vp ? *vp : VarParams{};
    if (!vp) s.var.dopant_spread = 0.0;
    s.var.validate();
    const int n = s.stack.n;
    s.k_map = conductivity_map(s.stack.die.conductivity, s.var, n);
    if (nominal_leak) {
        if (nominal_leak->n != n) fail(ST_CONFIG, "oracle", "leakage map does not match the stack grid");
        if (nominal_leak->min() < 0.0) fail(ST_CONFIG, "variation", "leakage_baseline: nominal leakage must be >= 0");
        // make_leakage_baseline (variation.cpp:197-211), run 0
        need_device();
        const int m = 2 * n;
        const size_t nn = static_cast<size_t>(n) * n;
        cudaStream_t stx = nullptr;
        cuda_ok(cudaStreamCreateWithFlags(&stx, cudaStreamNonBlocking), "stream");
        DBuf tw, dl, dt, nom, pl, flag;
        const std::vector<double> twh = host_twiddles(m);
        upload(tw, twh.data(), twh.size() * 8, stx);
        dl.ensure(nn * 8);
        dt.ensure(nn * 8);
        pl.ensure(nn * 8);
        flag.ensure(8);
        {
            VarDevice vd(n, tw.p, stx, s.var, s.stack.pitch());
            LeakNoise z = leak_noise(s.var, n, s.var.seed, 0);
            vd.field(s.var, z.sys_l, z.rnd_l, dl.as<double>());
            vd.field(s.var, z.sys_t, z.rnd_t, dt.as<double>());
        }
        upload(nom, nominal_leak->v.data(), nn * 8, stx);
        cuda_ok(cudaMemsetAsync(flag.p, 0, 8, stx), "memset");
        cuda_ok(gtd_leak_exp(nom.as<double>(), dl.as<double>(), dt.as<double>(), s.var.beta_l, s.var.beta_tox,
                             s.var.exponent_cap, n, pl.as<double>(), flag.as<int>(), stx),
                "leakage exponent");
        int fl = 0;
        d2h(&fl, flag.p, 4, stx);
        if (fl) fail(ST_VALIDATION, "variation", "leakage exponent exceeds cap (unphysical variation inputs)");
        s.p_leak0.resize(nn);
        d2h(s.p_leak0.data(), pl.p, nn * 8, stx);
        cudaStreamDestroy(stx);
        s.have_leak = true;
        s.temp_dep_leakage = tdl != 0;
    }
    if (tdc) {
        double k0p = 0.0;
        s.temp_dep_cond = true;
        linearize(s.stack.die.conductivity, s.var.eta, s.stack.ambient, &k0p, &s.cond_c);
    }
    return s;
}

}  // namespace

Field gt_ops_oracle_steady(const Stack& stack, const VarParams* var, const Field& p_dyn, const Field* nominal_leak,
                           int temp_dep_leakage, int temp_dep_conductivity, int* outer_iterations);

// f_sp0 alone (impulse_response for 1 W at (c, c), fdm.cpp:288-296) by the modal
// solution, for any power-of-two n the device memory allows (config 4: 8192).
void gt_ops_modal_kernel(const Stack& s, double* out_host) {
    s.validate();
    need_device();
    const int n = s.n;
    if (!pow2(n) || n < 16 || n > 16384)
        fail(ST_CONFIG, "calibrate", "modal kernel supports power-of-two grids 16..16384, got n=" + std::to_string(n));
    const gtd_stack ds = to_dev(s);
    const size_t nn = static_cast<size_t>(n) * n;
    DBuf work, f;
    work.ensure(3 * nn * 8);
    f.ensure(nn * 8);
    cuda_ok(gtd_modal_impulse(&ds, s.die.conductivity, work.as<double>(), f.as<double>(), nullptr), "modal impulse");
    d2h(out_host, f.p, nn * 8, nullptr);
}

Greens gt_ops_calibrate_modal(const Stack& s, const VarParams& v, const Field* nominal_leak, double leak_total) {
    s.validate();
    v.validate();
    need_device();
    const int n = s.n;
    if (!pow2(n) || n < 16 || n > 1024)
        fail(ST_CONFIG, "calibrate", "device calibration supports power-of-two grids 16..1024, got n=" + std::to_string(n));
    // Uniform die conductivity: the modal DCT-II solution is the exact network response.
    // Per-cell conductivity (dopant spread): the device FDM network (fdm.cu), like the reference.
    const bool uniform_k = v.dopant_spread == 0.0;
    const double pitch = s.pitch();
    Field leak = nominal_leak ? *nominal_leak
                              : Field(n, pitch, Unit::Watts, (leak_total > 0.0 ? leak_total : 15.0) / (double(n) * n));
    if (leak.n != n) fail(ST_CONFIG, "greens", "nominal leakage map does not match the stack grid");
    if (leak.min() < 0.0) fail(ST_CONFIG, "variation", "leakage_baseline: nominal leakage must be >= 0");

    int dev = 0;
    cudaGetDevice(&dev);
    const gtd_stack ds = to_dev(s);
    const size_t nn = static_cast<size_t>(n) * n;
    const int m = 2 * n;
    const size_t mm = static_cast<size_t>(m) * m;

    // --- kernel producer: f_sp0 by the modal solution (replaces impulse_response, fdm.cpp:288-296)
    Greens g;
    g.n = n;
    g.pitch = pitch;
    double k0p_lin = 0.0, cslope = 0.0;
    const double k0p = s.die.conductivity;  // calibrate() uses the stack value as k0' (greens.cpp:355-357)
    linearize(k0p, v.eta, s.ambient, &k0p_lin, &cslope);
    const std::vector<double> k_map = conductivity_map(k0p, v, n);  // conductivity_map (variation.cpp:224-238)
    g.f_sp0 = Field(n, pitch, Unit::KelvinPerWatt);
    if (uniform_k) {
        cudaStream_t st = nullptr;
        DBuf work, f;
        work.ensure(3 * nn * 8);
        f.ensure(nn * 8);
        cuda_ok(gtd_modal_impulse(&ds, k0p, work.as<double>(), f.as<double>(), st), "modal impulse");
        d2h(g.f_sp0.v.data(), f.p, nn * 8, st);
    } else {
        // impulse_response (fdm.cpp:288-296): 1 W at (c, c), effects off, one linear solve
        FdmNet net(s, k_map);
        std::vector<double> bh(net.N, 0.0);
        bh[static_cast<size_t>(n / 2) * n + n / 2] = 1.0;
        upload(net.b, bh.data(), net.N * 8, net.st);
        net.prepare(nullptr, 0.0, 0.0);
        net.solve(0.0, false, 1e-9);
        d2h(g.f_sp0.v.data(), net.x.p, nn * 8, net.st);
    }
    // extract_baseline (greens.cpp:108-124): phi = outer-ring mean, kappa_inf = farthest corner
    {
        double ring = 0.0;
        int cnt = 0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                if (i == 0 || j == 0 || i == n - 1 || j == n - 1) {
                    ring += g.f_sp0.at(i, j);
                    ++cnt;
                }
        g.phi = ring / cnt;
        const auto [ci, cj] = farthest_corner(n);
        g.kappa_inf = g.f_sp0.at(ci, cj);
        g.g_sp0 = g.f_sp0;
        const double shift = g.f_sp0.at(n / 2, n / 2) - g.kappa_inf;  // make_g_shift (greens.cpp:170-175)
        for (double& x : g.g_sp0.v) x += shift;
    }
    // --- fit_alpha (greens.cpp:126-168) with modal centre responses
    {
        const double fr[7] = {0.75, 0.80, 0.85, 0.90, 0.95, 1.00, 1.05};
        double ks[7], peaks[7];
        for (int i = 0; i < 7; ++i) ks[i] = fr[i] * k0p;
        DBuf nets, out;
        nets.ensure(gtd_modal_net_bytes() * 7);
        out.ensure(7 * 8);
        cuda_ok(gtd_modal_center(&ds, ks, 7, nets.as<double>(), out.as<double>(), nullptr), "modal sweep");
        d2h(peaks, out.p, 7 * 8, nullptr);
        double sx = 0, sy = 0, sxx = 0, sxy = 0;
        for (int i = 0; i < 7; ++i) {
            const double x = ks[i] - k0p;
            sx += x;
            sy += peaks[i];
            sxx += x * x;
            sxy += x * peaks[i];
            g.sweep.emplace_back(ks[i], peaks[i]);
        }
        const double slope = (7 * sxy - sx * sy) / (7 * sxx - sx * sx), icpt = (sy - slope * sx) / 7;
        double ss_res = 0, ss_tot = 0;
        for (int i = 0; i < 7; ++i) {
            const double fit = icpt + slope * (ks[i] - k0p);
            ss_res += (peaks[i] - fit) * (peaks[i] - fit);
            ss_tot += (peaks[i] - sy / 7) * (peaks[i] - sy / 7);
        }
        g.fit_r2 = ss_tot > 0.0 ? 1.0 - ss_res / ss_tot : 0.0;
        if (g.fit_r2 < 0.95)
            fail(ST_SOLVER, "greens", "response-vs-conductivity fit r^2 = " + std::to_string(g.fit_r2) +
                                          " < 0.95; linearization invalid for this stack");
        g.c_prime = -slope / icpt;
        g.c = cslope;
        g.alpha = g.c_prime * cslope * k0p;
        g.rep_alpha = g.alpha;
    }
    g.beta = v.beta;
    // Device tables of the set so far (fk, g, twiddles) for the closed forms and the capacitance fit.
    g.f_det = Field(n, pitch, Unit::KelvinPerWatt);
    g.f_rand = Field(n, pitch, Unit::KelvinPerWatt);
    g.p_var = Field(n, pitch, Unit::Watts);
    auto d = prepare_device(g, GT_FP64, dev);
    cudaStream_t st = d->stream;

    // --- make_leakage_baseline (variation.cpp:197-211), run 0
    DBuf dl, dtox, nom, pl, pv, flag, red;
    dl.ensure(nn * 8);
    dtox.ensure(nn * 8);
    pl.ensure(nn * 8);
    pv.ensure(nn * 8);
    flag.ensure(8);
    red.ensure(64);
    {
        VarDevice vd(d.get(), v, pitch);
        LeakNoise z = leak_noise(v, n, v.seed, 0);
        vd.field(v, z.sys_l, z.rnd_l, dl.as<double>());
        vd.field(v, z.sys_t, z.rnd_t, dtox.as<double>());
    }
    upload(nom, leak.v.data(), nn * 8, st);
    cuda_ok(cudaMemsetAsync(flag.p, 0, 8, st), "memset");
    cuda_ok(gtd_leak_exp(nom.as<double>(), dl.as<double>(), dtox.as<double>(), v.beta_l, v.beta_tox, v.exponent_cap, n,
                         pl.as<double>(), flag.as<int>(), st),
            "leakage exponent");
    int fl = 0;
    d2h(&fl, flag.p, 4, st);
    if (fl) fail(ST_VALIDATION, "variation", "leakage exponent exceeds cap (unphysical variation inputs)");
    double r3[3];
    cuda_ok(gtd_reduce(pl.as<double>(), nn, red.as<double>(), st), "reduce");
    d2h(r3, red.p, 24, st);
    double mu = r3[0] / double(nn);
    cuda_ok(gtd_sub_scalar(pl.as<double>(), mu, nn, pv.as<double>(), st), "p_var");
    cuda_ok(gtd_reduce(pv.as<double>(), nn, red.as<double>(), st), "reduce");
    d2h(r3, red.p, 24, st);
    const double resid = r3[0] / double(nn);
    if (resid != 0.0) {  // re-centre once (variation.cpp:181-192)
        mu += resid;
        cuda_ok(gtd_sub_scalar(pl.as<double>(), mu, nn, pv.as<double>(), st), "p_var");
    }
    g.mu = mu;
    d2h(g.p_var.v.data(), pv.p, nn * 8, st);

    // --- deterministic and random closed forms (greens.cpp:203-251), fp64 full spectra
    {
        DBuf Fd, Fp, qtab;
        Fd.ensure(mm * 16);
        Fp.ensure(mm * 16);
        qtab.ensure(static_cast<size_t>(n + 1) * (n + 1) * 8);
        cuda_ok(cudaMemsetAsync(flag.p, 0, 8, st), "memset");
        cuda_ok(gtd_fdet_full(d->fk_full.p, d->gtab.as<double>(), n, d->d.hp, g.alpha, g.beta, g.mu, Fd.p,
                              flag.as<int>(), st),
                "fdet");
        d2h(&fl, flag.p, 4, st);
        if (fl)
            fail(ST_SOLVER, "greens",
                 "deterministic_greens: spectral denominator collapsed below 1e-6 (leakage feedback gain reached unity)");
        // f_det = kernel_to_die(ifft2(F_det))
        cuda_ok(cudaMemcpyAsync(Fp.p, Fd.p, mm * 16, cudaMemcpyDeviceToDevice, st), "copy");
        cuda_ok(gtd_fft2d(Fp.p, m, 1, +1, 1, d->tw64.p, st), "ifft");
        DBuf out;
        out.ensure(nn * 8);
        const double inv = 1.0 / (double(m) * double(m));
        cuda_ok(gtd_kernel_to_die(Fp.p, n, inv, out.as<double>(), st), "kernel_to_die");
        d2h(g.f_det.v.data(), out.p, nn * 8, st);
        // f_rand: F(p_var) = kernel_fft(p_var); q = sym(p_var + p_var(c,c) - p_var(far corner))
        cuda_ok(gtd_center_kernel(pv.as<double>(), 0.0, n, Fp.p, st), "centre");
        cuda_ok(gtd_fft2d(Fp.p, m, 1, -1, 1, d->tw64.p, st), "fft");
        const auto [fi, fj] = farthest_corner(n);
        const double qshift = g.p_var.at(n / 2, n / 2) - g.p_var.at(fi, fj);
        cuda_ok(gtd_sym_table(pv.as<double>(), n, qshift, qtab.as<double>(), st), "q");
        cuda_ok(gtd_rand_spectrum(Fd.p, d->fk_full.p, d->gtab.as<double>(), d->d.hp, qtab.as<double>(), n, g.alpha,
                                  g.beta, g.mu, Fp.p, flag.as<int>(), st),
                "random_greens");
        d2h(&fl, flag.p, 4, st);
        if (fl)
            fail(ST_SOLVER, "greens",
                 "random_greens: spectral denominator collapsed below 1e-6 (leakage feedback gain reached unity)");
        cuda_ok(gtd_fft2d(Fp.p, m, 1, +1, 1, d->tw64.p, st), "ifft");
        cuda_ok(gtd_kernel_to_die(Fp.p, n, inv, out.as<double>(), st), "kernel_to_die");
        d2h(g.f_rand.v.data(), out.p, nn * 8, st);

        // rand_scale (greens.cpp:390-421): regress the Hadamard term's gain against the FDM network
        // on a uniform 100 W probe with every effect on (leakage and conductivity feedback)
        Field probe(n, pitch, Unit::Watts, 100.0 / (double(n) * n));
        int its = 0;
        const Field oracle = gt_ops_oracle_steady(s, &v, probe, &leak, 1, 1, &its);
        Field applied = probe;
        for (size_t k = 0; k < nn; ++k) applied.v[k] += g.p_var.v[k] + mu;  // probe + p_leak0
        DBuf ap, tdet;
        upload(ap, applied.v.data(), nn * 8, st);
        tdet.ensure(nn * 8);
        cuda_ok(gtd_mirror_pad(ap.as<double>(), nullptr, n, Fp.p, st), "mirror");
        cuda_ok(gtd_fft2d(Fp.p, m, 1, -1, 1, d->tw64.p, st), "fft");
        cuda_ok(gtd_spec_mul(Fp.p, Fd.p, mm, st), "spec mul");
        cuda_ok(gtd_fft2d(Fp.p, m, 1, +1, 1, d->tw64.p, st), "ifft");
        cuda_ok(gtd_crop(Fp.p, n, inv, tdet.as<double>(), st), "crop");
        std::vector<double> td(nn);
        d2h(td.data(), tdet.p, nn * 8, st);
        const double total = applied.sum();
        double num = 0.0, den = 0.0;
        for (size_t k = 0; k < nn; ++k) {
            const double bk = g.f_rand.v[k] * g.p_var.v[k] * total;
            num += (oracle.v[k] - td[k]) * bk;
            den += bk * bk;
        }
        g.rand_scale = den > 0.0 ? std::clamp(num / den, 0.0, 500.0) : 1.0;
    }

    // --- fit_capacitance (greens.cpp:274-344) with the modal backward-Euler transient
    {
        const double tms[11] = {0.2, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 5.0, 6.0, 8.0, 10.0};
        double times[11];
        int steps[11];
        const double dt = 2e-5;
        double t = 0.0;
        int k = 0;
        for (int i = 0; i < 11; ++i) {
            times[i] = 1e-3 * tms[i];
            while (t + 0.5 * dt < times[i]) {  // fdm.cpp:271-276 stepping rule
                t += dt;
                ++k;
            }
            steps[i] = k;
        }
        DBuf dsteps, dtimes, part, outv;
        upload(dsteps, steps, sizeof steps, st);
        upload(dtimes, times, sizeof times, st);
        const int blocks = 148;
        part.ensure(sizeof(double) * blocks * 11);
        outv.ensure(sizeof(double) * 11);
        double target[11];
        if (uniform_k) {
            cuda_ok(gtd_modal_transient(&ds, k0p, dt, dsteps.as<int>(), 11, part.as<double>(), blocks,
                                        outv.as<double>(), st),
                    "modal transient");
            d2h(target, outv.p, sizeof target, st);
        } else {
            // transient_impulse (fdm.cpp:250-286) on the per-cell network: backward Euler at dt
            FdmNet net(s, k_map);
            net.prepare(nullptr, 0.0, 1.0 / dt);
            std::vector<double> ph(nn, 0.0);
            ph[static_cast<size_t>(n / 2) * n + n / 2] = 1.0;
            DBuf pd;
            upload(pd, ph.data(), nn * 8, net.st);
            int done = 0;
            for (int i = 0; i < 11; ++i) {
                for (; done < steps[i]; ++done) {
                    cuda_ok(cudaMemcpyAsync(net.xo.p, net.x.p, net.N * 8, cudaMemcpyDeviceToDevice, net.st), "copy");
                    cuda_ok(gtd_fdm_rhs(pd.as<double>(), nullptr, 0, 0.0, net.xo.as<double>(), net.c_die, net.c_tim,
                                        net.c_spr, 1.0 / dt, static_cast<int>(nn), net.b.as<double>(), net.st),
                            "rhs");
                    net.solve(1.0 / dt, true, 1e-9);
                }
                d2h(&target[i], net.x.as<double>() + static_cast<size_t>(n / 2) * n + n / 2, 8, net.st);
            }
        }
        double c3[3];
        cuda_ok(gtd_creduce(d->fk_full.p, mm, red.as<double>(), st), "creduce");
        d2h(c3, red.p, 24, st);
        const double floor_abs = 1e-6 * c3[2];
        const double inv_m2 = 1.0 / (double(m) * double(m));
        auto sse = [&](double cap) {
            double vals[11];
            cuda_ok(gtd_cap_model(d->fk_full.p, mm, floor_abs, cap, dtimes.as<double>(), 11, inv_m2, part.as<double>(),
                                  blocks, outv.as<double>(), st),
                    "cap model");
            d2h(vals, outv.p, sizeof vals, st);
            double e = 0.0;
            for (int i = 0; i < 11; ++i) e += (vals[i] - target[i]) * (vals[i] - target[i]);
            return e;
        };
        double lo = -8.0, hi = 0.0;
        const double gr = 0.5 * (std::sqrt(5.0) - 1.0);
        double a = hi - gr * (hi - lo), b = lo + gr * (hi - lo);
        double fa = sse(std::pow(10.0, a)), fb = sse(std::pow(10.0, b));
        for (int it = 0; it < 90; ++it) {
            if (fa < fb) {
                hi = b;
                b = a;
                fb = fa;
                a = hi - gr * (hi - lo);
                fa = sse(std::pow(10.0, a));
            } else {
                lo = a;
                a = b;
                fa = fb;
                b = lo + gr * (hi - lo);
                fb = sse(std::pow(10.0, b));
            }
        }
        g.capacitance = std::pow(10.0, 0.5 * (lo + hi));
        g.cap_residual = std::sqrt(sse(g.capacitance) / 11.0) / g.f_sp0.at(n / 2, n / 2);
        if (g.cap_residual > 0.10)
            fail(ST_SOLVER, "greens", "transient capacitance fit residual " + std::to_string(g.cap_residual) +
                                          " exceeds 10% of the steady response");
    }
    // --- tran tensor (greens.cpp:427-442): transient Green's maps at t = 10 ms * i / 100,
    // F_det (1 - exp(-t/tau)) -> kernel_to_die -> clamp_small_negatives(1e-2)
    {
        DBuf Fd, Fp, out, flag2;
        Fd.ensure(mm * 16);
        Fp.ensure(mm * 16);
        out.ensure(nn * 8);
        flag2.ensure(8);
        cuda_ok(cudaMemsetAsync(flag2.p, 0, 8, st), "memset");
        cuda_ok(gtd_fdet_full(d->fk_full.p, d->gtab.as<double>(), n, d->d.hp, g.alpha, g.beta, g.mu, Fd.p,
                              flag2.as<int>(), st),
                "fdet");
        double c3[3];
        cuda_ok(gtd_creduce(d->fk_full.p, mm, red.as<double>(), st), "creduce");
        d2h(c3, red.p, 24, st);
        const double inv = 1.0 / (double(m) * double(m));
        const int samples = 100;
        const double horizon = 0.010;
        g.t_samples.clear();
        g.tran.clear();
        for (int i = 1; i <= samples; ++i) {
            const double t = horizon * i / samples;
            cuda_ok(gtd_transient(d->fk_full.p, d->gtab.as<double>(), Fd.p, n, d->d.hp, g.alpha, g.capacitance,
                                  1e-6 * c3[2], t, Fp.p, 0.0, 0, nullptr, nullptr, flag2.as<int>(), st),
                    "transient factors");
            cuda_ok(gtd_fft2d(Fp.p, m, 1, +1, 1, d->tw64.p, st), "ifft");
            cuda_ok(gtd_kernel_to_die(Fp.p, n, inv, out.as<double>(), st), "kernel_to_die");
            Field map(n, pitch, Unit::KelvinPerWatt);
            d2h(map.v.data(), out.p, nn * 8, st);
            int fl2 = 0;
            d2h(&fl2, flag2.p, 4, st);
            if (fl2 & 1)
                fail(ST_SOLVER, "greens",
                     "non-positive transient time constant at an energetic frequency; transient closed form is "
                     "invalid here");
            const double peak = map.max(), floor = -1e-2 * std::max(peak, 0.0);  // clamp_small_negatives
            for (double& x : map.v) {
                if (x < floor)
                    fail(ST_VALIDATION, "greens", "tran tensor: negative value beyond spectral-ringing tolerance");
                if (x < 0.0) x = 0.0;
            }
            g.t_samples.push_back(t);
            g.tran.push_back(std::move(map));
        }
    }
    g.validate();
    return g;
}

void gt_ops_monte_carlo(const Greens& g, const VarParams& v, const Field& nominal_leak, const Field& p_dyn,
                        const std::vector<unsigned long long>& seeds, int jobs, const std::string& csv_path,
                        double* mean_max, double* std_max) {
    // reference monte_carlo (solver.cpp:338-409) + gt_monte_carlo (capi.cpp:345-369)
    if (seeds.empty()) fail(ST_CONFIG, "solver", "monte_carlo: empty seed list");
    need_device();
    g.validate();
    const int n = g.n;
    if (p_dyn.n != n) fail(ST_CONFIG, "solver", "monte_carlo: power map does not match the GreensSet grid");
    p_dyn.check_finite("monte_carlo");
    if (p_dyn.min() < 0.0) fail(ST_CONFIG, "solver", "monte_carlo: powers must be >= 0");
    if (nominal_leak.n != n) fail(ST_CONFIG, "solver", "monte_carlo: leakage map shape mismatch");
    if (nominal_leak.min() < 0.0) fail(ST_CONFIG, "variation", "leakage_baseline: nominal leakage must be >= 0");
    v.validate();
    int dev = 0;
    cudaGetDevice(&dev);
    auto d = prepare_device(g, GT_FP64, dev);
    cudaStream_t st = d->stream;
    const size_t nn = static_cast<size_t>(n) * n;
    const int B = static_cast<int>(seeds.size());
    const auto t0 = wall::now();
    // PreparedGreens / deterministic_spectrum at gs.mu: a runaway fails the whole call (solver.cpp:350-351)
    {
        DBuf Fd, flag;
        Fd.ensure(static_cast<size_t>(4) * nn * 16);
        flag.ensure(8);
        cuda_ok(cudaMemsetAsync(flag.p, 0, 8, st), "memset");
        cuda_ok(gtd_fdet_full(d->fk_full.p, d->gtab.as<double>(), n, d->d.hp, g.alpha, g.beta, g.mu, Fd.p,
                              flag.as<int>(), st),
                "fdet");
        int fl = 0;
        d2h(&fl, flag.p, 4, st);
        if (fl)
            fail(ST_SOLVER, "greens",
                 "deterministic_greens: spectral denominator collapsed below 1e-6 (leakage feedback gain reached unity)");
    }
    // Seeds stream through in chunks (the reference runs them one per worker thread with
    // per-thread memory, solver.cpp:376-387). The libstdc++ noise of chunk k + 1 is drawn on
    // `jobs` host threads (one work item per (seed, noise stream), largest first) into a
    // pinned ring while the device shapes chunk k's maps (exp(beta_L dL + beta_tox dTox),
    // variation.cpp:162-195) and runs the fused mode-A passes on them; one stream
    // synchronisation per chunk, none per seed. The chunk is sized so the two ring halves
    // stay within 256 MB of pinned memory (small chunks also keep the un-overlapped first
    // draw short).
    const bool has_sys = v.sigma_sys != 0.0, has_rnd = v.sigma_rand != 0.0;
    const size_t mm = 4 * nn;
    const size_t per_seed_host = (has_sys ? 2 * mm : 0) + (has_rnd ? 2 * nn : 0);  // doubles
    int chunk = static_cast<int>(std::min<size_t>(64, std::max<size_t>(1, (128ull << 20) / std::max<size_t>(1, per_seed_host * 8))));
    if (const char* e = getenv("GT_MC_SEED_CHUNK")) chunk = std::max(1, atoi(e));  // tests: force several chunks
    chunk = std::min(chunk, B);
    DBuf V, dl, dtox, P, N, flags, stats, scratch;
    V.ensure(nn * 8 * chunk);
    dl.ensure(nn * 8);
    dtox.ensure(nn * 8);
    flags.ensure(sizeof(int) * chunk);
    stats.ensure(sizeof(gtd_sample_stats) * chunk);
    scratch.ensure(gtd_mc_scratch_bytes_per_sample(n, 1) * chunk);
    upload(P, p_dyn.v.data(), nn * 8, st);
    upload(N, nominal_leak.v.data(), nn * 8, st);
    std::vector<int> capfail(B, 0);
    std::vector<gtd_sample_stats> hs(B);
    VarDevice vd(d.get(), v, g.pitch);
    const int nj = std::max(1, jobs);
    // noise ring: a process-wide pinned slab when free, a private one for a concurrent call
    static PinnedSlab shared_ring;
    static std::mutex ring_mu;
    std::unique_lock<std::mutex> ring_lock(ring_mu, std::try_to_lock);
    PinnedSlab own_ring;
    PinnedSlab& ring = ring_lock.owns_lock() ? shared_ring : own_ring;
    const size_t half = per_seed_host * chunk;
    ring.ensure(std::max<size_t>(1, 2 * half));
    // seed i of a half: [sys_l | sys_t | rnd_l | rnd_t]
    auto slot = [&](int hsel, int i, int which) -> double* {
        if ((which < 2 && !has_sys) || (which >= 2 && !has_rnd)) return nullptr;
        double* base = ring.p + static_cast<size_t>(hsel) * half + static_cast<size_t>(i) * per_seed_host;
        if (which < 2) return base + which * mm;
        return base + (has_sys ? 2 * mm : 0) + (which - 2) * nn;
    };
    static const uint64_t purpose[4] = {GL_SYS, OX_SYS, GL_RAND, OX_RAND};
    auto draw = [&](int hsel, int s0, int cnt) {
        // items: the m^2 systematic streams first (4x the draws of an n^2 random stream)
        std::vector<std::pair<int, int>> items;
        for (int pass = 0; pass < 2; ++pass)
            for (int i = 0; i < cnt; ++i)
                for (int w = 2 * pass; w < 2 * pass + 2; ++w)
                    if (slot(hsel, i, w)) items.emplace_back(i, w);
        std::atomic<size_t> next{0};
        std::vector<std::thread> pool;
        const int nt = static_cast<int>(std::min<size_t>(nj, items.size()));
        for (int w = 0; w < nt; ++w)
            pool.emplace_back([&] {
                for (size_t k = next.fetch_add(1); k < items.size(); k = next.fetch_add(1)) {
                    const int i = items[k].first, which = items[k].second;
                    draw_normals(derived_seed(seeds[s0 + i], purpose[which], 0), which < 2 ? 1.0 : v.sigma_rand,
                                 which < 2 ? mm : nn, slot(hsel, i, which));
                }
            });
        for (auto& th : pool) th.join();
    };
    std::vector<int> hflags(chunk);
    draw(0, 0, std::min(chunk, B));
    int hsel = 0;
    for (int s0 = 0; s0 < B; s0 += chunk, hsel ^= 1) {
        const int cnt = std::min(chunk, B - s0);
        // the next chunk's draws start now, on their own threads, while this thread feeds the device
        std::thread drawer;
        if (s0 + cnt < B) drawer = std::thread(draw, hsel ^ 1, s0 + cnt, std::min(chunk, B - s0 - cnt));
        struct Joiner {
            std::thread& t;
            ~Joiner() {
                if (t.joinable()) t.join();
            }
        } joiner{drawer};
        cuda_ok(cudaMemsetAsync(flags.p, 0, sizeof(int) * cnt, st), "memset");
        for (int i = 0; i < cnt; ++i) {
            vd.field(v, slot(hsel, i, 0), slot(hsel, i, 2), dl.as<double>(), false);
            vd.field(v, slot(hsel, i, 1), slot(hsel, i, 3), dtox.as<double>(), false);
            cuda_ok(gtd_leak_exp(nullptr, dl.as<double>(), dtox.as<double>(), v.beta_l, v.beta_tox, v.exponent_cap, n,
                                 V.as<double>() + i * nn, flags.as<int>() + i, st),
                    "leakage exponent");
        }
        // run_one per seed on the fused mode-A kernels: P and nominal broadcast, closed forms at gs.mu
        gtd_mc_in in{};
        in.P = P.p;
        in.N = N.p;
        in.V = V.p;
        in.sP = 0;
        in.sN = 0;
        in.sV = static_cast<long long>(nn);
        in.nom_scale = 1.0;
        gtd_mc_opts o{};
        o.mu_per_sample = 0;
        o.with_rand = 1;
        o.exponent_cap = 1e300;  // the cap was checked on the exponent itself above
        cuda_ok(gtd_mc_batch(&d->d, &in, cnt, &o, nullptr, stats.as<gtd_sample_stats>(), scratch.p, cnt, st, nullptr,
                             nullptr),
                "mc batch");
        d2h(hs.data() + s0, stats.p, sizeof(gtd_sample_stats) * cnt, st);  // synchronises: this ring half is free again
        d2h(hflags.data(), flags.p, sizeof(int) * cnt, st);
        for (int i = 0; i < cnt; ++i) capfail[s0 + i] = hflags[i];
    }
    const double per_ms = std::chrono::duration<double, std::milli>(wall::now() - t0).count() / B;

    std::vector<double> maxima;
    std::vector<std::string> errors(B);
    for (int i = 0; i < B; ++i) {
        int sbits = hs[i].status;
        if (capfail[i]) errors[i] = "leakage exponent exceeds cap (unphysical variation inputs)";
        else if (sbits & (GTD_ST_RUNAWAY_DET | GTD_ST_RUNAWAY_RAND))
            errors[i] = "random_greens: spectral denominator collapsed below 1e-6 (leakage feedback gain reached unity)";
        else if (sbits)
            errors[i] = "sample status " + std::to_string(sbits);
        if (errors[i].empty()) maxima.push_back(hs[i].max_rise);
    }
    if (!csv_path.empty()) {  // write_monte_carlo_csv (solver.cpp:411-423)
        std::ofstream os(csv_path);
        if (!os) fail(ST_CONFIG, "solver", "cannot open '" + csv_path + "' for writing");
        os << "seed,max_rise,mean_rise,runtime_ms\n";
        os.precision(17);
        for (int i = 0; i < B; ++i) {
            if (!errors[i].empty())
                os << seeds[i] << ",error,error," << per_ms << '\n';
            else
                os << seeds[i] << ',' << hs[i].max_rise << ',' << hs[i].mean_rise << ',' << per_ms << '\n';
        }
    }
    double mean = 0.0, sd = 0.0;
    if (!maxima.empty()) {
        for (double x : maxima) mean += x;
        mean /= maxima.size();
        double acc = 0.0;
        for (double x : maxima) acc += (x - mean) * (x - mean);
        sd = maxima.size() > 1 ? std::sqrt(acc / (maxima.size() - 1)) : 0.0;
    }
    if (mean_max) *mean_max = mean;
    if (std_max) *std_max = sd;
    for (int i = 0; i < B; ++i)
        if (!errors[i].empty())
            fail(ST_VALIDATION, "solver", "monte carlo seed " + std::to_string(seeds[i]) + " failed: " + errors[i]);
}

// steady_solve (fdm.cpp:167-205) with SolveOptions defaults (max_iters 50, tol 0.01 K, linear_tol 1e-9)
Field gt_ops_oracle_steady(const Stack& stack, const VarParams* var, const Field& p_dyn, const Field* nominal_leak,
                           int temp_dep_leakage, int temp_dep_conductivity, int* outer_iterations) {
    need_device();
    OracleSetup o = oracle_setup(stack, var, nominal_leak, temp_dep_leakage, temp_dep_conductivity);
    const int n = o.stack.n;
    if (o.temp_dep_cond && !(o.cond_c > 0.0))
        fail(ST_CONFIG, "oracle", "temp-dependent conductivity needs cond_c > 0");
    if (o.temp_dep_leakage && !o.have_leak)
        fail(ST_CONFIG, "oracle", "temp-dependent leakage needs a leakage baseline");
    if (p_dyn.n != n) fail(ST_CONFIG, "oracle", "power map does not match the stack grid");
    if (p_dyn.min() < 0.0) fail(ST_CONFIG, "oracle", "dynamic power must be >= 0");
    FdmNet net(o.stack, o.k_map);
    const size_t nn = net.nn, N = net.N;
    DBuf pd, lk;
    upload(pd, p_dyn.v.data(), nn * 8, net.st);
    if (o.have_leak) upload(lk, o.p_leak0.data(), nn * 8, net.st);
    const bool iterate = o.temp_dep_cond || o.temp_dep_leakage;
    const int max_iters = 50;
    const double tol = 0.01, linear_tol = 1e-9;
    Field rise(n, o.stack.pitch(), Unit::Kelvin);
    int it = 0;
    for (int iter = 1; iter <= max_iters; ++iter) {
        // p = p_dyn + leakage at the current die rise (x's die plane), x_old kept for the delta
        cuda_ok(cudaMemcpyAsync(net.xo.p, net.x.p, N * 8, cudaMemcpyDeviceToDevice, net.st), "copy");
        cuda_ok(gtd_fdm_rhs(pd.as<double>(), o.have_leak ? lk.as<double>() : nullptr, o.temp_dep_leakage, o.var.beta,
                            net.xo.as<double>(), 0, 0, 0, 0.0, static_cast<int>(nn), net.b.as<double>(), net.st),
                "rhs");
        net.prepare(o.temp_dep_cond && iter > 1 ? net.xo.as<double>() : nullptr, o.cond_c, 0.0);
        net.solve(0.0, iter > 1, linear_tol);
        cuda_ok(gtd_absdiff(net.x.as<double>(), net.xo.as<double>(), N, net.tmp.as<double>(), net.st), "delta");
        double r3[3];
        cuda_ok(gtd_reduce(net.tmp.as<double>(), N, net.red.as<double>(), net.st), "reduce");
        d2h(r3, net.red.p, 24, net.st);
        const double delta = r3[2];
        it = iter;
        if (!iterate || (iter > 1 && delta < tol)) break;
        if (iter == max_iters)
            fail(ST_SOLVER, "oracle",
                 "fixed-point loop hit max_iters with |dT| change " + std::to_string(delta) +
                     " K (thermal runaway or tolerance too tight)");
    }
    d2h(rise.v.data(), net.x.p, nn * 8, net.st);
    rise.check_finite("oracle die map");
    if (outer_iterations) *outer_iterations = it;
    return rise;
}

// gt_oracle_transient (reference capi.cpp:302-334): per sample time, backward Euler
// over round(span / dt) equal sub-steps with leakage refreshed every sub-step.
std::vector<Field> gt_ops_oracle_transient(const Stack& stack, const VarParams* var, const Field& p_dyn,
                                           const Field* nominal_leak, int temp_dep_leakage,
                                           const std::vector<double>& times, double dt) {
    need_device();
    if (times.empty()) fail(ST_CONFIG, "capi", "transient needs times");
    OracleSetup o = oracle_setup(stack, var, nominal_leak, temp_dep_leakage, 0);
    if (o.temp_dep_leakage && !o.have_leak)
        fail(ST_CONFIG, "oracle", "temp-dependent leakage needs a leakage baseline");
    const int n = o.stack.n;
    if (p_dyn.n != n) fail(ST_CONFIG, "oracle", "trace frame does not match the stack grid");
    if (p_dyn.min() < 0.0) fail(ST_CONFIG, "oracle", "trace powers must be >= 0");
    const double base_dt = dt > 0.0 ? dt : 1e-4;
    FdmNet net(o.stack, o.k_map);
    const size_t nn = net.nn, N = net.N;
    DBuf pd, lk;
    upload(pd, p_dyn.v.data(), nn * 8, net.st);
    if (o.have_leak) upload(lk, o.p_leak0.data(), nn * 8, net.st);
    std::vector<Field> out;
    double t_prev = 0.0;
    for (double target : times) {
        if (target <= t_prev) fail(ST_CONFIG, "capi", "sample times must be increasing");
        const double span = target - t_prev;
        const int steps = std::max(1, static_cast<int>(std::round(span / base_dt)));
        const double h = span / steps;
        net.prepare(nullptr, 0.0, 1.0 / h);
        for (int k = 0; k < steps; ++k) {
            cuda_ok(cudaMemcpyAsync(net.xo.p, net.x.p, N * 8, cudaMemcpyDeviceToDevice, net.st), "copy");
            cuda_ok(gtd_fdm_rhs(pd.as<double>(), o.have_leak ? lk.as<double>() : nullptr, o.temp_dep_leakage,
                                o.var.beta, net.xo.as<double>(), net.c_die, net.c_tim, net.c_spr, 1.0 / h,
                                static_cast<int>(nn), net.b.as<double>(), net.st),
                    "rhs");
            net.solve(1.0 / h, true, 1e-9);
        }
        Field f(n, o.stack.pitch(), Unit::Kelvin);
        d2h(f.v.data(), net.x.p, nn * 8, net.st);
        f.check_finite("oracle die map");
        out.push_back(std::move(f));
        t_prev = target;
    }
    return out;
}
