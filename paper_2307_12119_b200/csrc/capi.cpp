// capi.cpp — the drop-in C ABI (include/greentherm.h) and its batched
// extension (include/greentherm_b200.h). Host code is C++; every solve is
// enqueued on the GPU through the internal POD interface of gt_device.h.
// There is no CPU compute fallback: without a CUDA device the solve entries
// fail with GT_ERR_INTERNAL (stage "device").
//
// Error plumbing mirrors the reference (capi.cpp:22-48): exceptions never
// cross the ABI, message and stage are thread-local.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/greentherm.h"
#include "../../include/greentherm_b200.h"
#include "gt_device.h"
#include "devctx.hpp"
#include "gt_ops.h"
#include "host.hpp"

using namespace gth;

static_assert(sizeof(gt_sample_stats) == sizeof(gtd_sample_stats), "stats layout");

namespace {

thread_local std::string t_err;
thread_local std::string t_stage;

template <typename Fn>
gt_status guarded(Fn&& fn) {
    try {
        fn();
        return GT_OK;
    } catch (const Error& e) {
        t_err = e.what();
        t_stage = e.stage;
        return static_cast<gt_status>(e.status);
    } catch (const std::exception& e) {
        t_err = e.what();
        t_stage = "internal";
        return GT_ERR_INTERNAL;
    }
}

using wall = std::chrono::steady_clock;
double ms_since(wall::time_point t0) {
    return std::chrono::duration<double, std::milli>(wall::now() - t0).count();
}

}  // namespace

// ------------------------------------------------------------ handle types
struct gt_field {
    Field f;
};
struct gt_greens {
    Greens g;
    mutable GtSolveSlot slot;  // prepared device set, built by the first gt_solve_* call
};
struct gt_result {
    std::vector<Field> rise;
    std::vector<double> times;
};
struct gt_trace {
    double dt = 0.0;
    std::vector<Field> frames;
};

namespace {

gtd_mc_opts to_dev_opts(const gt_batch_opts* o) {
    gtd_mc_opts r{};
    r.mu_per_sample = o ? o->mu_per_sample : 1;
    r.with_rand = o ? o->with_rand : 1;
    r.exponent_cap = (o && o->exponent_cap > 0.0) ? o->exponent_cap : 6.0;
    r.resolve = nullptr;
    return r;
}

// The fp64 re-solve attached to an fp32 batch ("fp32 with fp64 residual check",
// BASELINE config 1): pairs whose random_greens denominator came within
// 1/sqrt(thr) of singular are solved again in fp64 on the device. Measured on
// config-1 pairs (tools/diag_mf.py): every pair above 1e-3 K fp32 error had
// max 1/|den2|^2 > 2e5, every pair below 1e4 stayed under 2.6e-4 K; 1-2% of
// pairs exceed 1e4. Capacity: batch/16 pairs (at least 8).
const gtd_mc_resolve* attach_resolve(gt_device_greens* d, int slot, int batch, const gt_batch_opts* o) {
    if (d->fp64) return nullptr;
    double thr = o ? o->fp64_check : 0.0;
    if (thr < 0.0) return nullptr;
    if (thr == 0.0) thr = 1e4;
    if (!d->dev64) d->dev64 = gth::prepare_device(d->host, GT_FP64, d->device);
    const int n = d->d.n;
    const int cap = std::max(8, (batch + 15) / 16);
    const size_t nn = static_cast<size_t>(n) * n;
    auto& r = d->resolve[slot];
    r.in.ensure(static_cast<size_t>(cap) * 3 * nn * 8);
    r.out.ensure(static_cast<size_t>(cap) * nn * 8);
    r.stats.ensure(static_cast<size_t>(cap) * sizeof(gtd_sample_stats));
    r.scr.ensure(static_cast<size_t>(cap) * gtd_mc_scratch_bytes_per_sample(n, 1));
    r.sel.ensure(static_cast<size_t>(cap + 1) * sizeof(int));
    r.d.g64 = &d->dev64->d;
    r.d.in64 = r.in.p;
    r.d.out64 = r.out.p;
    r.d.stats64 = r.stats.as<gtd_sample_stats>();
    r.d.scratch64 = r.scr.p;
    r.d.sel = r.sel.as<int>();
    r.d.cap = cap;
    r.d.thr = static_cast<float>(thr);
    return &r.d;
}

// Scratch budget of the automatic chunking: 40% of the device's free memory,
// within [1.5 GiB, 32 GiB] (a 4096-sample chunk at n = 256 needs ~6.6 GB; at
// n = 1024 a sample alone needs ~25 MB fp32 / ~50 MB fp64).
size_t scratch_budget() {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) fr = 0;
    const size_t lo = 1536ull << 20, hi = 32ull << 30;
    return std::min(hi, std::max(lo, fr / 10 * 4));
}

// share: scratch buffers in flight; have: bytes of one scratch buffer already
// allocated (a call that fits in it skips the cudaMemGetInfo query: no driver
// round trip on the launch path of repeated calls)
#ifndef GT_E2E_CHUNK
#define GT_E2E_CHUNK 128  // first / last chunk of the host-input pipelines (pairs)
#endif
#ifndef GT_E2E_BIG
#define GT_E2E_BIG 256    // steady-state chunk of the host-input pipelines (pairs)
#endif

// Chunk sizes of the host-input pipelines (two slots in flight). On the B200 hosts a
// pinned H2D copy of 32 MiB runs at ~44 GB/s and one of >= 256 MiB at ~55 GB/s
// (tools/h2d_bw.py: a ~0.15 ms fixed cost per copy), while a small first chunk shortens
// the exposed first copy and a small last chunk the exposed last compute. So chunks ramp
// up from GT_E2E_CHUNK to GT_E2E_BIG by doublings and back down at the end. Measured on
// config 1 (4096 pairs, gt_mc_batch_seeded, tools/e2e_var.sh): uniform 128: 183k solves/s;
// ramp 128 -> 512: 183k; 128 -> 1024: 152k; 64 -> 128: 164k; 128 -> 256: 195k (the
// default: 21.0 ms per step against ~19.5 ms of pure PCIe time for its 1 GiB). A
// caller-set chunk (gt_batch_opts.chunk) is used as is.
std::vector<int> pipeline_chunks(int batch, const gt_batch_opts* o) {
    std::vector<int> out;
    if (o && o->chunk > 0) {
        for (int s0 = 0; s0 < batch; s0 += o->chunk) out.push_back(std::min(o->chunk, batch - s0));
        return out;
    }
    std::vector<int> up;
    for (int c = GT_E2E_CHUNK; c < GT_E2E_BIG; c *= 2) up.push_back(c);
    int ramp = 0;
    for (int c : up) ramp += 2 * c;
    if (batch <= ramp + GT_E2E_BIG) {
        for (int s0 = 0; s0 < batch; s0 += GT_E2E_CHUNK) out.push_back(std::min(GT_E2E_CHUNK, batch - s0));
        return out;
    }
    out = up;
    int mid = batch - ramp;
    while (mid > 0) {
        out.push_back(std::min(GT_E2E_BIG, mid));
        mid -= GT_E2E_BIG;
    }
    out.insert(out.end(), up.rbegin(), up.rend());
    return out;
}

int auto_chunk(int n, int fp64, int batch, const gt_batch_opts* o, int share = 1, size_t have = 0) {
    if (o && o->chunk > 0) return std::min(o->chunk, batch);
    const int want = std::min(4096, batch);
    if (have >= gtd_mc_scratch_bytes_per_sample(n, fp64) * static_cast<size_t>(want)) return want;
    // Large chunks win: the passes are SM-issue bound, not HBM bound (a sweep of
    // 24..4096 pairs per chunk on B200 went 232k -> 325k solves/s; L2 residency
    // of the intermediates at <= 48 MB bought nothing), every launch ends in a
    // partly idle tail (config 1 at 4096 vs 1024 pairs per chunk: +1.7%), and a
    // chunk that leaves a small remainder runs that tail at low occupancy.
    const size_t per = gtd_mc_scratch_bytes_per_sample(n, fp64);
    int c = static_cast<int>(std::max<size_t>(1, std::min<size_t>(4096, scratch_budget() / share / per)));
    return std::min(c, batch);
}

}  // namespace

extern "C" {

// ------------------------------------------------------------- status / errors
const char* gt_status_name(gt_status s) {
    switch (s) {
        case GT_OK: return "ok";
        case GT_ERR_CONFIG: return "config";
        case GT_ERR_SOLVER: return "solver";
        case GT_ERR_VALIDATION: return "validation";
        case GT_ERR_INTERNAL: return "internal";
    }
    return "unknown";
}
const char* gt_last_error(void) { return t_err.c_str(); }
const char* gt_last_error_stage(void) { return t_stage.c_str(); }

// ------------------------------------------------------------------ fields
gt_status gt_field_create(int n, double pitch, const char* unit, gt_field** out) {
    return guarded([&] { *out = new gt_field{Field(n, pitch, parse_unit(unit ? unit : "watts"))}; });
}
gt_status gt_field_load(const char* path, gt_field** out) {
    return guarded([&] { *out = new gt_field{read_field(path)}; });
}
gt_status gt_field_save(const gt_field* f, const char* path) {
    return guarded([&] { write_field(f->f, path); });
}
void gt_field_free(gt_field* f) { delete f; }
int gt_field_n(const gt_field* f) { return f->f.n; }
double gt_field_pitch(const gt_field* f) { return f->f.pitch; }
const char* gt_field_unit(const gt_field* f) { return unit_str(f->f.unit); }
double gt_field_get(const gt_field* f, int i, int j) { return f->f.at(i, j); }
void gt_field_set(gt_field* f, int i, int j, double value) { f->f.at(i, j) = value; }
const double* gt_field_data(const gt_field* f) { return f->f.v.data(); }
double gt_field_max(const gt_field* f) { return f->f.max(); }
double gt_field_sum(const gt_field* f) { return f->f.sum(); }

gt_status gt_field_render(const gt_field* f, const char* path, int cell_px) {
    // P6 raster with the legend in header comments (reference heatmap.cpp:41-76).
    return guarded([&] {
        const Field& F = f->f;
        F.check_finite("render_heatmap input");
        const int px = cell_px < 1 ? 4 : cell_px;
        const double lo = F.min(), hi = F.max(), span = hi - lo;
        static const unsigned char stops[5][3] = {{0, 0, 96}, {0, 128, 255}, {0, 224, 128}, {255, 224, 0}, {224, 16, 16}};
        std::ofstream os(path, std::ios::binary);
        if (!os) fail(ST_CONFIG, "heatmap", std::string("cannot open '") + path + "' for writing");
        char hdr[160];
        const int w = F.n * px;
        const int len = std::snprintf(hdr, sizeof hdr, "P6\n# legend_min %.12g K\n# legend_max %.12g K\n%d %d\n255\n",
                                      lo, hi, w, w);
        os.write(hdr, len);
        std::string row(static_cast<size_t>(w) * 3, '\0');
        for (int i = 0; i < F.n; ++i) {
            for (int j = 0; j < F.n; ++j) {
                const double t = span > 0.0 ? std::clamp((F.at(i, j) - lo) / span, 0.0, 1.0) : 0.0;
                const double x = t * 4.0;
                const int k = std::min(static_cast<int>(x), 3);
                const double a = x - k;
                unsigned char rgb[3];
                for (int ch = 0; ch < 3; ++ch)
                    rgb[ch] = static_cast<unsigned char>(stops[k][ch] + (stops[k + 1][ch] - stops[k][ch]) * a + 0.5);
                for (int p = 0; p < px; ++p) std::memcpy(&row[(static_cast<size_t>(j) * px + p) * 3], rgb, 3);
            }
            for (int p = 0; p < px; ++p) os.write(row.data(), static_cast<std::streamsize>(row.size()));
        }
        if (!os) fail(ST_CONFIG, "heatmap", std::string("write failed for '") + path + "'");
    });
}

gt_status gt_write_default_stack(const char* path) {
    return guarded([&] { save_stack_file(Stack{}, path); });
}
gt_status gt_write_default_variation(const char* path) {
    return guarded([&] { save_var_file(VarParams{}, path); });
}

// ------------------------------------------------------------------ greens
gt_status gt_calibrate(const char* stack_path, const char* variation_path, const gt_field* nominal_leak,
                       double leak_total, gt_greens** out, double* offline_ms) {
    return guarded([&] {
        auto t0 = wall::now();
        Stack s = stack_path ? load_stack_file(stack_path) : Stack{};
        VarParams v = variation_path ? load_var_file(variation_path) : VarParams{};
        Greens g = gt_ops_calibrate_modal(s, v, nominal_leak ? &nominal_leak->f : nullptr, leak_total);
        if (offline_ms) *offline_ms = ms_since(t0);
        *out = new gt_greens{std::move(g)};
    });
}
gt_status gt_modal_kernel(const char* stack_path, int* n_out, double* f_sp0_out) {
    return guarded([&] {
        Stack s = stack_path ? load_stack_file(stack_path) : Stack{};
        if (n_out) *n_out = s.n;
        if (f_sp0_out) gt_ops_modal_kernel(s, f_sp0_out);
    });
}
gt_status gt_greens_save(const gt_greens* g, const char* dir) {
    return guarded([&] { save_greens_dir(g->g, dir); });
}
gt_status gt_greens_load(const char* dir, gt_greens** out) {
    return guarded([&] { *out = new gt_greens{load_greens_dir(dir)}; });
}
void gt_greens_free(gt_greens* g) { delete g; }
int gt_greens_n(const gt_greens* g) { return g->g.n; }
double gt_greens_alpha(const gt_greens* g) { return g->g.alpha; }
double gt_greens_beta(const gt_greens* g) { return g->g.beta; }
double gt_greens_mu(const gt_greens* g) { return g->g.mu; }
double gt_greens_capacitance(const gt_greens* g) { return g->g.capacitance; }
double gt_greens_kappa_inf(const gt_greens* g) { return g->g.kappa_inf; }
gt_status gt_greens_field(const gt_greens* g, const char* which, gt_field** out) {
    return guarded([&] {
        const std::string w = which ? which : "";
        const Field* f = w == "f_sp0"    ? &g->g.f_sp0
                         : w == "g_sp0"  ? &g->g.g_sp0
                         : w == "f_det"  ? &g->g.f_det
                         : w == "f_rand" ? &g->g.f_rand
                         : w == "p_var"  ? &g->g.p_var
                                         : nullptr;
        if (!f) fail(ST_CONFIG, "capi", "unknown greens field '" + w + "'");
        *out = new gt_field{*f};
    });
}

// ------------------------------------------------------------------ results
int gt_result_count(const gt_result* r) { return static_cast<int>(r->rise.size()); }
double gt_result_time(const gt_result* r, int idx) {
    return (idx < 0 || static_cast<size_t>(idx) >= r->times.size()) ? 0.0 : r->times[idx];
}
gt_status gt_result_map(const gt_result* r, int idx, gt_field** out) {
    return guarded([&] {
        if (idx < 0 || static_cast<size_t>(idx) >= r->rise.size()) fail(ST_CONFIG, "capi", "result index out of range");
        *out = new gt_field{r->rise[idx]};
    });
}
void gt_result_free(gt_result* r) { delete r; }

// ------------------------------------------------------------------ solves
gt_status gt_solve_steady(const gt_greens* g, const gt_field* p_dyn, int with_rand, gt_field** out,
                          double* online_ms) {
    return guarded([&] {
        double ms = 0.0;
        Field f = gt_ops_steady(g->g, g->slot, p_dyn->f, with_rand != 0, &ms);
        if (online_ms) *online_ms = ms;
        *out = new gt_field{std::move(f)};
    });
}

gt_status gt_solve_step(const gt_greens* g, const gt_field* p_dyn, const double* times, int n_times,
                        int with_rand, gt_result** out, double* online_ms) {
    return guarded([&] {
        if (!times || n_times < 1) fail(ST_CONFIG, "capi", "step solve needs times");
        double ms = 0.0;
        std::vector<double> tv(times, times + n_times);
        auto r = std::make_unique<gt_result>();
        r->rise = gt_ops_step(g->g, g->slot, p_dyn->f, tv, with_rand != 0, &ms);
        r->times = tv;
        if (online_ms) *online_ms = ms;
        *out = r.release();
    });
}

gt_status gt_trace_load(const char* dir, gt_trace** out) {
    return guarded([&] {
        const Kv kv = Kv::parse(std::string(dir) + "/trace.txt");
        auto t = std::make_unique<gt_trace>();
        t->dt = kv.num("dt");
        const long long cnt = kv.integer("frames");
        for (long long i = 0; i < cnt; ++i) {
            char b[32];
            std::snprintf(b, sizeof b, "frame_%04lld.map", i);
            t->frames.push_back(read_field(std::string(dir) + "/" + b));
        }
        gt_ops_check_trace(t->dt, t->frames);
        *out = t.release();
    });
}
gt_status gt_trace_create(double dt, gt_trace** out) {
    return guarded([&] {
        if (!(dt > 0.0)) fail(ST_CONFIG, "capi", "trace dt must be positive");
        auto t = std::make_unique<gt_trace>();
        t->dt = dt;
        *out = t.release();
    });
}
gt_status gt_trace_push(gt_trace* t, const gt_field* frame) {
    return guarded([&] { t->frames.push_back(frame->f); });
}
gt_status gt_trace_save(const gt_trace* t, const char* dir) {
    return guarded([&] {
        gt_ops_check_trace(t->dt, t->frames);
        std::filesystem::create_directories(dir);
        Kv kv;
        kv.put_num("dt", t->dt);
        kv.put_int("frames", static_cast<long long>(t->frames.size()));
        kv.save(std::string(dir) + "/trace.txt");
        for (size_t i = 0; i < t->frames.size(); ++i) {
            char b[32];
            std::snprintf(b, sizeof b, "frame_%04zu.map", i);
            write_field(t->frames[i], std::string(dir) + "/" + b);
        }
    });
}
int gt_trace_frames(const gt_trace* t) { return static_cast<int>(t->frames.size()); }
double gt_trace_dt(const gt_trace* t) { return t->dt; }
void gt_trace_free(gt_trace* t) { delete t; }

gt_status gt_solve_trace(const gt_greens* g, const gt_trace* trace, int window, int with_rand,
                         gt_result** out, double* online_ms) {
    return guarded([&] {
        double ms = 0.0;
        auto r = std::make_unique<gt_result>();
        r->rise = gt_ops_trace(g->g, g->slot, trace->dt, trace->frames, window, with_rand != 0, &r->times, &ms);
        if (online_ms) *online_ms = ms;
        *out = r.release();
    });
}

// ---------------------------------------------------- FDM reference solver (device, fdm.cu)
gt_status gt_oracle_steady(const char* stack_path, const char* variation_path, const gt_field* p_dyn,
                           const gt_field* nominal_leak, int temp_dep_leakage, int temp_dep_conductivity,
                           gt_field** out, int* outer_iterations) {
    return guarded([&] {
        if (!p_dyn || !out) fail(ST_CONFIG, "capi", "oracle needs a power map and an output");
        Stack s = stack_path ? load_stack_file(stack_path) : Stack{};
        VarParams v;
        if (variation_path) v = load_var_file(variation_path);
        Field f = gt_ops_oracle_steady(s, variation_path ? &v : nullptr, p_dyn->f,
                                       nominal_leak ? &nominal_leak->f : nullptr, temp_dep_leakage,
                                       temp_dep_conductivity, outer_iterations);
        *out = new gt_field{std::move(f)};
    });
}
gt_status gt_oracle_transient(const char* stack_path, const char* variation_path, const gt_field* p_dyn,
                              const gt_field* nominal_leak, int temp_dep_leakage, const double* times, int n_times,
                              double dt, gt_result** out) {
    return guarded([&] {
        if (!times || n_times < 1) fail(ST_CONFIG, "capi", "transient needs times");
        if (!p_dyn || !out) fail(ST_CONFIG, "capi", "oracle needs a power map and an output");
        Stack s = stack_path ? load_stack_file(stack_path) : Stack{};
        VarParams v;
        if (variation_path) v = load_var_file(variation_path);
        std::vector<double> tv(times, times + n_times);
        auto r = std::make_unique<gt_result>();
        r->rise = gt_ops_oracle_transient(s, variation_path ? &v : nullptr, p_dyn->f,
                                          nominal_leak ? &nominal_leak->f : nullptr, temp_dep_leakage, tv, dt);
        r->times = tv;
        *out = r.release();
    });
}

gt_status gt_error_metrics(const gt_field* calc, const gt_field* ref, gt_error_report* out) {
    // reference solver.cpp:289-312
    return guarded([&] {
        const Field& a = calc->f;
        const Field& b = ref->f;
        if (!a.same_shape(b)) fail(ST_CONFIG, "solver", "error_metrics: map shapes differ");
        double sum = 0.0, mx = 0.0;
        for (size_t k = 0; k < a.v.size(); ++k) {
            const double e = std::abs(a.v[k] - b.v[k]);
            sum += e;
            mx = std::max(mx, e);
        }
        const double mae = sum / static_cast<double>(a.v.size());
        const double rmax = b.max();
        out->mae = mae;
        out->max_err = mx;
        out->pct_of_max_rise = rmax > 0.0 ? 100.0 * mae / rmax : 0.0;
        out->max_pct_of_max_rise = rmax > 0.0 ? 100.0 * mx / rmax : 0.0;
        const auto [ci, cj] = a.argmax();
        const auto [ri, rj] = b.argmax();
        out->hotspot_hit = std::max(std::abs(ci - ri), std::abs(cj - rj)) <= 1 ? 1 : 0;
    });
}

gt_status gt_monte_carlo(const gt_greens* g, const char* variation_path, const gt_field* nominal_leak,
                         double leak_total, const gt_field* p_dyn, const unsigned long long* seeds, int n_seeds,
                         int jobs, const char* csv_path, double* mean_max, double* std_max) {
    return guarded([&] {
        if (!seeds || n_seeds < 1) fail(ST_CONFIG, "capi", "monte carlo needs seeds");
        VarParams v = variation_path ? load_var_file(variation_path) : VarParams{};
        const Greens& G = g->g;
        Field leak = nominal_leak ? nominal_leak->f
                                  : Field(G.n, G.pitch, Unit::Watts,
                                          (leak_total > 0.0 ? leak_total : 15.0) / (static_cast<double>(G.n) * G.n));
        std::vector<unsigned long long> sv(seeds, seeds + n_seeds);
        gt_ops_monte_carlo(G, v, leak, p_dyn->f, sv, jobs, csv_path ? csv_path : "", mean_max, std_max);
    });
}

gt_status gt_write_builtin_suite(const char*, const char*) {
    return guarded([&] {
        fail(ST_INTERNAL, "validate",
             "the oracle-vs-Green validation suite needs the FDM solver, which is not part of the device build");
    });
}
gt_status gt_validate_suite(const char*, const char*, int, int*, int*) {
    return guarded([&] {
        fail(ST_INTERNAL, "validate",
             "the oracle-vs-Green validation suite needs the FDM solver, which is not part of the device build");
    });
}

// ------------------------------------------------------ batched extension
gt_status gt_greens_from_arrays(int n, double pitch, const double* f_sp0, const double* g_sp0, double phi,
                                double kappa_inf, double alpha, double beta, double mu, double capacitance,
                                double rand_scale, const double* f_det, const double* f_rand,
                                const double* p_var, gt_greens** out) {
    return guarded([&] {
        if (!f_sp0) fail(ST_CONFIG, "greens", "f_sp0 is required");
        Greens g;
        g.n = n;
        g.pitch = pitch;
        const size_t nn = static_cast<size_t>(n) * n;
        auto mk = [&](const double* src, Unit u) {
            Field f(n, pitch, u);
            if (src) std::copy(src, src + nn, f.v.begin());
            return f;
        };
        g.f_sp0 = mk(f_sp0, Unit::KelvinPerWatt);
        if (g_sp0) {
            g.g_sp0 = mk(g_sp0, Unit::KelvinPerWatt);
        } else {
            g.g_sp0 = g.f_sp0;
            const double shift = g.f_sp0.at(n / 2, n / 2) - kappa_inf;
            for (double& x : g.g_sp0.v) x += shift;
        }
        g.f_det = mk(f_det, Unit::KelvinPerWatt);
        g.f_rand = mk(f_rand, Unit::KelvinPerWatt);
        g.p_var = mk(p_var, Unit::Watts);
        g.phi = phi;
        g.kappa_inf = kappa_inf;
        g.alpha = alpha;
        g.beta = beta;
        g.mu = mu;
        g.capacitance = capacitance;
        g.rand_scale = rand_scale;
        g.validate();
        *out = new gt_greens{std::move(g)};
    });
}

gt_status gt_greens_to_device(const gt_greens* g, int precision, int device, gt_device_greens** out) {
    return guarded([&] { *out = prepare_device(g->g, precision, device).release(); });
}
void gt_device_greens_free(gt_device_greens* d) { delete d; }
int gt_device_greens_precision(const gt_device_greens* d) { return d->fp64 ? GT_FP64 : GT_FP32; }

void gt_batch_opts_default(gt_batch_opts* o) {
    o->leak_frac = 0.3;
    o->mu_per_sample = 1;
    o->with_rand = 1;
    o->chunk = 0;
    o->exponent_cap = 6.0;
    o->fp64_check = 0.0;
}

size_t gt_mc_scratch_bytes(int n, int precision) { return gtd_mc_scratch_bytes_per_sample(n, precision == GT_FP64); }
int gt_mc_kernel_launches(int batch, int chunk) { return gtd_mc_launch_count(batch, chunk); }

int gt_device_count(void) {
    int n = 0;
    return cudaGetDeviceCount(&n) == cudaSuccess ? n : 0;
}

gt_status gt_mc_batch_device(const gt_device_greens* dc, const void* p_dyn, const void* var, int batch,
                             const gt_batch_opts* opts, void* t_out, gt_sample_stats* stats, void* stream) {
    return guarded([&] {
        if (batch < 1 || !p_dyn || !var || !stats) fail(ST_CONFIG, "capi", "batch needs inputs and a stats array");
        auto* d = const_cast<gt_device_greens*>(dc);
        std::lock_guard<std::mutex> lk(d->mu);
        cuda_ok(cudaSetDevice(d->device), "cudaSetDevice");
        const int n = d->d.n;
        const int chunk = auto_chunk(n, d->fp64, batch, opts, 1, d->scratch.bytes);
        d->scratch.ensure(gtd_mc_scratch_bytes_per_sample(n, d->fp64) * chunk);
        gtd_mc_opts o = to_dev_opts(opts);
        o.resolve = attach_resolve(d, 0, batch, opts);
        gtd_mc_in in{};
        in.P = p_dyn;
        in.N = p_dyn;
        in.V = var;
        in.sP = in.sN = in.sV = static_cast<long long>(n) * n;
        in.nom_scale = opts ? opts->leak_frac : 0.3;
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->stream;
        d->order_in(st);
        cuda_ok(gtd_mc_batch(&d->d, &in, batch, &o, t_out, reinterpret_cast<gtd_sample_stats*>(stats),
                             d->scratch.p, chunk, st, d->profiling ? &gt_device_greens::mark : nullptr, d),
                "mc batch launch");
        d->order_out(st);
        d->kernels += gtd_mc_launch_count(batch, chunk) + (o.resolve ? gtd_mc_resolve_launch_count() : 0);
        d->calls += 1;
    });
}

gt_status gt_mc_batch(const gt_device_greens* dc, const void* p_dyn, const void* var, int batch,
                      const gt_batch_opts* opts, void* t_out, double* max_out, double* mean_out, int* status_out,
                      double* online_ms) {
    return guarded([&] {
        if (batch < 1 || !p_dyn || !var) fail(ST_CONFIG, "capi", "batch needs inputs");
        auto t0 = wall::now();
        auto* d = const_cast<gt_device_greens*>(dc);
        std::lock_guard<std::mutex> lk(d->mu);
        cuda_ok(cudaSetDevice(d->device), "cudaSetDevice");
        const int n = d->d.n;
        const size_t es = d->fp64 ? 8 : 4;
        const size_t map = static_cast<size_t>(n) * n * es;
        // Pipeline chunks: two slots in flight, sizes ramping up and down (pipeline_chunks)
        const std::vector<int> chunks = pipeline_chunks(batch, opts);
        const int chunk = *std::max_element(chunks.begin(), chunks.end());
        const int inner = auto_chunk(n, d->fp64, chunk, nullptr, 2, d->slot_scr[1].bytes);
        gtd_mc_opts o = to_dev_opts(opts);
        for (int s = 0; s < 2; ++s) {
            if (!d->slot_stream[s]) cuda_ok(cudaStreamCreateWithFlags(&d->slot_stream[s], cudaStreamNonBlocking), "stream");
            d->slot_in[s].ensure(2 * map * chunk);
            if (t_out) d->slot_out[s].ensure(map * chunk);
            d->slot_scr[s].ensure(gtd_mc_scratch_bytes_per_sample(n, d->fp64) * inner);
            d->slot_stats[s].ensure(sizeof(gtd_sample_stats) * chunk);
        }
        const size_t hs_bytes = sizeof(gtd_sample_stats) * static_cast<size_t>(batch);
        if (d->host_stats_bytes < hs_bytes) {
            if (d->host_stats) cudaFreeHost(d->host_stats);
            d->host_stats = nullptr;
            d->host_stats_bytes = 0;
            cuda_ok(cudaMallocHost(&d->host_stats, hs_bytes), "cudaMallocHost");
            d->host_stats_bytes = hs_bytes;
        }
        auto* hs = static_cast<gtd_sample_stats*>(d->host_stats);
        const char* P = static_cast<const char*>(p_dyn);
        const char* V = static_cast<const char*>(var);
        for (int s0 = 0, k = 0; k < static_cast<int>(chunks.size()); s0 += chunks[k], ++k) {
            const int cnt = chunks[k];
            const int s = k & 1;
            cudaStream_t st = d->slot_stream[s];
            char* din = static_cast<char*>(d->slot_in[s].p);
            cuda_ok(cudaMemcpyAsync(din, P + s0 * map, cnt * map, cudaMemcpyHostToDevice, st), "h2d p");
            cuda_ok(cudaMemcpyAsync(din + chunk * map, V + s0 * map, cnt * map, cudaMemcpyHostToDevice, st), "h2d var");
            gtd_mc_in in{};
            in.P = din;
            in.N = din;
            in.V = din + chunk * map;
            in.sP = in.sN = in.sV = static_cast<long long>(n) * n;
            in.nom_scale = opts ? opts->leak_frac : 0.3;
            auto* dst = static_cast<gtd_sample_stats*>(d->slot_stats[s].p);
            o.resolve = attach_resolve(d, 1 + s, chunk, opts);
            cuda_ok(gtd_mc_batch(&d->d, &in, cnt, &o, t_out ? d->slot_out[s].p : nullptr, dst, d->slot_scr[s].p,
                                 std::min(inner, cnt), st, nullptr, nullptr),
                    "mc batch launch");
            d->kernels += gtd_mc_launch_count(cnt, std::min(inner, cnt)) + (o.resolve ? gtd_mc_resolve_launch_count() : 0);
            if (t_out)
                cuda_ok(cudaMemcpyAsync(static_cast<char*>(t_out) + s0 * map, d->slot_out[s].p, cnt * map,
                                        cudaMemcpyDeviceToHost, st),
                        "d2h maps");
            cuda_ok(cudaMemcpyAsync(hs + s0, dst, sizeof(gtd_sample_stats) * cnt, cudaMemcpyDeviceToHost, st), "d2h stats");
        }
        for (auto& st : d->slot_stream) cuda_ok(cudaStreamSynchronize(st), "batch sync");
        for (int i = 0; i < batch; ++i) {
            if (max_out) max_out[i] = hs[i].max_rise;
            if (mean_out) mean_out[i] = hs[i].mean_rise;
            if (status_out) status_out[i] = hs[i].status;
        }
        if (online_ms) *online_ms = ms_since(t0);
    });
}

gt_status gt_var_model(gt_device_greens* d, double sigma_over_mu, double range_frac) {
    return guarded([&] {
        if (!d) fail(ST_CONFIG, "capi", "null device GreensSet");
        if (!(sigma_over_mu >= 0.0) || !(range_frac > 0.0))
            fail(ST_CONFIG, "variation", "variation model needs sigma/mu >= 0 and a positive correlation range");
        const int n = d->d.n, m = d->d.m;
        if (m != 128 && m != 256 && m != 512)
            fail(ST_CONFIG, "device", "seeded device variation supports n = 64, 128, 256");
        std::lock_guard<std::mutex> lk(d->mu);
        cuda_ok(cudaSetDevice(d->device), "cudaSetDevice");
        cudaStream_t st = d->stream;
        const size_t mm = static_cast<size_t>(m) * m;
        DBuf work, lam, red;
        work.ensure(mm * 16);
        lam.ensure(mm * 8);
        red.ensure(64);
        d->order_in(st);  // earlier calls' generation may still read the old model
        d->var_sqlam.ensure(static_cast<size_t>(m) * gtd_var_pitch(n) * (d->fp64 ? 8 : 4));
        const double pitch = d->host.pitch;
        cuda_ok(gtd_var_model(&d->d, d->tw64.p, pitch, range_frac * pitch * n, work.p, lam.as<double>(),
                              red.as<double>(), d->var_sqlam.p, st),
                "variation model");
        cuda_ok(cudaStreamSynchronize(st), "sync");
        d->var_sigma = sigma_over_mu;
    });
}

namespace {
void need_var_model(const gt_device_greens* d) {
    if (!d->var_sqlam.p) fail(ST_CONFIG, "variation", "call gt_var_model before generating seeded variation maps");
}
}  // namespace

gt_status gt_var_generate_device(const gt_device_greens* dc, const unsigned long long* seeds, int batch, void* var_out,
                                 void* stream) {
    return guarded([&] {
        if (!dc || batch < 1 || !seeds || !var_out) fail(ST_CONFIG, "capi", "variation generation needs seeds and output");
        auto* d = const_cast<gt_device_greens*>(dc);
        need_var_model(d);
        std::lock_guard<std::mutex> lk(d->mu);
        cuda_ok(cudaSetDevice(d->device), "cudaSetDevice");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->stream;
        const int chunk = std::min(batch, 1024);
        d->order_in(st);
        d->var_scratch.ensure(gtd_var_scratch_bytes_per_sample(d->d.n, d->fp64) * chunk);
        cuda_ok(gtd_var_generate(&d->d, d->var_sqlam.p, seeds, batch, d->var_sigma, var_out, d->var_scratch.p, chunk, st),
                "variation generation");
        d->order_out(st);
        d->kernels += 2 * ((batch + chunk - 1) / chunk);
    });
}

gt_status gt_mc_batch_seeded(const gt_device_greens* dc, const void* p_dyn, const unsigned long long* seeds, int batch,
                             const gt_batch_opts* opts, void* t_out, double* max_out, double* mean_out,
                             int* status_out, double* online_ms) {
    return guarded([&] {
        if (batch < 1 || !p_dyn || !seeds) fail(ST_CONFIG, "capi", "batch needs power maps and seeds");
        auto t0 = wall::now();
        auto* d = const_cast<gt_device_greens*>(dc);
        need_var_model(d);
        std::lock_guard<std::mutex> lk(d->mu);
        cuda_ok(cudaSetDevice(d->device), "cudaSetDevice");
        const int n = d->d.n;
        const size_t es = d->fp64 ? 8 : 4;
        const size_t map = static_cast<size_t>(n) * n * es;
        const std::vector<int> chunks = pipeline_chunks(batch, opts);
        const int chunk = *std::max_element(chunks.begin(), chunks.end());
        const int inner = auto_chunk(n, d->fp64, chunk, nullptr, 2, d->slot_scr[1].bytes);
        gtd_mc_opts o = to_dev_opts(opts);
        d->var_scratch.ensure(gtd_var_scratch_bytes_per_sample(n, d->fp64) * chunk);
        for (int s = 0; s < 2; ++s) {
            if (!d->slot_stream[s]) cuda_ok(cudaStreamCreateWithFlags(&d->slot_stream[s], cudaStreamNonBlocking), "stream");
            d->slot_in[s].ensure(2 * map * chunk);
            d->slot_seeds[s].ensure(sizeof(unsigned long long) * chunk);
            if (t_out) d->slot_out[s].ensure(map * chunk);
            d->slot_scr[s].ensure(gtd_mc_scratch_bytes_per_sample(n, d->fp64) * inner);
            d->slot_stats[s].ensure(sizeof(gtd_sample_stats) * chunk);
        }
        const size_t hs_bytes = sizeof(gtd_sample_stats) * static_cast<size_t>(batch);
        if (d->host_stats_bytes < hs_bytes) {
            if (d->host_stats) cudaFreeHost(d->host_stats);
            d->host_stats = nullptr;
            d->host_stats_bytes = 0;
            cuda_ok(cudaMallocHost(&d->host_stats, hs_bytes), "cudaMallocHost");
            d->host_stats_bytes = hs_bytes;
        }
        auto* hs = static_cast<gtd_sample_stats*>(d->host_stats);
        const char* P = static_cast<const char*>(p_dyn);
        // the variation scratch is shared by both slots: serialise generation across slots with an event
        cudaEvent_t gen_done[2];
        for (auto& e : gen_done) cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        for (auto& ss : d->slot_stream) d->order_in(ss);
        for (int s0 = 0, k = 0; k < static_cast<int>(chunks.size()); s0 += chunks[k], ++k) {
            const int cnt = chunks[k];
            const int s = k & 1;
            cudaStream_t st = d->slot_stream[s];
            char* din = static_cast<char*>(d->slot_in[s].p);
            cuda_ok(cudaMemcpyAsync(din, P + s0 * map, cnt * map, cudaMemcpyHostToDevice, st), "h2d p");
            cuda_ok(cudaMemcpyAsync(d->slot_seeds[s].p, seeds + s0, sizeof(unsigned long long) * cnt,
                                    cudaMemcpyHostToDevice, st),
                    "h2d seeds");
            if (k > 0) cuda_ok(cudaStreamWaitEvent(st, gen_done[s ^ 1], 0), "wait");
            cuda_ok(gtd_var_generate(&d->d, d->var_sqlam.p, static_cast<const unsigned long long*>(d->slot_seeds[s].p),
                                     cnt, d->var_sigma, din + chunk * map, d->var_scratch.p, cnt, st),
                    "variation generation");
            cuda_ok(cudaEventRecord(gen_done[s], st), "record");
            gtd_mc_in in{};
            in.P = din;
            in.N = din;
            in.V = din + chunk * map;
            in.sP = in.sN = in.sV = static_cast<long long>(n) * n;
            in.nom_scale = opts ? opts->leak_frac : 0.3;
            auto* dst = static_cast<gtd_sample_stats*>(d->slot_stats[s].p);
            o.resolve = attach_resolve(d, 1 + s, chunk, opts);
            cuda_ok(gtd_mc_batch(&d->d, &in, cnt, &o, t_out ? d->slot_out[s].p : nullptr, dst, d->slot_scr[s].p,
                                 std::min(inner, cnt), st, nullptr, nullptr),
                    "mc batch launch");
            d->kernels += gtd_mc_launch_count(cnt, std::min(inner, cnt)) + 2 +
                          (o.resolve ? gtd_mc_resolve_launch_count() : 0);
            if (t_out)
                cuda_ok(cudaMemcpyAsync(static_cast<char*>(t_out) + s0 * map, d->slot_out[s].p, cnt * map,
                                        cudaMemcpyDeviceToHost, st),
                        "d2h maps");
            cuda_ok(cudaMemcpyAsync(hs + s0, dst, sizeof(gtd_sample_stats) * cnt, cudaMemcpyDeviceToHost, st), "d2h stats");
        }
        for (auto& st : d->slot_stream) cuda_ok(cudaStreamSynchronize(st), "batch sync");
        for (auto& e : gen_done) cudaEventDestroy(e);
        for (int i = 0; i < batch; ++i) {
            if (max_out) max_out[i] = hs[i].max_rise;
            if (mean_out) mean_out[i] = hs[i].mean_rise;
            if (status_out) status_out[i] = hs[i].status;
        }
        if (online_ms) *online_ms = ms_since(t0);
    });
}

void gt_fp_opts_default(gt_fp_opts* o) {
    o->leak_frac = 0.3;
    o->law = 1;
    o->kirchhoff = 1;
    o->beta = 0.017;
    o->t_ambient = 318.15;
    o->eta = 1.3;
    o->tol = 1e-4;
    o->max_iters = 50;
    o->chunk = 0;
    o->fp32_stage_tol = 0.0;
    o->with_rand = 0;
    o->accel = 0;
    o->warm_start = 0;
}

size_t gt_fp_scratch_bytes(int n, int precision) { return gtd_fp_scratch_bytes_per_sample(n, precision == GT_FP64); }

namespace {
void run_fp_stage(gt_device_greens* d, const void* p_dyn, const void* var, int batch, const gt_fp_opts* opts,
                  double tol, int warm, const void* H, void* t_out, int* iters, int* status, double* mx, double* mean,
                  cudaStream_t st, const void* lm_src = nullptr);

// Per-sample shift-variant maps h = f_rand o p_var * rand_scale of the combined config-2
// loop: the mode-A passes with with_rand = 2 (closed forms at gs.mu as the reference
// monte_carlo, the fp64 re-solve for ill-conditioned fp32 pairs). Their per-sample status
// (bad inputs, random_greens runaway) lands in d->fp_hstats.
void shift_variant_maps(gt_device_greens* d, const void* p_dyn, const void* var, int batch, double leak_frac,
                        void* H, cudaStream_t st) {
    const int n = d->d.n;
    const int chunk = auto_chunk(n, d->fp64, batch, nullptr, 1, d->scratch.bytes);
    d->scratch.ensure(gtd_mc_scratch_bytes_per_sample(n, d->fp64) * chunk);
    d->fp_hstats.ensure(sizeof(gtd_sample_stats) * batch);
    gtd_mc_opts o{};
    o.mu_per_sample = 0;
    o.with_rand = 2;
    o.exponent_cap = 6.0;
    o.resolve = attach_resolve(d, 0, batch, nullptr);
    gtd_mc_in in{};
    in.P = p_dyn;
    in.N = p_dyn;
    in.V = var;
    in.sP = in.sN = in.sV = static_cast<long long>(n) * n;
    in.nom_scale = leak_frac;
    cuda_ok(gtd_mc_batch(&d->d, &in, batch, &o, H, d->fp_hstats.as<gtd_sample_stats>(), d->scratch.p, chunk, st,
                         nullptr, nullptr),
            "shift-variant maps");
    d->kernels += gtd_mc_launch_count(batch, chunk) + (o.resolve ? gtd_mc_resolve_launch_count() : 0);
}

gt_device_greens* fp64_twin(gt_device_greens* d) {
    if (!d->dev64) d->dev64 = gth::prepare_device(d->host, GT_FP64, d->device);
    return d->dev64.get();
}

void run_fp(gt_device_greens* d, const void* p_dyn, const void* var, int batch, const gt_fp_opts* opts, void* t_out,
            int* iters, int* status, double* mx, double* mean, cudaStream_t st) {
    if (!opts) fail(ST_CONFIG, "capi", "fixed point needs options");
    if (!(opts->tol > 0.0)) fail(ST_CONFIG, "oracle", "outer tolerance must be positive");
    // default hand-over: the fp32 noise floor for Picard / Chebyshev (tools/fp_stage_sweep.py); with the
    // low-mode mixing the fp64 stage continues the history, and an earlier hand-over (1e-2 K) costs
    // fewer iterations in total (profiles/r2s4_notes.md)
    const double stage_tol = opts->fp32_stage_tol == 0.0 ? (opts->accel < 0 ? 1e-2 : 5e-4) : opts->fp32_stage_tol;
    const size_t nn = static_cast<size_t>(d->d.n) * d->d.n, cnt = nn * batch;
    const void* H = nullptr;
    if (opts->with_rand) {
        d->fp_h.ensure(cnt * (d->fp64 ? 8 : 4));
        d->order_in(st);
        shift_variant_maps(d, p_dyn, var, batch, opts->leak_frac, d->fp_h.p, st);
        H = d->fp_h.p;
    }
    auto or_mode_a_status = [&] {
        if (opts->with_rand)
            cuda_ok(gtd_fp_or_status(status, d->fp_hstats.as<gtd_sample_stats>(), batch, st), "status");
    };
    if (d->fp64 || stage_tol < 0.0 || opts->tol >= stage_tol) {
        run_fp_stage(d, p_dyn, var, batch, opts, opts->tol, opts->warm_start, H, t_out, iters, status, mx, mean, st);
        or_mode_a_status();
        return;
    }
    // "fp32 with fp64 residual check" (BASELINE config 1): the fp32 iteration runs to its
    // noise floor (stage_tol), then fp64 iterations warm-started from that iterate finish the
    // reference stop rule max|dT| < tol (fdm.cpp:190-200) on the fp64 fixed point.
    run_fp_stage(d, p_dyn, var, batch, opts, stage_tol, opts->warm_start, H, t_out, iters, status, nullptr, nullptr,
                 st);
    gt_device_greens* d64 = fp64_twin(d);
    if (H) {
        d->fin_h.ensure(cnt * 8);
        cuda_ok(gtd_widen(static_cast<const float*>(H), d->fin_h.as<double>(), cnt, st), "widen");
    }
    d->fin_p.ensure(cnt * 8);
    d->fin_v.ensure(cnt * 8);
    d->fin_t.ensure(cnt * 8);
    d->fin_it.ensure(sizeof(int) * batch);
    d->fin_st.ensure(sizeof(int) * batch);
    cuda_ok(gtd_widen(static_cast<const float*>(p_dyn), d->fin_p.as<double>(), cnt, st), "widen");
    cuda_ok(gtd_widen(static_cast<const float*>(var), d->fin_v.as<double>(), cnt, st), "widen");
    cuda_ok(gtd_widen(static_cast<const float*>(t_out), d->fin_t.as<double>(), cnt, st), "widen");
    run_fp_stage(d64, d->fin_p.p, d->fin_v.p, batch, opts, opts->tol, 2, H ? d->fin_h.p : nullptr, d->fin_t.p,
                 d->fin_it.as<int>(), d->fin_st.as<int>(), mx, mean, st, opts->accel < 0 ? d->fp_lm.p : nullptr);
    cuda_ok(gtd_narrow(d->fin_t.as<double>(), static_cast<float*>(t_out), cnt, st), "narrow");
    cuda_ok(gtd_fp_combine(iters, status, d->fin_it.as<int>(), d->fin_st.as<int>(), batch, opts->max_iters, st),
            "combine");
    or_mode_a_status();
    d->kernels += 5 + d64->kernels;
    d64->kernels = 0;
}

void run_fp_stage(gt_device_greens* d, const void* p_dyn, const void* var, int batch, const gt_fp_opts* opts,
                  double tol, int warm, const void* H, void* t_out, int* iters, int* status, double* mx, double* mean,
                  cudaStream_t st, const void* lm_src) {
    if (!(opts->tol > 0.0)) fail(ST_CONFIG, "oracle", "outer tolerance must be positive");
    if (opts->max_iters < 1) fail(ST_CONFIG, "oracle", "max_iters must be >= 1");
    const int n = d->d.n;
    int chunk = opts->chunk > 0 ? std::min(opts->chunk, batch) : 0;
    if (!chunk) {
        const size_t per = gtd_fp_scratch_bytes_per_sample(n, d->fp64);
        const int want = std::min(1024, batch);
        // a repeated call whose scratch is already allocated skips the free-memory query
        chunk = d->fp_scratch.bytes >= per * static_cast<size_t>(want)
                    ? want
                    : static_cast<int>(std::max<size_t>(1, std::min<size_t>(1024, scratch_budget() / per)));
        chunk = std::min(chunk, batch);
    }
    d->fp_scratch.ensure(gtd_fp_scratch_bytes_per_sample(n, d->fp64) * chunk);
    d->fp_state.ensure(gtd_fp_state_bytes() * batch);
    d->fp_counter.ensure(sizeof(int));
    if (!d->fp_counter_h) cuda_ok(cudaMallocHost(reinterpret_cast<void**>(&d->fp_counter_h), sizeof(int)), "pinned");
    gtd_mc_in in{};
    in.P = p_dyn;
    in.N = p_dyn;
    in.V = var;
    in.sP = in.sN = in.sV = static_cast<long long>(n) * n;
    in.nom_scale = opts->leak_frac;
    gtd_fp_opts o{};
    o.law = opts->law;
    o.kirchhoff = opts->kirchhoff;
    o.beta = opts->beta;
    o.t_ambient = opts->t_ambient;
    o.eta = opts->eta;
    o.tol = tol;
    o.max_iters = opts->max_iters;
    o.poll = 4;
    o.warm_start = warm ? 1 : 0;
    o.min_iters = warm == 2 ? 1 : 2;  // 2: the fp64 stage continuing an fp32 iteration (run_fp)
    o.H = H;
    o.sH = static_cast<long long>(n) * n;
    o.accel = opts->accel;
    o.Tprev = o.Yout = nullptr;
    o.lm_state = nullptr;
    o.lm_cos = nullptr;
    if (o.accel < 0) {
        if (o.accel < -4) fail(ST_CONFIG, "oracle", "accel < 0 selects Anderson(m) on the low modes, m = -accel <= 4");
        d->fp_lm.ensure(gtd_fp_lowmode_bytes() * batch);
        const size_t cb = sizeof(double) * 16 * n;
        if (d->fp_lmcos.bytes < cb) {
            d->fp_lmcos.ensure(cb);
            cuda_ok(gtd_fp_lowmode_cos(n, d->fp_lmcos.as<double>(), st), "low-mode cosine table");
        }
        o.lm_state = d->fp_lm.p;
        o.lm_cos = d->fp_lmcos.as<double>();
        if (lm_src) {  // the fp64 stage continues the fp32 stage's mixing history (fp64 coefficients)
            cuda_ok(cudaMemcpyAsync(d->fp_lm.p, lm_src, gtd_fp_lowmode_bytes() * batch, cudaMemcpyDeviceToDevice, st),
                    "low-mode state");
            o.lm_keep = 1;
        }
    }
    if (o.accel > 0) {
        d->fp_tprev.ensure(static_cast<size_t>(n) * n * batch * (d->fp64 ? 8 : 4));
        d->fp_yout.ensure(static_cast<size_t>(n) * n * batch * (d->fp64 ? 8 : 4));
        o.Tprev = d->fp_tprev.p;
        o.Yout = d->fp_yout.p;
    }
    long long launches = 0;
    d->order_in(st);
    cuda_ok(gtd_fp_batch(&d->d, &in, batch, &o, t_out, iters, status, mx, mean, d->fp_scratch.p, d->fp_state.p,
                         d->fp_counter.as<int>(), d->fp_counter_h, chunk, st, &launches),
            "fixed point");
    d->order_out(st);
    d->kernels += launches;
    d->calls += 1;
}
}  // namespace

namespace {
gtd_lg large_geom(const gt_device_greens* d) {
    if (!d) fail(ST_CONFIG, "capi", "null device GreensSet");
    if (!d->fp64) fail(ST_CONFIG, "device", "the large-grid path runs in fp64: prepare the GreensSet with GT_FP64");
    gtd_lg g{};
    g.n = d->d.n;
    g.m = d->d.m;
    if (gtd_lg_split(g.m, &g.M1, &g.M2))
        fail(ST_CONFIG, "device", "the large-grid path needs a power-of-two grid with m = 2n in [1024, 262144]");
    g.tw = d->tw64.p;
    g.fk = d->fk.p;
    g.fkp = d->d.hp;
    g.hs = d->hs.p;
    return g;
}
}  // namespace

gt_status gt_large_geometry(const gt_device_greens* d, int* m1, int* m2) {
    return guarded([&] {
        const gtd_lg g = large_geom(d);
        if (m1) *m1 = g.M1;
        if (m2) *m2 = g.M2;
    });
}

gt_status gt_large_row_layout(const gt_device_greens* d, int* dct_rows) {
    return guarded([&] {
        const gtd_lg g = large_geom(d);
        if (dct_rows) *dct_rows = gtd_lg_row_layout(&g);
    });
}

size_t gt_large_lowmode_state_bytes(void) { return gtd_lg_lowmode_state_bytes(); }
int gt_large_lowmode_partial_blocks(int rows) { return gtd_lg_lowmode_partial_blocks(rows); }

gt_status gt_large_lowmode_init(void* state, void* stream) {
    return guarded([&] {
        if (!state) fail(ST_CONFIG, "capi", "large lowmode: null state");
        cuda_ok(gtd_lg_lowmode_init(state, static_cast<cudaStream_t>(stream)), "large lowmode init");
    });
}

gt_status gt_large_lowmode_project(const gt_device_greens* d, const void* y, int hy, int rows, int row0,
                                   double* partial, double* coef, void* stream) {
    return guarded([&] {
        const gtd_lg g = large_geom(d);
        if (!y || !partial || !coef || rows < 1 || row0 < 0 || row0 + rows > g.n || hy < 16)
            fail(ST_CONFIG, "capi", "large lowmode project: bad row range or buffers");
        cuda_ok(gtd_lg_lowmode_project(&g, y, hy, rows, row0, partial, coef, static_cast<cudaStream_t>(stream)),
                "large lowmode project");
    });
}

gt_status gt_large_lowmode_mix(void* state, const double* coef, int depth, double res_prev, double* corr,
                               void* stream) {
    return guarded([&] {
        if (!state || !coef || !corr) fail(ST_CONFIG, "capi", "large lowmode mix: null buffer");
        if (depth < 1 || depth > 4) fail(ST_CONFIG, "capi", "large lowmode mix: depth must be 1..4");
        cuda_ok(gtd_lg_lowmode_mix(state, coef, depth, res_prev, corr, static_cast<cudaStream_t>(stream)),
                "large lowmode mix");
    });
}

gt_status gt_large_lowmode_apply(const gt_device_greens* d, void* y, int hy, int rows, int row0, const double* corr,
                                 void* stream) {
    return guarded([&] {
        const gtd_lg g = large_geom(d);
        if (!y || !corr || rows < 1 || row0 < 0 || row0 + rows > g.n || hy < 16)
            fail(ST_CONFIG, "capi", "large lowmode apply: bad row range or buffers");
        cuda_ok(gtd_lg_lowmode_apply(&g, y, hy, rows, row0, corr, static_cast<cudaStream_t>(stream)),
                "large lowmode apply");
    });
}

gt_status gt_large_rows_fwd(const gt_device_greens* d, const double* app, int pairs, void* s1, void* z,
                            void* stream) {
    return guarded([&] {
        const gtd_lg g = large_geom(d);
        cuda_ok(gtd_lg_rows_fwd(&g, app, pairs, s1, z, static_cast<cudaStream_t>(stream)), "large rows fwd");
    });
}

gt_status gt_large_cols(const gt_device_greens* d, const void* z, int compact, int c0, int hc, void* c1, void* c2,
                        void* y, void* stream) {
    return guarded([&] {
        const gtd_lg g = large_geom(d);
        if (c0 < 0 || hc < 1 || c0 + hc > g.n + 1) fail(ST_CONFIG, "capi", "column range outside [0, n]");
        cuda_ok(gtd_lg_cols(&g, z, compact, c0, hc, c1, c2, y, static_cast<cudaStream_t>(stream)), "large cols");
    });
}

gt_status gt_large_cols_peer(const gt_device_greens* d, const void* z_ranks, int world, int pairs_per_rank, int c0,
                             int hc, void* c1, void* c2, const void* y_ranks, int hy, void* stream) {
    return guarded([&] {
        const gtd_lg g = large_geom(d);
        if (world < 1 || pairs_per_rank < 1 || world * pairs_per_rank * 2 != g.n)
            fail(ST_CONFIG, "capi", "large cols_peer: world * pairs_per_rank must be n / 2");
        if (c0 < 0 || hc < 1 || c0 + hc > g.n + 1) fail(ST_CONFIG, "capi", "column range outside [0, n]");
        if (hy < g.n + 1) fail(ST_CONFIG, "capi", "large cols_peer: row buffers need n + 1 columns");
        if (!z_ranks || !y_ranks) fail(ST_CONFIG, "capi", "large cols_peer: null rank table");
        cuda_ok(gtd_lg_cols_peer(&g, static_cast<const void* const*>(z_ranks), pairs_per_rank, c0, hc, c1, c2,
                                 const_cast<void* const*>(static_cast<const void* const*>(y_ranks)), hy,
                                 static_cast<cudaStream_t>(stream)),
                "large cols peer");
    });
}

/* CUDA IPC for the peer-memory exchange: a cudaMalloc'ed buffer (base == pointer, so the
 * handle maps the buffer itself) and its 64-byte handle; another process opens it with
 * peer access enabled. */
gt_status gt_ipc_alloc(size_t bytes, void** ptr, void* handle64) {
    return guarded([&] {
        if (!ptr || !handle64 || bytes == 0) fail(ST_CONFIG, "capi", "gt_ipc_alloc: bad arguments");
        void* p = nullptr;
        cuda_ok(static_cast<int>(cudaMalloc(&p, bytes)), "ipc alloc");
        cudaIpcMemHandle_t h;
        const cudaError_t e = cudaIpcGetMemHandle(&h, p);
        if (e != cudaSuccess) {
            cudaFree(p);
            cuda_ok(static_cast<int>(e), "ipc handle");
        }
        std::memcpy(handle64, &h, sizeof(h));
        *ptr = p;
    });
}

gt_status gt_ipc_open(const void* handle64, void** ptr) {
    return guarded([&] {
        if (!ptr || !handle64) fail(ST_CONFIG, "capi", "gt_ipc_open: bad arguments");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle64, sizeof(h));
        cuda_ok(static_cast<int>(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess)), "ipc open");
    });
}

gt_status gt_ipc_close(void* ptr) {
    return guarded([&] { cuda_ok(static_cast<int>(cudaIpcCloseMemHandle(ptr)), "ipc close"); });
}

gt_status gt_ipc_free(void* ptr) {
    return guarded([&] { cuda_ok(static_cast<int>(cudaFree(ptr)), "ipc free"); });
}

gt_status gt_large_rows_inv(const gt_device_greens* d, const void* y, int hy, int pairs, void* s1, double* t,
                            double* app, const double* p, const double* l0, const gt_fp_opts* opts,
                            unsigned long long* res_bits, int* status, void* stream) {
    return gt_large_rows_inv_accel(d, y, hy, pairs, s1, t, app, p, l0, opts, res_bits, status, nullptr, nullptr,
                                   0.0, 1.0, stream);
}

gt_status gt_large_rows_inv_accel(const gt_device_greens* d, const void* y, int hy, int pairs, void* s1, double* t,
                                  double* app, const double* p, const double* l0, const gt_fp_opts* opts,
                                  unsigned long long* res_bits, int* status, double* x_prev, double* g_out,
                                  double omega, double gamma, void* stream) {
    return guarded([&] {
        if (omega > 0.0 && !x_prev) fail(ST_CONFIG, "capi", "large rows_inv: a Chebyshev step needs x_prev");
        if (!opts) fail(ST_CONFIG, "capi", "large rows_inv needs fixed-point options");
        const gtd_lg g = large_geom(d);
        gtd_fp_opts o{};
        o.law = opts->law;
        o.kirchhoff = opts->kirchhoff;
        o.beta = opts->beta;
        o.t_ambient = opts->t_ambient;
        o.eta = opts->eta;
        cuda_ok(gtd_lg_rows_inv(&g, y, hy, pairs, s1, t, app, p, l0, &o, res_bits, status, x_prev, g_out, omega,
                                gamma, static_cast<cudaStream_t>(stream)),
                "large rows inv");
    });
}

void gt_trace_opts_default(gt_trace_opts* o) {
    if (!o) return;
    o->dt = 1e-5;
    o->steps = 2000;
    o->window = 0;
    o->law = 0;
    o->beta = 0.017;
    o->out_stride = 100;
    o->chunk = 0;
}

size_t gt_trace_scratch_bytes(int n, int precision, int window) {
    return gtd_trace_bytes_per_trace(n, precision == GT_FP64, window);
}

gt_status gt_trace_batch_device(const gt_device_greens* dc, const int* blk, long long blk_stride, const void* sched,
                                int nblk, const void* leak0, long long leak_stride, int batch,
                                const gt_trace_opts* opts, void* t_out, double* max_out, void* stream) {
    return guarded([&] {
        if (!dc || !opts || batch < 1 || !blk || !sched || !leak0 || !t_out || nblk < 1)
            fail(ST_CONFIG, "capi", "trace batch needs block maps, schedule, leakage base and an output buffer");
        if (!(opts->dt > 0.0)) fail(ST_CONFIG, "solver", "power trace dt must be positive");
        if (opts->steps < 1) fail(ST_CONFIG, "solver", "power trace is empty");
        if (opts->out_stride < 1 || opts->out_stride > opts->steps)
            fail(ST_CONFIG, "capi", "out_stride must be in [1, steps]");
        if (opts->law != 0 && opts->law != 1) fail(ST_CONFIG, "capi", "law must be 0 (linear) or 1 (exp)");
        auto* d = const_cast<gt_device_greens*>(dc);
        std::lock_guard<std::mutex> lk(d->mu);
        const Greens& g = d->host;
        if (!(g.capacitance > 0.0)) fail(ST_SOLVER, "solver", "GreensSet has no fitted capacitance");
        const int n = g.n, m = 2 * n;
        if (gtd_trace_pitch(n, d->fp64) < 0) fail(ST_CONFIG, "device", "trace batch supports n = 32..1024");
        int k = opts->window > 0 ? opts->window : static_cast<int>(std::ceil(0.005 / opts->dt));  // solver.cpp:224-226
        k = std::max(1, std::min(k, opts->steps));
        cuda_ok(cudaSetDevice(d->device), "cudaSetDevice");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->stream;
        // fp64 spectra exactly as gt_solve_trace: F_det at the set's mu, r = exp(-dt/tau), r^(k+1)
        auto d64 = prepare_device(g, GT_FP64, d->device);
        cudaStream_t s64 = d64->stream;
        const size_t mm = static_cast<size_t>(m) * m;
        DBuf Fd, r, rk, flag, red;
        Fd.ensure(mm * 16);
        r.ensure(mm * 16);
        rk.ensure(mm * 16);
        flag.ensure(sizeof(int) * 4);
        red.ensure(sizeof(double) * 8);
        cuda_ok(cudaMemsetAsync(flag.p, 0, sizeof(int) * 4, s64), "memset");
        cuda_ok(gtd_fdet_full(d64->fk_full.p, d64->gtab.as<double>(), n, d64->d.hp, g.alpha, g.beta, g.mu, Fd.p,
                              flag.as<int>(), s64),
                "fdet");
        double fk3[3];
        cuda_ok(gtd_creduce(d64->fk_full.p, mm, red.as<double>(), s64), "creduce");
        cuda_ok(cudaMemcpyAsync(fk3, red.p, sizeof fk3, cudaMemcpyDeviceToHost, s64), "d2h");
        int fl = 0;
        cuda_ok(cudaMemcpyAsync(&fl, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s64), "d2h");
        cuda_ok(cudaStreamSynchronize(s64), "sync");
        if (fl & GTD_ST_RUNAWAY_DET)
            fail(ST_SOLVER, "greens",
                 "deterministic_greens: spectral denominator collapsed below 1e-6 (leakage feedback gain reached unity)");
        cuda_ok(cudaMemsetAsync(flag.p, 0, sizeof(int), s64), "memset");
        cuda_ok(gtd_transient(d64->fk_full.p, d64->gtab.as<double>(), Fd.p, n, d64->d.hp, g.alpha, g.capacitance,
                              1e-6 * fk3[2], 0.0, nullptr, opts->dt, k, r.p, rk.p, flag.as<int>(), s64),
                "transient");
        cuda_ok(cudaMemcpyAsync(&fl, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s64), "d2h");
        cuda_ok(cudaStreamSynchronize(s64), "sync");
        if (fl & 1) fail(ST_SOLVER, "solver", "non-positive transient time constant");
        d->order_in(s64);  // an earlier call's traces may still read the tables
        d->trace_tab.ensure(gtd_trace_table_bytes(n, d->fp64));
        cuda_ok(gtd_trace_tables(&d->d, Fd.p, r.p, rk.p, d->trace_tab.p, s64), "trace tables");
        cuda_ok(cudaStreamSynchronize(s64), "sync");
        // traces in flight: the power ring is (k + 2) maps per trace; up to 60% of free memory
        const size_t per = gtd_trace_bytes_per_trace(n, d->fp64, k);
        int chunk = opts->chunk > 0 ? std::min(opts->chunk, batch) : 0;
        if (!chunk) {
            size_t fr = 0, tot = 0;
            cuda_ok(cudaMemGetInfo(&fr, &tot), "meminfo");
            fr += d->trace_scratch.bytes;
            const int fit = static_cast<int>(std::max<size_t>(1, std::min<size_t>(batch, (fr / 10 * 6) / per)));
            // balanced chunks: 64 traces that fit 62 at a time run as 32 + 32, not 62 + 2
            const int nchunks = (batch + fit - 1) / fit;
            chunk = (batch + nchunks - 1) / nchunks;
        }
        d->trace_scratch.ensure(per * chunk);
        gtd_trace_in in{blk, blk_stride, sched, nblk, opts->steps, leak0, leak_stride};
        gtd_trace_opts o{k, opts->law, opts->beta, opts->out_stride};
        long long launches = 0;
        d->order_in(st);
        cuda_ok(gtd_trace_batch(&d->d, d->trace_tab.p, &in, batch, &o, t_out, max_out, d->trace_scratch.p, chunk, st,
                                &launches),
                "trace batch");
        d->order_out(st);
        d->kernels += launches;
        d->calls += 1;
    });
}

gt_status gt_fp_batch_device(const gt_device_greens* dc, const void* p_dyn, const void* var, int batch,
                             const gt_fp_opts* opts, void* t_out, int* iters_out, int* status_out, double* max_out,
                             double* mean_out, void* stream) {
    return guarded([&] {
        if (batch < 1 || !p_dyn || !var || !t_out || !iters_out || !status_out)
            fail(ST_CONFIG, "capi", "fixed point needs inputs, t_out, iters and status arrays");
        auto* d = const_cast<gt_device_greens*>(dc);
        std::lock_guard<std::mutex> lk(d->mu);
        cuda_ok(cudaSetDevice(d->device), "cudaSetDevice");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->stream;
        run_fp(d, p_dyn, var, batch, opts, t_out, iters_out, status_out, max_out, mean_out, st);
    });
}

gt_status gt_fp_batch(const gt_device_greens* dc, const void* p_dyn, const void* var, int batch,
                      const gt_fp_opts* opts, void* t_out, int* iters_out, int* status_out, double* max_out,
                      double* online_ms) {
    return guarded([&] {
        if (batch < 1 || !p_dyn || !var) fail(ST_CONFIG, "capi", "fixed point needs inputs");
        auto t0 = wall::now();
        auto* d = const_cast<gt_device_greens*>(dc);
        std::lock_guard<std::mutex> lk(d->mu);
        cuda_ok(cudaSetDevice(d->device), "cudaSetDevice");
        const int n = d->d.n;
        const size_t es = d->fp64 ? 8 : 4, map = static_cast<size_t>(n) * n * es;
        DBuf P, V, T, it, st, mx;
        P.ensure(map * batch);
        V.ensure(map * batch);
        T.ensure(map * batch);
        it.ensure(sizeof(int) * batch);
        st.ensure(sizeof(int) * batch);
        mx.ensure(sizeof(double) * batch);
        cudaStream_t s = d->stream;
        cuda_ok(cudaMemcpyAsync(P.p, p_dyn, map * batch, cudaMemcpyHostToDevice, s), "h2d");
        cuda_ok(cudaMemcpyAsync(V.p, var, map * batch, cudaMemcpyHostToDevice, s), "h2d");
        if (opts && opts->warm_start) {
            if (!t_out) fail(ST_CONFIG, "capi", "warm_start needs the initial maps in t_out");
            cuda_ok(cudaMemcpyAsync(T.p, t_out, map * batch, cudaMemcpyHostToDevice, s), "h2d");
        }
        run_fp(d, P.p, V.p, batch, opts, T.p, it.as<int>(), st.as<int>(), mx.as<double>(), nullptr, s);
        if (t_out) cuda_ok(cudaMemcpyAsync(t_out, T.p, map * batch, cudaMemcpyDeviceToHost, s), "d2h");
        if (iters_out) cuda_ok(cudaMemcpyAsync(iters_out, it.p, sizeof(int) * batch, cudaMemcpyDeviceToHost, s), "d2h");
        if (status_out) cuda_ok(cudaMemcpyAsync(status_out, st.p, sizeof(int) * batch, cudaMemcpyDeviceToHost, s), "d2h");
        if (max_out) cuda_ok(cudaMemcpyAsync(max_out, mx.p, sizeof(double) * batch, cudaMemcpyDeviceToHost, s), "d2h");
        cuda_ok(cudaStreamSynchronize(s), "sync");
        if (online_ms) *online_ms = ms_since(t0);
    });
}

gt_status gt_profile_begin(gt_device_greens* d) { return gt_profile_begin_mode(d, 0); }

gt_status gt_profile_begin_mode(gt_device_greens* d, int mode) {
    return guarded([&] {
        if (mode != 0 && mode != 1) fail(ST_CONFIG, "profile", "profile mode must be 0 or 1");
        std::lock_guard<std::mutex> lk(d->mu);
        d->profiling = true;
        d->profile_mode = mode;
        d->marks.clear();
        d->pool_used = 0;
        d->kernels = 0;
        d->calls = 0;
    });
}

gt_status gt_profile_end(gt_device_greens* d, double* pass_ms, long long* kernels, long long* calls) {
    return guarded([&] {
        std::lock_guard<std::mutex> lk(d->mu);
        cuda_ok(cudaSetDevice(d->device), "cudaSetDevice");
        double acc[4] = {0, 0, 0, 0};
        if (d->profile_mode == 1) {
            for (size_t i = 0; i + 1 < d->marks.size(); i += 2) {
                if (d->marks[i].first != 1 || d->marks[i + 1].first != 2)
                    fail(ST_INTERNAL, "profile", "unbalanced profiling marks");
                cuda_ok(cudaEventSynchronize(d->marks[i + 1].second), "event sync");
                float ms = 0.f;
                cuda_ok(cudaEventElapsedTime(&ms, d->marks[i].second, d->marks[i + 1].second), "elapsed");
                acc[1] += ms;
            }
        }
        for (size_t i = 0; d->profile_mode == 0 && i + 3 < d->marks.size(); i += 4) {
            for (int k = 0; k < 3; ++k) {
                if (d->marks[i + k].first != k || d->marks[i + k + 1].first != k + 1)
                    fail(ST_INTERNAL, "profile", "unbalanced profiling marks");
                cuda_ok(cudaEventSynchronize(d->marks[i + k + 1].second), "event sync");
                float ms = 0.f;
                cuda_ok(cudaEventElapsedTime(&ms, d->marks[i + k].second, d->marks[i + k + 1].second), "elapsed");
                acc[k] += ms;
            }
        }
        acc[3] = acc[0] + acc[1] + acc[2];
        if (pass_ms)
            for (int k = 0; k < 4; ++k) pass_ms[k] = acc[k];
        if (kernels) *kernels = d->kernels;
        if (calls) *calls = d->calls;
        d->profiling = false;
        d->profile_mode = 0;
        d->marks.clear();
        d->pool_used = 0;
    });
}

long long gt_kernel_launches(const gt_device_greens* d) { return d->kernels; }

}  // extern "C"
