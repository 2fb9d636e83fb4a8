// devctx.hpp — device-side context shared by the C-ABI entry points: RAII
// device buffers, error mapping and the prepared, device-resident GreensSet
// (the reference's PreparedGreens, solver.cpp:113-121, plus the per-frequency
// tables the kernels read).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/greentherm_b200.h"
#include "gt_device.h"
#include "host.hpp"

namespace gth {

void cuda_ok(cudaError_t e, const char* what);
inline void cuda_ok(int e, const char* what) { cuda_ok(static_cast<cudaError_t>(e), what); }
void need_device();
inline bool pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

// RAII device buffer.
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    void ensure(size_t b);
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

void upload(DBuf& b, const void* src, size_t bytes, cudaStream_t st);

}  // namespace gth

struct gt_device_greens {
    // fp64 full-spectrum tables for the reference-API solves (steady/step/trace)
    gth::DBuf fk_full;  // [m][m] double2: baseline kernel spectrum incl. DC term
    int device = 0;
    int fp64 = 0;
    gtd_greens d{};
    gth::Greens host;  // copy of the set the tables were built from
    cudaStream_t stream = nullptr;
    gth::DBuf hs, fg, fgm, fk, gtab, k1, tw, tw64, fsp0, gsp0, work;
    // batch scratch (guarded by mu)
    std::mutex mu;
    gth::DBuf fp_scratch, fp_state, fp_counter;
    gth::DBuf fin_p, fin_v, fin_t, fin_it, fin_st, fin_h;  // fp64 finish stage of an fp32 fixed point
    gth::DBuf fp_h, fp_hstats;  // shift-variant maps of the combined config-2 fixed point
    gth::DBuf fp_tprev, fp_yout;  // x_{k-1} and G(x_k) of the Chebyshev-accelerated fixed point
    gth::DBuf fp_lm, fp_lmcos;    // low-mode Anderson state and its cosine table (accel < 0)
    gth::DBuf trace_scratch, trace_tab;
    gth::DBuf var_sqlam, var_scratch, slot_seeds[2];  // seeded variation model (gt_var_model)
    double var_sigma = 0.0;
    int* fp_counter_h = nullptr;
    gth::DBuf scratch, stats, slot_in[2], slot_out[2], slot_scr[2], slot_stats[2];
    cudaStream_t slot_stream[2] = {nullptr, nullptr};
    void* host_stats = nullptr;
    size_t host_stats_bytes = 0;
    // profiling (gt_profile_begin/end): events recorded between pass launches
    bool profiling = false;
    std::vector<std::pair<int, cudaEvent_t>> marks;
    std::vector<cudaEvent_t> event_pool;
    size_t pool_used = 0;
    long long kernels = 0, calls = 0;
    // Successive calls on one handle share its scratch; they may enqueue on
    // different streams, so each call's stream waits for the previous call's work.
    cudaEvent_t busy = nullptr;
    void order_in(cudaStream_t st) {
        if (!busy) cudaEventCreateWithFlags(&busy, cudaEventDisableTiming);
        cudaStreamWaitEvent(st, busy, 0);
    }
    void order_out(cudaStream_t st) {
        if (busy) cudaEventRecord(busy, st);
    }
    // fp64 re-solve of ill-conditioned fp32 Monte-Carlo pairs (gtd_mc_resolve):
    // fp64 tables of the same GreensSet, built on first use, and per-pipeline-slot
    // buffers (0: device-resident entry, 1 / 2: the two host-pipeline slots)
    std::unique_ptr<gt_device_greens> dev64;
    struct Resolve {
        gth::DBuf in, out, stats, scr, sel;
        gtd_mc_resolve d{};
    } resolve[3];
    int profile_mode = 0;  // 1: column pass only (points 1, 2)
    static void mark(void* ctx, int point, cudaStream_t st) {
        auto* self = static_cast<gt_device_greens*>(ctx);
        if (self->profile_mode == 1 && (point == 0 || point == 3)) return;
        if (self->pool_used == self->event_pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            self->event_pool.push_back(e);
        }
        cudaEvent_t e = self->event_pool[self->pool_used++];
        cudaEventRecord(e, st);
        self->marks.emplace_back(point, e);
    }
    ~gt_device_greens() {
        for (auto e : event_pool) cudaEventDestroy(e);
        if (busy) cudaEventDestroy(busy);
        if (host_stats) cudaFreeHost(host_stats);
        if (fp_counter_h) cudaFreeHost(fp_counter_h);
        for (auto& s : slot_stream)
            if (s) cudaStreamDestroy(s);
        if (stream) cudaStreamDestroy(stream);
    }
};


namespace gth {
std::unique_ptr<gt_device_greens> prepare_device(const Greens& g, int precision, int device);
}
