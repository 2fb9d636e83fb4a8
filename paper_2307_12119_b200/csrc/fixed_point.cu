// fixed_point.cu — north-star mode B: the leakage-temperature fixed point
// with the Kirchhoff transform, batched over samples, two fused passes per
// iteration.
//
// Per sample (oracle: oracle/restate.cpp ref_fixed_point_batch; loop
// structure and stop rule of the reference FDM outer loop, fdm.cpp:167-205):
//   theta_{k+1} - T0 = crop(IFFT(fk . FFT(mirror(P + L0 f(T_k)))))
//   L0 = nom_scale * N * V,  f(dT) = exp(beta dT) (law 1) or 1 + beta dT (law 0)
//   T_{k+1} = Kirchhoff inverse of theta for k = k_ref (T/T0)^-eta (kirchhoff=1)
//   stop when max|T_{k+1} - T_k| < tol after iteration 1; max_iters -> error.
//
// Kernels per iteration:
//   fp_cols : per half-spectrum column tile: mirror-expand the row spectra,
//             forward column FFT, multiply by fk, inverse column FFT, keep rows
//             [0, n) -- in place.
//   fp_rows : per block of die-row PAIRS (two real rows share one complex
//             line): inverse row FFT -> theta rows -> Kirchhoff inverse ->
//             residual vs T_k -> T_{k+1} written in place -> next leakage ->
//             forward row FFT of the mirrored applied rows -> row spectra.
//   fp_update: per-sample iteration count / convergence / failure state.
#include <cuda_runtime.h>

#include <type_traits>

#include "launch_once.cuh"
#include "col_pass.cuh"
#include "fft_tile.cuh"
#include "fft_warp.cuh"
#include "gt_device.h"
#include "kirchhoff.cuh"
#include "lowmode.cuh"

#ifndef GT_FP_UB
#define GT_FP_UB 4  // global loads issued ahead per thread in the tile row pass (tuning)
#endif

namespace gtb {
namespace {

template <typename T, int M>
struct FPGeom {
    using G = TileGeom<T, M>;
    static constexpr int n = M / 2;
    static constexpr int h = n + 1;
    static constexpr int L = G::L;
    static constexpr int NT = G::NT;
    static constexpr int hp = ((h + L - 1) / L) * L;  // column tiles of L columns
    // tile pitch: fp32 line pairs are 16-byte loads (even pitch); fp64 pairs are two
    // 16-byte loads, so an odd pitch pads less (M = 2048: 3 instead of 4 lines)
    static constexpr int LP = sizeof(T) == 8 ? L + 1 : L + 2;
    // a twiddle table of >= 32 KB is read from global (L1) so two CTAs fit an SM
    static constexpr bool GTW = M * sizeof(cplx<T>) >= 32768;
    static constexpr int RP = n / 2;                   // die-row pairs
    static constexpr int RB = (RP + L - 1) / L;        // row-pair blocks per sample
    static constexpr int CT = hp / L;                  // column tiles per sample
};

struct FPState {
    unsigned long long res_bits;  // max |T_{k+1} - T_k| of the current iteration (double bits)
    int iters;
    int active;
    double sum_app[2];  // sum of the applied map of iterations k (slot k & 1): shift-variant term
    // Chebyshev acceleration (gtd_fp_opts.accel): x_{k+1} = omega (gamma G(x_k) + (1 - gamma) x_k
    // - x_{k-1}) + x_{k-1}; omega = 0 runs plain Picard (the reference outer loop).
    double res_prev;    // residual of the previous iteration
    double omega, gamma, sigma2;
};

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <typename T>
struct FPIn {
    const T* P;
    const T* N;
    const T* V;
    long long sP, sN, sV;
    T nom_scale;
};

__device__ __forceinline__ void or_flags_fp(int* dst, int flags) {
    const int w = __reduce_or_sync(0xffffffffu, flags);
    if ((threadIdx.x & 31) == 0 && w) atomicOr(dst, w);
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <typename T>
__device__ __forceinline__ bool finite_val(T v) {
    return isfinite(v);
}

// ----------------------------------------------------------------- rows
// Register budget of the tile row pass: the tile engine's 64 (fp32) leaves the M >= 1024
// epilogue (theta -> T, Kirchhoff, shift-variant term, Chebyshev state) spilling; those
// grids take one 512-thread CTA per SM with 128 registers instead (GT_FP_ROWS_MINB).
#ifndef GT_FP_ROWS_MINB
#define GT_FP_ROWS_MINB 0
#endif
template <typename T, int M>
struct FPRowsMinB {
    static constexpr int value = GT_FP_ROWS_MINB > 0 ? GT_FP_ROWS_MINB : TileGeom<T, M>::MINB;
};

// FEAT bit 0: shift-variant maps (H) in use; bit 1: Chebyshev state (Tprev) in use. The
// per-thread register arrays of an unused feature vanish at compile time (FEAT = 0, the plain
// loop and the low-mode mixing: the warp row pass drops its spills at 128 registers, +9% on
// the config-1 loop; profiles/r2s4_notes.md).
template <typename T, int M, bool FIRST, int FEAT>
__global__ void __launch_bounds__(TileGeom<T, M>::NT, FPRowsMinB<T, M>::value)
fp_rows(FPIn<T> in, int sample0, int count, cplx<T>* __restrict__ A, T* __restrict__ Ar, T* __restrict__ Tst,
        FPState* __restrict__ state, int* __restrict__ status, const cplx<T>* __restrict__ g_tw,
        const cplx<T>* __restrict__ g_hs, T beta, int law, int kirchhoff, T ka, T kb, T kexp, T t_ambient,
        int warm, const T* __restrict__ H_, long long sH, int it, T* __restrict__ Tprev_, T* __restrict__ Yout) {
    const T* const H = (FEAT & 1) ? H_ : nullptr;
    T* const Tprev = (FEAT & 2) ? Tprev_ : nullptr;
    using Gm = FPGeom<T, M>;
    constexpr int n = Gm::n, h = Gm::h, L = Gm::L, LP = Gm::LP, NT = Gm::NT, hp = Gm::hp;
    constexpr int RB = Gm::RB;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_tw = tile + M * LP;
    if constexpr (!Gm::GTW) load_twiddles<T, M, NT>(s_tw, g_tw);
    const cplx<T>* tw = Gm::GTW ? g_tw : s_tw;
    const T kc = kb / ka;  // Kirchhoff inverse (kirchhoff.cuh)
    __syncthreads();

    for (int item = blockIdx.x; item < count * RB; item += gridDim.x) {
        const int s = item / RB;
        const int p0 = (item - s * RB) * L;  // first row pair of the block
        const size_t sg = static_cast<size_t>(sample0) + s;
        if (!FIRST && !state[sg].active) continue;
        const T* P = in.P + sg * in.sP;
        const T* Nm = in.N + sg * in.sN;
        const T* V = in.V + sg * in.sV;
        T* Ts = Tst + sg * n * n;
        cplx<T>* As = A + static_cast<size_t>(s) * n * hp;
        constexpr T inv = T(1.0 / (double(M) * double(M)));
        double dmax = 0.0, app_part = 0.0;
        int bad = 0;
        const T sig_prev = (!FIRST && H) ? T(state[sg].sum_app[(it - 1) & 1]) : T(0);
        const double om = (!FIRST && Tprev) ? state[sg].omega : 0.0;  // Chebyshev acceleration
        const T omt = T(om), gmt = T(om > 0.0 ? state[sg].gamma : 1.0);
        T* Qs = Tprev ? Tprev + sg * n * n : nullptr;

        // Every global input of a stage is issued in batches of UB items ahead of
        // its use (one exposed HBM latency per batch, not one per element).
        constexpr int UB = GT_FP_UB;
        if (!FIRST) {
            // pack rows (2p, 2p+1) of the column-pass output into one Hermitian line pair
            constexpr int IPH = (L * h + NT - 1) / NT;
#pragma unroll
            for (int i0 = 0; i0 < IPH; i0 += UB) {
                cplx<T> yv[UB], rv[UB];
#pragma unroll
                for (int u = 0; u < UB; ++u) {
                    const int idx = threadIdx.x + (i0 + u) * NT;
                    const int l = idx / h, v = idx - l * h;
                    const int xa = 2 * (p0 + l);
                    yv[u] = rv[u] = mk<T>(T(0), T(0));
                    if (i0 + u < IPH && idx < L * h && xa < n) {
                        yv[u] = As[static_cast<size_t>(xa) * hp + v];
                        rv[u] = As[static_cast<size_t>(xa + 1) * hp + v];
                    }
                }
#pragma unroll
                for (int u = 0; u < UB; ++u) {
                    const int idx = threadIdx.x + (i0 + u) * NT;
                    if (i0 + u >= IPH || idx >= L * h) continue;
                    const int l = idx / h, v = idx - l * h;
                    const cplx<T> y = yv[u], r = rv[u];
                    if (v == 0 || v == n) {
                        tile[v * LP + l] = mk<T>(y.x, r.x);
                    } else {
                        tile[v * LP + l] = mk<T>(y.x - r.y, y.y + r.x);
                        tile[(M - v) * LP + l] = mk<T>(y.x + r.y, r.x - y.y);
                    }
                }
            }
            __syncthreads();
            tile_fft<T, M, L, LP, NT, +1>(tile, tw);
        }
        // theta -> T_{k+1}, residual, state write, and the next applied rows
        // z = mirror(a_2p) + i mirror(a_2p+1), in place: a thread owns cell j of
        // both rows of its pair, so it alone reads and rewrites tile slot j (and
        // the mirror slot M-1-j, never read here).
        {
            constexpr int IPT = (L * n + NT - 1) / NT;
#pragma unroll
            for (int i0 = 0; i0 < IPT; i0 += UB) {
                T told[UB][2], pv[UB][2], lv[UB][2], hv[UB][2], qv[UB][2];
#pragma unroll
                for (int u = 0; u < UB; ++u) {
                    const int idx = threadIdx.x + (i0 + u) * NT;
                    const int l = idx / n, j = idx - l * n;
                    const int x = 2 * (p0 + l);
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        told[u][half] = pv[u][half] = lv[u][half] = hv[u][half] = qv[u][half] = T(0);
                        if (i0 + u < IPT && idx < L * n && x < n) {
                            const size_t o = static_cast<size_t>(x + half) * n + j;
                            if (!FIRST || warm) told[u][half] = Ts[o];
                            pv[u][half] = P[o];
                            lv[u][half] = in.nom_scale * Nm[o] * V[o];
                            // the shift-variant map and the Chebyshev x_{k-1} join the same batch
                            if (!FIRST && H) hv[u][half] = H[sg * sH + o];
                            if (om > 0.0) qv[u][half] = Qs[o];
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < UB; ++u) {
                    const int idx = threadIdx.x + (i0 + u) * NT;
                    if (i0 + u >= IPT || idx >= L * n) continue;
                    const int l = idx / n, j = idx - l * n;
                    const int x = 2 * (p0 + l);
                    T a[2] = {T(0), T(0)};
                    if (x < n) {
                        const cplx<T> z = FIRST ? mk<T>(T(0), T(0)) : tile[j * LP + l];
#pragma unroll
                        for (int half = 0; half < 2; ++half) {
                            T t = FIRST ? told[u][half] : T(0);  // warm start: the caller's T_0
                            if (!FIRST) {
                                T th = (half ? z.y : z.x) * inv;  // theta - T0
                                if (H) th += hv[u][half] * sig_prev;
                                t = th;
                                if (kirchhoff) t = kirchhoff_rise(th, kc, kexp, t_ambient, bad);
                                if (!finite_val(t)) bad |= GTD_ST_NONFINITE;
                                dmax = fmax(dmax, double(fabs(t - told[u][half])));
                                const size_t oq = static_cast<size_t>(x + half) * n + j;
                                if (Qs) {
                                    const T xprev = qv[u][half];
                                    Qs[oq] = told[u][half];
                                    Yout[sg * n * n + oq] = t;
                                    if (om > 0.0) t = omt * (gmt * t + (T(1) - gmt) * told[u][half] - xprev) + xprev;
                                }
                                Ts[oq] = t;
                            }
                            const T f = law ? T(exp(beta * t)) : T(1) + beta * t;
                            a[half] = pv[u][half] + lv[u][half] * f;
                            app_part += double(a[half]);
                        }
                    }
                    tile[j * LP + l] = mk<T>(a[0], a[1]);
                    tile[(M - 1 - j) * LP + l] = mk<T>(a[0], a[1]);
                }
            }
        }
        __syncthreads();
        tile_fft<T, M, L, LP, NT, -1>(tile, tw);
        for (int idx = threadIdx.x; idx < 2 * L * hp; idx += NT) {
            const int lr = idx / hp, v = idx - lr * hp;
            const int l = lr >> 1, half = lr & 1;
            const int x = 2 * p0 + lr;
            if (x >= n) continue;
            T o = T(0);  // real DCT part of the row's half spectrum (col_pass.cuh)
            if (v < n) {
                const cplx<T> Z = tile[v * LP + l];
                const cplx<T> Zc = cconj<T>(tile[((M - v) & (M - 1)) * LP + l]);
                o = half ? dct_part_im<T>(Z, Zc, g_hs[v]) : dct_part<T>(Z, Zc, g_hs[v]);
            }
            Ar[static_cast<size_t>(s) * n * hp + static_cast<size_t>(x) * hp + v] = o;
        }
        if (H) {
            app_part = warp_sum_d(app_part);
            if ((threadIdx.x & 31) == 0) atomicAdd(&state[sg].sum_app[it & 1], app_part);
        }
        if (!FIRST) {
            or_flags_fp(&status[sg], bad);
            dmax = warp_max_d(dmax);
            if ((threadIdx.x & 31) == 0) {
                // non-negative doubles order like their bit patterns
                atomicMax(&state[sg].res_bits, static_cast<unsigned long long>(__double_as_longlong(dmax)));
            }
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------------- rows (warp per row pair)
// M = 128 / 256 / 512: one warp owns the die-row pair (2p, 2p+1) of a sample:
// inverse row transform of Y_2p + i Y_2p+1 (both Hermitian) -> theta rows ->
// Kirchhoff inverse -> residual -> T written -> next applied rows -> forward
// transform of mirror(a_2p) + i mirror(a_2p+1) -> the two rows' real DCT parts.
// Rows are loaded / stored coalesced straight from registers.
constexpr int FPW_WARPS = 8;

template <typename T, int M>
constexpr bool fp_warp_rows() {
    return M == 128 || M == 256 || M == 512;
}

template <typename T, int M, bool FIRST, int FEAT>
__global__ void __launch_bounds__(FPW_WARPS * 32, sizeof(T) == 8 ? 1 : 2)
fp_rows_w(FPIn<T> in, int sample0, int count, const cplx<T>* __restrict__ Yspec, T* __restrict__ Ar,
          T* __restrict__ Tst, FPState* __restrict__ state, int* __restrict__ status,
          const cplx<T>* __restrict__ g_tw, const cplx<T>* __restrict__ g_hs, T beta, int law, int kirchhoff, T ka,
          T kb, T kexp, T t_ambient, int warm, const T* __restrict__ H_, long long sH, int it,
          T* __restrict__ Tprev_, T* __restrict__ Yout) {
    const T* const H = (FEAT & 1) ? H_ : nullptr;
    T* const Tprev = (FEAT & 2) ? Tprev_ : nullptr;
    using Gm = FPGeom<T, M>;
    using WF = WarpFFT<T, M>;
    constexpr int n = Gm::n, h = Gm::h, hp = Gm::hp, P = WF::P, E = n / 32, RP = n / 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* s_tw = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_tw1 = s_tw + M;
    cplx<T>* s_hs = s_tw1 + WF::TW1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    cplx<T>* scr = s_hs + n + warp * WF::SCRATCH;
    for (int t = threadIdx.x; t < M; t += FPW_WARPS * 32) s_tw[t] = g_tw[t];
    for (int t = threadIdx.x; t < n; t += FPW_WARPS * 32) s_hs[t] = g_hs[t];
    WF::build_tw1(s_tw1, g_tw, threadIdx.x, FPW_WARPS * 32);
    __syncthreads();
    constexpr T inv = T(1.0 / (double(M) * double(M)));
    const T kc = kb / ka;  // Kirchhoff inverse (kirchhoff.cuh)

    for (int item = blockIdx.x * FPW_WARPS + warp; item < count * RP; item += gridDim.x * FPW_WARPS) {
        const int s = item / RP, x0 = 2 * (item - s * RP);
        const size_t sg = static_cast<size_t>(sample0) + s;
        if (!FIRST && !state[sg].active) continue;  // warp-uniform
        T* T0r = Tst + sg * n * n + static_cast<size_t>(x0) * n;
        T* T1r = T0r + n;
        // Every global input of the item is requested up front (one exposed
        // round trip per row pair instead of three): previous T rows, P rows,
        // leakage rows L0 = nom N V.
        T t0[E], t1[E], p0[E], p1[E], l0[E], l1[E], h0[E], h1[E], q0[E], q1[E];
        const T sig_prev = (!FIRST && H) ? T(state[sg].sum_app[(it - 1) & 1]) : T(0);
        // Chebyshev acceleration state (omega > 0: x_{k+1} from G(x_k), x_k and x_{k-1})
        const double om = (!FIRST && Tprev) ? state[sg].omega : 0.0;
        const T omt = T(om), gmt = T(om > 0.0 ? state[sg].gamma : 1.0);
        T* Q0r = Tprev ? Tprev + sg * n * n + static_cast<size_t>(x0) * n : nullptr;
        {
            const T* P0 = in.P + sg * in.sP + static_cast<size_t>(x0) * n;
            const T* N0 = in.N + sg * in.sN + static_cast<size_t>(x0) * n;
            const T* V0 = in.V + sg * in.sV + static_cast<size_t>(x0) * n;
            const bool n_is_p = in.N == in.P && in.sN == in.sP;
#pragma unroll
            for (int t = 0; t < E; ++t) {
                const int j = lane + 32 * t;
                if (!FIRST || warm) {  // warm start (FIRST): the caller's T_0 instead of 0
                    t0[t] = T0r[j];
                    t1[t] = T1r[j];
                }
                p0[t] = P0[j];
                p1[t] = P0[n + j];
                h0[t] = h1[t] = q0[t] = q1[t] = T(0);
                if (om > 0.0) {
                    q0[t] = Q0r[j];
                    q1[t] = Q0r[n + j];
                }
                if (!FIRST && H) {
                    const T* H0 = H + sg * sH + static_cast<size_t>(x0) * n;
                    h0[t] = H0[j];
                    h1[t] = H0[n + j];
                }
                const T n0 = n_is_p ? p0[t] : N0[j], n1 = n_is_p ? p1[t] : N0[n + j];
                l0[t] = in.nom_scale * n0 * V0[j];
                l1[t] = in.nom_scale * n1 * V0[n + j];
            }
        }
        double dmax = 0.0;
        int bad = 0;
        if constexpr (!FIRST) {
            const cplx<T>* Y0 = Yspec + (static_cast<size_t>(s) * n + x0) * hp;
            const cplx<T>* Y1 = Y0 + hp;
            cplx<T> z[P];
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const int v = lane + 32 * k;
                const int w = v <= n ? v : M - v;
                const cplx<T> y = Y0[w], r = Y1[w];
                if (v == 0 || v == n)
                    z[k] = mk<T>(y.x, r.x);
                else if (v < n)
                    z[k] = mk<T>(y.x - r.y, y.y + r.x);
                else
                    z[k] = mk<T>(y.x + r.y, r.x - y.y);
            }
            WF::template run<+1>(z, scr, s_tw, s_tw1, lane);
            __syncwarp();
#pragma unroll
            for (int m1 = 0; m1 < P; ++m1) scr[WF::out_pos(lane, m1)] = z[m1];
            __syncwarp();
#pragma unroll
            for (int t = 0; t < E; ++t) {
                const int j = lane + 32 * t;
                const cplx<T> th = scr[j];
                T a = th.x * inv + h0[t] * sig_prev, b = th.y * inv + h1[t] * sig_prev;  // theta - T0, rows x0, x0+1
                if (kirchhoff) {
                    a = kirchhoff_rise(a, kc, kexp, t_ambient, bad);
                    b = kirchhoff_rise(b, kc, kexp, t_ambient, bad);
                }
                if (!finite_val(a) || !finite_val(b)) bad |= GTD_ST_NONFINITE;
                dmax = fmax(dmax, fmax(double(fabs(a - t0[t])), double(fabs(b - t1[t]))));
                if (Tprev) {  // keep x_k for the next accelerated step and G(x_k) as the result
                    Q0r[j] = t0[t];
                    Q0r[n + j] = t1[t];
                    T* Y0r = Yout + sg * n * n + static_cast<size_t>(x0) * n;
                    Y0r[j] = a;
                    Y0r[n + j] = b;
                }
                if (om > 0.0) {  // x_{k+1} = omega (gamma G(x_k) + (1 - gamma) x_k - x_{k-1}) + x_{k-1}
                    a = omt * (gmt * a + (T(1) - gmt) * t0[t] - q0[t]) + q0[t];
                    b = omt * (gmt * b + (T(1) - gmt) * t1[t] - q1[t]) + q1[t];
                }
                T0r[j] = a;
                T1r[j] = b;
                t0[t] = a;
                t1[t] = b;
            }
            __syncwarp();
        } else if (!warm) {
#pragma unroll
            for (int t = 0; t < E; ++t) t0[t] = t1[t] = T(0);
        }
        // next applied rows a = P + L0 f(T)
        T a0[E], a1[E];
#pragma unroll
        for (int t = 0; t < E; ++t) {
            const T f0 = law ? T(exp(beta * t0[t])) : T(1) + beta * t0[t];
            const T f1 = law ? T(exp(beta * t1[t])) : T(1) + beta * t1[t];
            a0[t] = p0[t] + l0[t] * f0;
            a1[t] = p1[t] + l1[t] * f1;
        }
        if (H) {
            double part = 0.0;
#pragma unroll
            for (int t = 0; t < E; ++t) part += double(a0[t]) + double(a1[t]);
            part = warp_sum_d(part);
            if (lane == 0) atomicAdd(&state[sg].sum_app[it & 1], part);
        }
        // z[i] = mirror(a0)[i] + i mirror(a1)[i]: mirror(i) = (31 - lane) + 32 (P-1-k) for k >= E
        cplx<T> z[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
            if (k < E)
                z[k] = mk<T>(a0[k], a1[k]);
            else
                z[k] = mk<T>(__shfl_xor_sync(0xffffffffu, a0[P - 1 - k], 31),
                             __shfl_xor_sync(0xffffffffu, a1[P - 1 - k], 31));
        }
        WF::template run<-1>(z, scr, s_tw, s_tw1, lane);
        __syncwarp();
#pragma unroll
        for (int m1 = 0; m1 < P; ++m1) scr[WF::out_pos(lane, m1)] = z[m1];
        __syncwarp();
        T* A0 = Ar + (static_cast<size_t>(s) * n + x0) * hp;
        T* A1 = A0 + hp;
        for (int v = lane; v < hp; v += 32) {
            T r0 = T(0), r1 = T(0);
            if (v < n) {
                const cplx<T> Z = scr[v];
                const cplx<T> Zc = cconj<T>(scr[(M - v) & (M - 1)]);
                const cplx<T> hv = s_hs[v];
                r0 = dct_part<T>(Z, Zc, hv);
                r1 = dct_part_im<T>(Z, Zc, hv);
            }
            A0[v] = r0;
            A1[v] = r1;
        }
        if constexpr (!FIRST) {
            or_flags_fp(&status[sg], bad);
            dmax = warp_max_d(dmax);
            if (lane == 0) atomicMax(&state[sg].res_bits, static_cast<unsigned long long>(__double_as_longlong(dmax)));
        }
        __syncwarp();
    }
}

// ----------------------------------------------------------------- columns (real-DCT packed)
// Per tile of W = 2 GA half-spectrum columns: GA packed A lines (two columns'
// real DCT parts At_v + i At_{v+GA}, mirror expansion in the stage-0 address),
// forward column FFT, C_v + i C_v' = w^{u/2} Z[u], Y_v = fk (conj(w^{(u+v)/2}) C_v)
// in registers between the last forward and first inverse stage, inverse column
// FFT on the pairs (Y_g, Y_{g+GA}), rows [0, n) stored.
template <typename T, int M>
struct FPCGeom {
    static constexpr int n = M / 2, h = n + 1;
    static constexpr int GA = FPGeom<T, M>::L / 2 > 0 ? FPGeom<T, M>::L / 2 : 1;
    static constexpr int W = 2 * GA;
    static constexpr int hp = FPGeom<T, M>::hp;
    static constexpr int CT = hp / W;
    static constexpr int U8 = (M / 8) * GA;
    static constexpr int NT = U8 >= 256 ? 256 : (U8 < 32 ? 32 : U8);
#ifndef GT_FPC_MINB64
#define GT_FPC_MINB64 2  // resident CTAs the fp64 column pass's register budget targets at M <= 512
                         // (128 registers, no spills: +2.5% on the fp64 stage, profiles/r2s4_notes.md)
#endif
    static constexpr int MINB = sizeof(T) == 8 ? (M <= 512 ? GT_FPC_MINB64 : 1) : ((512 / NT) < 1 ? 1 : 512 / NT);
    static constexpr int APLANE = (M + M / 8) * GA;
    static constexpr int TILE = InvLayout<GA, M>::SIZE > APLANE ? InvLayout<GA, M>::SIZE : APLANE;
    static_assert(hp % W == 0, "column tiles");
    static constexpr size_t SMEM =
        sizeof(cplx<T>) * (size_t(TILE) + StageTw<M, false>::SIZE + StageTw<M, true>::SIZE + M);
};

template <typename T, int M, int GA, int NT, int S>
__device__ __forceinline__ void fwd_stage_a(cplx<T>* tile, const cplx<T>* twf) {
    using ST = StageTw<M, false>;
    constexpr int R = ST::R(S), NS = ST::NS(S);
    constexpr int NB = (M / R) * GA;
    constexpr int BPT = (NB + NT - 1) / NT;
    cplx<T> v[BPT][1][R];
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int id = threadIdx.x + b * NT;
        if (NB % NT != 0 && id >= NB) break;
        const int g = id % GA, j = id / GA;
#pragma unroll
        for (int r = 0; r < R; ++r) v[b][0][r] = tile[prow<M / R>(j, r) * GA + g];
        stage_twiddle<T, M, false, S, 1>(v[b], j, twf);
        dftR<R, -1, T>(v[b][0]);
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int id = threadIdx.x + b * NT;
        if (NB % NT != 0 && id >= NB) break;
        const int g = id % GA, j = id / GA;
        const int k = j % NS;
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) tile[prow<NS>(base, r) * GA + g] = v[b][0][r];
    }
    __syncthreads();
}

template <typename T, int M, int GA, int NT, int S, int E>
struct FwdStagesA {
    __device__ __forceinline__ static void run(cplx<T>* tile, const cplx<T>* twf) {
        if constexpr (S < E) {
            fwd_stage_a<T, M, GA, NT, S>(tile, twf);
            FwdStagesA<T, M, GA, NT, S + 1, E>::run(tile, twf);
        }
    }
};

template <typename T, int M>
__global__ void __launch_bounds__(FPCGeom<T, M>::NT, FPCGeom<T, M>::MINB)
fp_cols_d(int sample0, int count, const T* __restrict__ Ar, cplx<T>* __restrict__ Yspec,
          const FPState* __restrict__ state, const cplx<T>* __restrict__ g_tw, const cplx<T>* __restrict__ g_hs,
          const cplx<T>* __restrict__ fk, int fk_pitch) {
    using Gc = FPCGeom<T, M>;
    using Pl = Plan<M>;
    using IL = InvLayout<Gc::GA, M>;
    constexpr int n = Gc::n, h = Gc::h, GA = Gc::GA, W = Gc::W, hp = Gc::hp, CT = Gc::CT, NT = Gc::NT;
    constexpr int K = Pl::K, RL = Pl::RLAST_F;
    constexpr int U0 = (M / 8) * GA, B0 = (U0 + NT - 1) / NT;
    constexpr int UL = (M / RL) * GA, BL = (UL + NT - 1) / NT;
    constexpr int BPTI = (M / 8) * GA / NT;
    constexpr int TWF = StageTw<M, false>::SIZE, TWI = StageTw<M, true>::SIZE;
    static_assert(K >= 2 && Pl::fr(0) == 8 && Pl::ir(K - 1) == 8, "plan");
    static_assert((M / 8) * GA % NT == 0 && BPTI >= 1, "threads");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_twf = tile + Gc::TILE;
    cplx<T>* s_twi = s_twf + TWF;
    cplx<T>* s_hs = s_twi + TWI;
    build_stage_tw<T, M, false, NT>(s_twf, g_tw);
    build_stage_tw<T, M, true, NT>(s_twi, g_tw);
    for (int t = threadIdx.x; t < M; t += NT) s_hs[t] = g_hs[t];

    for (int item = blockIdx.x; item < count * CT; item += gridDim.x) {
        const int s = item / CT, v0 = (item - s * CT) * W;
        const size_t sg = static_cast<size_t>(sample0) + s;
        if (!state[sg].active) continue;  // CTA-uniform
        const size_t sbase = static_cast<size_t>(s) * n * hp;
        __syncthreads();  // previous item's tile readers done (and the tables are built)
        // ---- forward stage 0 straight from the real DCT rows (mirror in the address)
        {
            cplx<T> v[B0][8];
#pragma unroll
            for (int b = 0; b < B0; ++b) {
                const int id = threadIdx.x + b * NT;
                if (U0 % NT != 0 && id >= U0) break;
                const int g = id % GA, j = id / GA;
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int i = j + r * (M / 8);
                    const int xa = i < n ? i : M - 1 - i;
                    const T* ar = Ar + sbase + static_cast<size_t>(xa) * hp + v0 + g;
                    v[b][r] = mk<T>(ar[0], ar[GA]);
                }
            }
#pragma unroll
            for (int b = 0; b < B0; ++b) {
                const int id = threadIdx.x + b * NT;
                if (U0 % NT != 0 && id >= U0) break;
                const int g = id % GA, j = id / GA;
                dftR<8, -1, T>(v[b]);
#pragma unroll
                for (int r = 0; r < 8; ++r) tile[prow<1>(j * 8, r) * GA + g] = v[b][r];
            }
        }
        __syncthreads();
        FwdStagesA<T, M, GA, NT, 1, K - 1>::run(tile, s_twf);
        // ---- last forward stage + spectral multiply + first inverse stage, in registers
        {
            cplx<T> y[BL][2][RL];
#pragma unroll
            for (int b = 0; b < BL; ++b) {
                const int id = threadIdx.x + b * NT;
                if (UL % NT != 0 && id >= UL) break;
                const int g = id % GA, j = id / GA;
                cplx<T> z[1][RL];
#pragma unroll
                for (int q = 0; q < RL; ++q) z[0][q] = tile[prow<M / RL>(j, q) * GA + g];
                stage_twiddle<T, M, false, K - 1, 1>(z, j, s_twf);
                dftR<RL, -1, T>(z[0]);
#pragma unroll
                for (int q = 0; q < RL; ++q) z[0][q] = cmul<T>(s_hs[j + q * (M / RL)], z[0][q]);  // C_v + i C_v'
#pragma unroll
                for (int col = 0; col < 2; ++col) {
                    const int vv = v0 + g + col * GA;
                    const cplx<T> hv = s_hs[vv];
#pragma unroll
                    for (int q = 0; q < RL; ++q) {
                        const int u = j + q * (M / RL);
                        const cplx<T> ph = cconj<T>(cmul<T>(s_hs[u], hv));
                        const cplx<T> f = vv < h ? fk[static_cast<size_t>(u) * fk_pitch + vv] : mk<T>(T(0), T(0));
                        y[b][col][q] = cscale<T>(cmul<T>(f, ph), col == 0 ? z[0][q].x : z[0][q].y);
                    }
                    dftR<RL, +1, T>(y[b][col]);
                }
            }
            __syncthreads();
#pragma unroll
            for (int b = 0; b < BL; ++b) {
                const int id = threadIdx.x + b * NT;
                if (UL % NT != 0 && id >= UL) break;
                const int g = id % GA, j = id / GA;
#pragma unroll
                for (int r = 0; r < RL; ++r)
                    st_pair(&tile[IL::template off<1>(j * RL, r, g)], LinePair<T>{y[b][0][r], y[b][1][r]});
            }
            __syncthreads();
        }
        InvStagesPairs<T, M, GA, NT, 1, K - 1>::run(tile, s_twi);
        // ---- last inverse stage: rows [0, n) of both columns
#pragma unroll
        for (int b = 0; b < BPTI; ++b) {
            const int id = threadIdx.x + b * NT;
            const int g = id % GA, j = id / GA;
            cplx<T> o[2][8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const LinePair<T> q = ld_pair(&tile[IL::template off<M / 8>(j, r, g)]);
                o[0][r] = q.a;
                o[1][r] = q.b;
            }
            stage_twiddle<T, M, true, K - 1, 2>(o, j, s_twi);
            dftR<8, +1, T>(o[0]);
            dftR<8, +1, T>(o[1]);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int i = j + r * (M / 8);
                if (i < n) {
                    cplx<T>* yr = Yspec + sbase + static_cast<size_t>(i) * hp + v0 + g;
                    yr[0] = o[0][r];
                    yr[GA] = o[1][r];
                }
            }
        }
    }
}

// ----------------------------------------------------------------- state
__global__ void fp_init(FPState* st, int* status, int* iters, int sample0, int count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    st[sample0 + i] = FPState{0ull, 0, 1, {0.0, 0.0}, 0.0, 0.0, 1.0, 0.0};
    status[sample0 + i] = 0;
    iters[sample0 + i] = 0;
}

// Reference stop rule (fdm.cpp:190-200): converge check first, then max_iters.
// Chebyshev semi-iteration on the Picard map G (opt-in, gtd_fp_opts.accel = k0 > 0): for
// x = J x + b with the spectrum of the Jacobian J in [0, rho] (a positive kernel times a
// positive leakage: L0^1/2 K L0^1/2 is symmetric positive), gamma = 2 / (2 - rho) maps it to
// [-sigma, sigma], sigma = rho / (2 - rho), and omega_1 = 1, omega_2 = 2 / (2 - sigma^2),
// omega_{k+1} = 1 / (1 - sigma^2 omega_k / 4) give the optimal polynomial error reduction.
// rho is estimated per sample from the Picard residual ratio at iteration k0; a residual
// that grows by 2x under acceleration drops the sample back to plain Picard.
__global__ void fp_update(FPState* st, int* status, int* iters, int sample0, int count, double tol, int max_iters,
                          int* active_count, int it, int accel, int min_iters) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    FPState& s = st[sample0 + i];
    if (!s.active) return;
    s.sum_app[(it - 1) & 1] = 0.0;  // read by this iteration's row pass; the next one accumulates into it
    s.iters += 1;
    iters[sample0 + i] = s.iters;
    const double res = __longlong_as_double(static_cast<long long>(s.res_bits));
    s.res_bits = 0ull;
    if (accel < 0) s.res_prev = res;
    if (accel > 0) {
        if (s.omega > 0.0) {
            if (res > 2.0 * s.res_prev) {
                s.omega = -1.0;  // diverging under acceleration: plain Picard from here on
                s.gamma = 1.0;
            } else {
                s.omega = s.omega == 1.0 ? 2.0 / (2.0 - s.sigma2) : 1.0 / (1.0 - 0.25 * s.sigma2 * s.omega);
            }
        } else if (s.omega == 0.0 && s.iters == accel && s.res_prev > 0.0) {
            const double rho = fmin(0.97, fmax(0.0, 1.02 * res / s.res_prev));
            s.gamma = 2.0 / (2.0 - rho);
            s.sigma2 = (rho / (2.0 - rho)) * (rho / (2.0 - rho));
            s.omega = 1.0;
        }
        s.res_prev = res;
    }
    if (status[sample0 + i]) {
        s.active = 0;
    } else if (s.iters >= min_iters && res < tol) {
        s.active = 0;
    } else if (s.iters >= max_iters) {
        status[sample0 + i] |= GTD_ST_NOCONVERGE;
        s.active = 0;
    }
    if (s.active) atomicAdd(active_count, 1);
}


// ---------------------------------------------------------------- low-mode Anderson mixing
// gtd_fp_opts.accel = -m: Anderson(m) acceleration of the Picard map restricted to the
// LMK x LMK lowest cosine modes of the die field (the leakage feedback operator beta G diag(L0)
// is a smoothing operator: its slow eigenvectors are smooth, everything else contracts in a few
// plain iterations). It runs between the column pass and the row pass on the row spectra Y:
//   a_pq   = low cosine coefficients of G(x_k), read from Y[x][q], q < LMK (a mirrored row with
//            cosine content d_q has Y[q] = conj(hs_q) M^2 eps_q d_q, eps_0 = 1, eps_q = 1/2),
//   f      = a - xlow  (xlow: the same coefficients of x_k, known by construction),
//   gamma  = argmin |f - dF gamma| over the last m residual differences (Tikhonov-regularised
//            normal equations in fp64), corr = -dG gamma,
//   Y[x][q] += conj(hs_q) M^2 eps_q sum_p corr_pq cos(pi p (x + 1/2) / n):  x_{k+1} = G(x_k) + corr.
// The fixed point is unchanged (corr -> 0 with f); the reference stop rule then applies to
// max|x_{k+1} - x_k|. State per sample: LMState (gtd_fp_lowmode_bytes()).
__global__ void fp_lowmode_init(LMState* lms, int sample0, int count, int warm) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count * LMN) return;
    LMState& L = lms[sample0 + i / LMN];
    const int t = i % LMN;
    L.xlow[t] = 0.0;
    if (t == 0) {
        L.calls = 0;
        L.nd = 0;
        L.have_x = warm ? 0 : 1;
        L.have_prev = 0;
        L.rprev = 0.0;
    }
}

__global__ void k_lowmode_cos(int n, double* table) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= LMK * n) return;
    const int p = i / n, x = i - p * n;
    table[i] = cospi(double(p) * (2.0 * x + 1.0) / (2.0 * n));
}

template <typename T>
__global__ void __launch_bounds__(LMN)
fp_lowmode(cplx<T>* __restrict__ Y, int n, int hp, int sample0, const FPState* __restrict__ state,
           LMState* __restrict__ lms, const cplx<T>* __restrict__ g_hs, const double* __restrict__ costab, int depth) {
    const int s = blockIdx.x;
    const size_t sg = static_cast<size_t>(sample0) + s;
    if (!state[sg].active) return;
    LMState& L = lms[sg];
    const int tid = threadIdx.x, p = tid / LMK, q = tid % LMK;
    const double M = 2.0 * n;
    cplx<T>* Ys = Y + static_cast<size_t>(s) * n * hp;
    const cplx<T> hq = g_hs[q];
    const double eq = q == 0 ? 1.0 : 0.5, ep = p == 0 ? 1.0 : 0.5;
    // 1. projection of G(x_k) on mode (p, q)
    double acc = 0.0;
    {
        const double* cp = costab + static_cast<size_t>(p) * n;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        for (int x = 0; x < n; x += 4) {  // n: a power of two >= 16
            const cplx<T> y0 = Ys[static_cast<size_t>(x) * hp + q], y1 = Ys[static_cast<size_t>(x + 1) * hp + q];
            const cplx<T> y2 = Ys[static_cast<size_t>(x + 2) * hp + q], y3 = Ys[static_cast<size_t>(x + 3) * hp + q];
            a0 += (double(hq.x) * y0.x - double(hq.y) * y0.y) * cp[x];
            a1 += (double(hq.x) * y1.x - double(hq.y) * y1.y) * cp[x + 1];
            a2 += (double(hq.x) * y2.x - double(hq.y) * y2.y) * cp[x + 2];
            a3 += (double(hq.x) * y3.x - double(hq.y) * y3.y) * cp[x + 3];
        }
        acc = (a0 + a1) + (a2 + a3);
    }
    const double g = acc / (M * M * eq * double(n) * ep);
    // 2. Anderson step on the LMN coefficients (lowmode.cuh)
    __shared__ double s_corr[LMN];
    bool mixed = false;
    const double corr = lowmode_mix(L, g, state[sg].res_prev, depth, tid, &mixed);
    const int k = mixed ? 1 : 0;
    s_corr[tid] = corr;
    __syncthreads();
    // 3. the correction's row spectra into Y (columns q < LMK of every die row)
    if (k > 0) {
        double cq[LMK];
#pragma unroll
        for (int pp = 0; pp < LMK; ++pp) cq[pp] = s_corr[pp * LMK + q];
        const double sc = M * M * eq;
        for (int x = p; x < n; x += LMK) {
            double v = 0.0;
#pragma unroll
            for (int pp = 0; pp < LMK; ++pp) v += cq[pp] * costab[static_cast<size_t>(pp) * n + x];
            v *= sc;
            cplx<T> y = Ys[static_cast<size_t>(x) * hp + q];
            y.x += T(v * double(hq.x));   // conj(hs_q) v
            y.y -= T(v * double(hq.y));
            Ys[static_cast<size_t>(x) * hp + q] = y;
        }
    }
}

// per-sample max / mean of the converged maps
template <typename T>
__global__ void __launch_bounds__(512) fp_stats(const T* __restrict__ Tst, int n, int sample0, double* __restrict__ mx,
                                                double* __restrict__ mean) {
    // one CTA per sample; each thread streams 4-element vectors with independent
    // accumulators (fixed order: deterministic), 8 loads in flight per iteration
    const size_t sg = static_cast<size_t>(sample0) + blockIdx.x;
    const T* t = Tst + sg * n * n;
    const size_t cnt = static_cast<size_t>(n) * n;  // n >= 16 even: a multiple of 8
    double m[8], s[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        m[k] = -1.0 / 0.0;
        s[k] = 0.0;
    }
    for (size_t i = static_cast<size_t>(threadIdx.x) * 8; i < cnt; i += static_cast<size_t>(blockDim.x) * 8) {
        T v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = t[i + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            m[k] = fmax(m[k], double(v[k]));
            s[k] += double(v[k]);
        }
    }
#pragma unroll
    for (int k = 1; k < 8; ++k) {
        m[0] = fmax(m[0], m[k]);
        s[0] += s[k];
    }
    double mm = m[0], ss = s[0];
    __shared__ double rm[32], rs[32];
    for (int o = 16; o > 0; o >>= 1) {
        mm = fmax(mm, __shfl_xor_sync(0xffffffffu, mm, o));
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    if ((threadIdx.x & 31) == 0) {
        rm[threadIdx.x >> 5] = mm;
        rs[threadIdx.x >> 5] = ss;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w) {
            mm = fmax(mm, rm[w]);
            ss += rs[w];
        }
        if (mx) mx[sg] = mm;
        if (mean) mean[sg] = ss / (double(n) * double(n));
    }
}

template <typename T, int M>
struct FPLaunch {
    using Gm = FPGeom<T, M>;
    using Gc = FPCGeom<T, M>;
    static size_t smem_rows() { return sizeof(cplx<T>) * (M * Gm::LP + (Gm::GTW ? 0 : M)); }
    static size_t smem_rows_w() {
        if constexpr (fp_warp_rows<T, M>())
            return sizeof(cplx<T>) * (M + WarpFFT<T, M>::TW1 + M / 2 + FPW_WARPS * WarpFFT<T, M>::SCRATCH);
        else
            return 0;
    }
    static size_t smem_cols() { return Gc::SMEM; }

    static int run(const gtd_greens* g, const FPIn<T>& in, int batch, const gtd_fp_opts* o, T* Tst, int* iters,
                   int* status, double* mx, double* mean, void* scratch, FPState* state, int* counter_d,
                   int* counter_h, int chunk, cudaStream_t st, long long* launches) {
        constexpr int n = Gm::n, hp = Gm::hp, NT = Gm::NT;
        constexpr int RP = n / 2;
        // res_r[FEAT] / res_w[FEAT]: resident CTAs per SM of the tile / warp row pass variants
        static int res_r[4] = {0, 0, 0, 0}, res_w[4] = {0, 0, 0, 0}, res_c = 0, sms = 0;
        static DeviceOnce once_;
        once_([&] {
            auto rows_attr = [&](auto feat_c) {
                constexpr int FE = decltype(feat_c)::value;
                cudaFuncSetAttribute(fp_rows<T, M, true, FE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_rows()));
                cudaFuncSetAttribute(fp_rows<T, M, false, FE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_rows()));
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res_r[FE], fp_rows<T, M, false, FE>, NT, smem_rows());
                if constexpr (fp_warp_rows<T, M>()) {
                    cudaFuncSetAttribute(fp_rows_w<T, M, true, FE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem_rows_w()));
                    cudaFuncSetAttribute(fp_rows_w<T, M, false, FE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem_rows_w()));
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res_w[FE], fp_rows_w<T, M, false, FE>,
                                                                  FPW_WARPS * 32, smem_rows_w());
                }
            };
            rows_attr(std::integral_constant<int, 0>{});
            rows_attr(std::integral_constant<int, 1>{});
            rows_attr(std::integral_constant<int, 2>{});
            rows_attr(std::integral_constant<int, 3>{});
            cudaFuncSetAttribute(fp_cols_d<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_cols()));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res_c, fp_cols_d<T, M>, Gc::NT, smem_cols());
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            for (int& r : res_r) r = r < 1 ? 1 : r;
            for (int& r : res_w) r = r < 1 ? 1 : r;
            res_c = res_c < 1 ? 1 : res_c;
        });
        const size_t per = static_cast<size_t>(n) * hp;
        cplx<T>* A = static_cast<cplx<T>*>(scratch);             // Y: column pass -> row pass
        T* Ar = reinterpret_cast<T*>(A + per * chunk);           // real DCT rows: row pass -> column pass
        const cplx<T>* tw = static_cast<const cplx<T>*>(g->tw);
        const cplx<T>* hs = static_cast<const cplx<T>*>(g->hs);
        const cplx<T>* fk = static_cast<const cplx<T>*>(g->fk);
        const T kexp = T(1.0 / (1.0 - o->eta));
        const T ka = T(pow(o->t_ambient, 1.0 - o->eta)), kb = T((1.0 - o->eta) * pow(o->t_ambient, -o->eta));
        auto grid = [&](int items, int r) { return items < sms * r ? items : sms * r; };
        const int poll = o->poll > 0 ? o->poll : 4;
        long long k = 0;
        const int feat = (o->H ? 1 : 0) | (o->Tprev ? 2 : 0);
        auto rows = [&](bool first, int s0, int cnt, int it_) {
            auto go = [&](auto first_c, auto feat_c) {
                constexpr bool F = decltype(first_c)::value;
                constexpr int FE = decltype(feat_c)::value;
                if constexpr (fp_warp_rows<T, M>()) {
                    const int gw = grid((cnt * RP + FPW_WARPS - 1) / FPW_WARPS, res_w[FE]);
                    fp_rows_w<T, M, F, FE><<<gw, FPW_WARPS * 32, smem_rows_w(), st>>>(
                        in, s0, cnt, A, Ar, Tst, state, status, tw, hs, T(o->beta), o->law, o->kirchhoff, ka, kb,
                        kexp, T(o->t_ambient), o->warm_start, static_cast<const T*>(o->H), o->sH, it_,
                        static_cast<T*>(o->Tprev), static_cast<T*>(o->Yout));
                } else {
                    const int gr = grid(cnt * Gm::RB, res_r[FE]);
                    fp_rows<T, M, F, FE><<<gr, NT, smem_rows(), st>>>(
                        in, s0, cnt, A, Ar, Tst, state, status, tw, hs, T(o->beta), o->law, o->kirchhoff, ka, kb,
                        kexp, T(o->t_ambient), o->warm_start, static_cast<const T*>(o->H), o->sH, it_,
                        static_cast<T*>(o->Tprev), static_cast<T*>(o->Yout));
                }
            };
            auto by_feat = [&](auto first_c) {
                switch (feat) {
                    case 0: go(first_c, std::integral_constant<int, 0>{}); break;
                    case 1: go(first_c, std::integral_constant<int, 1>{}); break;
                    case 2: go(first_c, std::integral_constant<int, 2>{}); break;
                    default: go(first_c, std::integral_constant<int, 3>{}); break;
                }
            };
            if (first) by_feat(std::true_type{});
            else by_feat(std::false_type{});
        };
        for (int s0 = 0; s0 < batch; s0 += chunk) {
            const int cnt = batch - s0 < chunk ? batch - s0 : chunk;
            const int gc = grid(cnt * Gc::CT, res_c);
            fp_init<<<(cnt + 127) / 128, 128, 0, st>>>(state, status, iters, s0, cnt);
            const bool lowmode = o->accel < 0 && o->lm_state && o->lm_cos && n >= LMK;
            if (lowmode && !o->lm_keep) {
                fp_lowmode_init<<<(cnt * LMN + 255) / 256, 256, 0, st>>>(static_cast<LMState*>(o->lm_state), s0, cnt,
                                                                         o->warm_start);
                k += 1;
            }
            rows(true, s0, cnt, 0);
            k += 2;
            for (int it = 1; it <= o->max_iters; ++it) {
                fp_cols_d<T, M><<<gc, Gc::NT, smem_cols(), st>>>(s0, cnt, Ar, A, state, tw, hs, fk, g->hp);
                if (lowmode) {
                    fp_lowmode<T><<<cnt, LMN, 0, st>>>(A, n, hp, s0, state, static_cast<LMState*>(o->lm_state), hs,
                                                       o->lm_cos, -o->accel);
                    k += 1;
                }
                rows(false, s0, cnt, it);
                cudaMemsetAsync(counter_d, 0, sizeof(int), st);
                fp_update<<<(cnt + 127) / 128, 128, 0, st>>>(state, status, iters, s0, cnt, o->tol, o->max_iters,
                                                            counter_d, it, o->accel,
                                                            o->min_iters > 0 ? o->min_iters : 2);
                k += 3;
                if (it % poll == 0 || it == o->max_iters) {
                    cudaMemcpyAsync(counter_h, counter_d, sizeof(int), cudaMemcpyDeviceToHost, st);
                    cudaStreamSynchronize(st);
                    if (*counter_h == 0) break;
                }
            }
            if (o->Tprev)  // accelerated: the result is G(x_k) of the last iteration (its error
                           // bound is the reference stop rule's, not that of the extrapolated x_{k+1})
                cudaMemcpyAsync(Tst + static_cast<size_t>(s0) * n * n, static_cast<T*>(o->Yout) + static_cast<size_t>(s0) * n * n,
                                sizeof(T) * n * n * cnt, cudaMemcpyDeviceToDevice, st);
            fp_stats<T><<<cnt, 512, 0, st>>>(Tst, n, s0, mx, mean);
            k += 1;
        }
        if (launches) *launches = k;
        return static_cast<int>(cudaGetLastError());
    }
};

template <typename T>
int dispatch_fp(const gtd_greens* g, const gtd_mc_in* i, int batch, const gtd_fp_opts* o, void* Tst, int* iters,
                int* status, double* mx, double* mean, void* scratch, void* state, int* counter_d, int* counter_h,
                int chunk, cudaStream_t st, long long* launches) {
    FPIn<T> in{static_cast<const T*>(i->P), static_cast<const T*>(i->N), static_cast<const T*>(i->V),
               i->sP, i->sN, i->sV, T(i->nom_scale)};
    T* t = static_cast<T*>(Tst);
    FPState* s = static_cast<FPState*>(state);
    switch (g->m) {
#define GT_FP_CASE(MM) \
    case MM: return FPLaunch<T, MM>::run(g, in, batch, o, t, iters, status, mx, mean, scratch, s, counter_d, counter_h, chunk, st, launches);
        GT_FP_CASE(32)
        GT_FP_CASE(64)
        GT_FP_CASE(128)
        GT_FP_CASE(256)
        GT_FP_CASE(512)
        GT_FP_CASE(1024)
        GT_FP_CASE(2048)
#undef GT_FP_CASE
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}

template <typename T>
int fp_hp(int m) {
    switch (m) {
        case 32: return FPGeom<T, 32>::hp;
        case 64: return FPGeom<T, 64>::hp;
        case 128: return FPGeom<T, 128>::hp;
        case 256: return FPGeom<T, 256>::hp;
        case 512: return FPGeom<T, 512>::hp;
        case 1024: return FPGeom<T, 1024>::hp;
        case 2048: return FPGeom<T, 2048>::hp;
        default: return -1;
    }
}

__global__ void k_widen(const float* __restrict__ a, double* __restrict__ b, size_t count) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x)
        b[i] = double(a[i]);
}
__global__ void k_narrow(const double* __restrict__ a, float* __restrict__ b, size_t count) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x)
        b[i] = float(a[i]);
}
__global__ void k_fp_or_status(int* status, const gtd_sample_stats* stats, int batch) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < batch) status[i] |= stats[i].status;
}
__global__ void k_fp_combine(int* iters, int* status, const int* it64, const int* st64, int batch, int max_iters) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= batch) return;
    const int it = iters[i] + it64[i];
    iters[i] = it;
    status[i] = st64[i] | (it > max_iters ? GTD_ST_NOCONVERGE : 0);
}

}  // namespace
}  // namespace gtb

using namespace gtb;

extern "C" {

size_t gtd_fp_scratch_bytes_per_sample(int n, int fp64) {
    const int hp = fp64 ? fp_hp<double>(2 * n) : fp_hp<float>(2 * n);
    if (hp < 0) return 0;
    return static_cast<size_t>(n) * hp * (fp64 ? 16 + 8 : 8 + 4);  // Y (complex) + real DCT rows
}

size_t gtd_fp_state_bytes(void) { return sizeof(FPState); }
size_t gtd_fp_lowmode_bytes(void) { return sizeof(LMState); }
int gtd_fp_lowmode_cos(int n, double* table, cudaStream_t st) {
    k_lowmode_cos<<<(LMK * n + 255) / 256, 256, 0, st>>>(n, table);
    return static_cast<int>(cudaGetLastError());
}

int gtd_widen(const float* src, double* dst, size_t count, cudaStream_t st) {
    k_widen<<<1184, 256, 0, st>>>(src, dst, count);
    return static_cast<int>(cudaGetLastError());
}
int gtd_narrow(const double* src, float* dst, size_t count, cudaStream_t st) {
    k_narrow<<<1184, 256, 0, st>>>(src, dst, count);
    return static_cast<int>(cudaGetLastError());
}
int gtd_fp_or_status(int* status, const gtd_sample_stats* stats, int batch, cudaStream_t st) {
    k_fp_or_status<<<(batch + 127) / 128, 128, 0, st>>>(status, stats, batch);
    return static_cast<int>(cudaGetLastError());
}
int gtd_fp_combine(int* iters, int* status, const int* it64, const int* st64, int batch, int max_iters,
                   cudaStream_t st) {
    k_fp_combine<<<(batch + 127) / 128, 128, 0, st>>>(iters, status, it64, st64, batch, max_iters);
    return static_cast<int>(cudaGetLastError());
}

int gtd_fp_batch(const gtd_greens* g, const gtd_mc_in* in, int batch, const gtd_fp_opts* opts, void* t_state,
                 int* iters, int* status, double* max_out, double* mean_out, void* scratch, void* state,
                 int* counter_d, int* counter_h, int chunk, cudaStream_t stream, long long* launches) {
    if (!g || !in || !opts || batch < 1 || chunk < 1 || !t_state) return static_cast<int>(cudaErrorInvalidValue);
    return g->fp64 ? dispatch_fp<double>(g, in, batch, opts, t_state, iters, status, max_out, mean_out, scratch, state,
                                         counter_d, counter_h, chunk, stream, launches)
                   : dispatch_fp<float>(g, in, batch, opts, t_state, iters, status, max_out, mean_out, scratch, state,
                                        counter_d, counter_h, chunk, stream, launches);
}

}  // extern "C"
