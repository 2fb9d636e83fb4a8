// mc_modeA.cu — fused three-pass Monte-Carlo steady composition (mode A).
//
// One unit of work = the reference's monte_carlo run_one (solver.cpp:353-374)
// on a (power map, variation map) pair:
//   p_leak0 = leak_frac * p_dyn * var               (leakage_baseline, variation.cpp:162-195)
//   mu = mean(p_leak0), p_var = p_leak0 - mu
//   F_det  = fk / (1 - alpha g (1+F(mu)) - mu beta fk)           (greens.cpp:203-216)
//   F_rand = F_det (beta fk q + alpha F(p_var) g) /
//            (1 - alpha (1+F(mu)+F(p_var)) g - mu beta fk - beta fk q)  (greens.cpp:225-251)
//   T = max(0, crop(IFFT(F_det . FFT(mirror(p_dyn+p_leak0))))
//            + kernel_to_die(IFFT(F_rand)) o p_var * sum(applied) * rand_scale)
//
// All transforms are on the mirror-padded m = 2n torus. Instead of the
// reference's four full m x m complex FFTs per sample, the path runs:
//   pass 1 (rows)   : per die row x, ONE complex length-m FFT of
//                     z = mirror(applied row) + i * centre-embedded(p_leak0 row),
//                     split into the two half spectra A[x][v], B[x][v] (v < n+1),
//                     plus the row-symmetrised p_leak0 S[x][dv] for q.
//   pass 2 (columns): per column v, expand A (mirror) and B (centre embedding)
//                     to length m, forward FFT, closed-form spectral algebra,
//                     inverse FFT, keep only the n rows the die needs.
//   pass 3 (rows)   : per die row, one complex length-m inverse FFT of
//                     Y + i R (both Hermitian), crop / kernel_to_die gather,
//                     Hadamard term, clamp, per-sample max / sum.
// F(p_var) is formed in pass 2 as F(p_leak0) - mu * K1 with K1 = k1 (x) k1 the
// analytic spectrum of the centred die box, so pass 1 never waits for mu.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "fft_tile.cuh"
#include "col_pass.cuh"
#include "fft_warp.cuh"
#include "bulk_copy.cuh"
#include "gt_device.h"

namespace gtb {

template <typename T>
struct Real;
template <>
struct Real<float> {
    static constexpr float max() { return 3.402823466e38f; }
};
template <>
struct Real<double> {
    static constexpr double max() { return 1.7976931348623157e308; }
};

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_max_t(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Sum of `v` over the CTA, result valid in thread 0. `red` >= 32 doubles.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    if (ln == 0) red[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = ln < (NT >> 5) ? red[ln] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;
}
template <int NT>
__device__ __forceinline__ double block_max(double v, double* red) {
    v = warp_max(v);
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    if (ln == 0) red[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = ln < (NT >> 5) ? red[ln] : 0.0;
        r = warp_max(r);
    }
    __syncthreads();
    return r;
}

// Bitwise OR of per-thread status flags into the sample's status word.
__device__ __forceinline__ void or_flags(int* dst, int flags) {
    const int w = __reduce_or_sync(0xffffffffu, flags);
    if ((threadIdx.x & 31) == 0 && w) atomicOr(dst, w);
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ float fast_rcp(float x) { return __fdividef(1.0f, x); }
__device__ __forceinline__ double fast_rcp(double x) { return 1.0 / x; }

template <typename T>
__device__ __forceinline__ bool finite_(T v) {
    return isfinite(v);
}

template <typename T>
struct BitsOf;
template <>
struct BitsOf<float> {
    using U = unsigned;
    __device__ __forceinline__ static U get(float v) { return __float_as_uint(v); }
};
template <>
struct BitsOf<double> {
    using U = unsigned long long;
    __device__ __forceinline__ static U get(double v) { return static_cast<U>(__double_as_longlong(v)); }
};

template <typename T>
struct MCIn {
    const T* P;
    const T* N;
    const T* V;
    long long sP, sN, sV;
    T nom_scale;
    __device__ __forceinline__ const T* p(size_t s) const { return P + s * sP; }
    __device__ __forceinline__ const T* nn(size_t s) const { return N + s * sN; }
    __device__ __forceinline__ const T* v(size_t s) const { return V + s * sV; }
};

template <typename T, int M>
struct MCGeom {
    using G = TileGeom<T, M>;
    static constexpr int n = M / 2;
    static constexpr int c = n / 2;
    static constexpr int h = n + 1;
    static constexpr int L = G::L;
    static constexpr int NT = G::NT;
    // fp32 at M = 2048: 4 columns per pass-2 tile (one 512-thread CTA per SM; the
    // default 2 give 8-16-byte row segments and 8 warps per SM: +4.5% for config 2)
    static constexpr bool WIDE2048 = M == 2048 && sizeof(T) == 4;
#ifdef GT_P2_W
    static constexpr int W = M >= 512 ? GT_P2_W : L / 2;  // pass-2 tile width (tuning override)
#else
    static constexpr int W = WIDE2048 ? 4 : L / 2;  // columns per pass-2 tile
#endif
    static constexpr int hp = ((h + W - 1) / W) * W;
    static constexpr int LP = L + 2;  // padded pitch for row tiles (transposing I/O; even for pairs)
    static constexpr int SP = n + 1;  // padded pitch of the row staging arrays
    // pass 2 threads: GT_P2_NT caps the CTA (more butterflies per thread, more
    // registers each); the register budget still targets P2_CTAS CTAs per SM
#ifndef GT_P2_NT
#define GT_P2_NT 256
#endif
#ifndef GT_P2_TILE_MAJOR
#define GT_P2_TILE_MAJOR 0
#endif
#ifndef GT_P2_CTAS
#define GT_P2_CTAS 2
#endif
    static constexpr int NT2C = WIDE2048 ? 512 : GT_P2_NT;
    static constexpr int NT2 = (M / 8) * W > NT2C ? NT2C : (M / 8) * W;
    static constexpr int REGS2 = (65536 / GT_P2_CTAS) / NT2 > 255 ? 255 : (65536 / GT_P2_CTAS) / NT2;
    // pass 2 holds three lines per thread-butterfly: 128 registers (fp32) / 255 (fp64)
#ifdef GT_P2_MINB
    static constexpr int MINB2 = sizeof(T) == 8 ? 1 : GT_P2_MINB;  // tuning override (occupancy sweeps)
#else
    static constexpr int MINB2 = sizeof(T) == 8 ? 1 : ((512 / NT2) < 1 ? 1 : (512 / NT2));
#endif
};

// ------------------------------------------------------------------ pass 1
// The applied map enters the row transform mirror-padded, so its half spectrum
// is A[v] = w^{-v/2} At[v] with At real (the DCT-II of the row; w = e^{-2 pi i/M}).
// Pass 1 stores only At = Re(w^{v/2} A), A = (Z[v] + conj Z[M-v]) / 2, with
// hs[v] = w^{v/2}; At[n] = 0 exactly.

// Persistent over (sample, block of L die rows). Each die row x becomes one
// complex line z = mirror(applied row) + i * centre-embedded(p_leak0 row).
template <typename T, int M>
__global__ void __launch_bounds__(TileGeom<T, M>::NT, TileGeom<T, M>::MINB)
mc_pass1(const MCIn<T> in, int sample0, int count, T* __restrict__ Areal,
         cplx<T>* __restrict__ Bspec, T* __restrict__ Srow, gtd_sample_stats* __restrict__ stats,
         const cplx<T>* __restrict__ g_tw, const cplx<T>* __restrict__ g_hs, T var_lo, T var_hi) {
    using Gm = MCGeom<T, M>;
    constexpr int n = Gm::n, c = Gm::c, h = Gm::h, L = Gm::L, LP = Gm::LP, NT = Gm::NT;
    constexpr int hp = Gm::hp;
    constexpr int RB = (n + L - 1) / L;
    constexpr int EPT = (L * n + NT - 1) / NT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    T* tileT = reinterpret_cast<T*>(tile);
    cplx<T>* s_tw = tile + M * LP;
    double* red = reinterpret_cast<double*>(s_tw + M);

    load_twiddles<T, M, NT>(s_tw, g_tw);
    for (int item = blockIdx.x; item < count * RB; item += gridDim.x) {
        const int s = item / RB;
        const int x0 = (item - s * RB) * L;
        const size_t sg = static_cast<size_t>(sample0) + s;
        const T* P = in.p(sg);
        const T* Nm = in.nn(sg);
        const T* V = in.v(sg);
        const bool n_is_p = Nm == P;

        // imaginary part outside the centre embedding is zero
        for (int idx = threadIdx.x; idx < (M - 2 * c) * L; idx += NT) {
            const int l = idx % L, j = c + idx / L;
            tileT[2 * (j * LP + l) + 1] = T(0);
        }
        T pv[EPT], nv[EPT], vv[EPT];
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            const int idx = threadIdx.x + k * NT;
            const int l = idx / n, y = idx - l * n, x = x0 + l;
            pv[k] = nv[k] = T(0);
            vv[k] = T(1);
            if (idx < L * n && x < n) {
                pv[k] = P[x * n + y];
                nv[k] = n_is_p ? pv[k] : Nm[x * n + y];
                vv[k] = V[x * n + y];
            }
        }
        T part_l = T(0), part_a = T(0);  // per-thread partials (<= EPT terms), fp64 across threads
        int bad = 0;
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            const int idx = threadIdx.x + k * NT;
            if (idx >= L * n) break;
            const int l = idx / n, y = idx - l * n;
            const T p = pv[k], nm = nv[k], vr = vv[k];
            if (!(p >= T(0)) || !finite_(p) || !(nm >= T(0)) || !finite_(nm)) bad |= GTD_ST_BAD_POWER;
            if (!(vr >= var_lo && vr <= var_hi)) bad |= GTD_ST_BAD_VAR;
            const T lk = in.nom_scale * nm * vr;
            const T a = p + lk;
            part_l += lk;
            part_a += a;
            tileT[2 * (y * LP + l)] = a;
            tileT[2 * ((M - 1 - y) * LP + l)] = a;
            tileT[2 * (((y - c) & (M - 1)) * LP + l) + 1] = lk;
        }
        or_flags(&stats[sg].status, bad);
        const double tl = block_sum<NT>(double(part_l), red);  // (contains the barrier for the tile)
        const double ta = block_sum<NT>(double(part_a), red);
        if (threadIdx.x == 0) {
            atomicAdd(&stats[sg].sum_leak, tl);
            atomicAdd(&stats[sg].sum_applied, ta);
        }
        // Row-symmetrised leakage for q (symmetric_multiplier, spectral.cpp:167-185),
        // read back from the embedded imaginary part: p_leak0(l, y) at j = (y - c) mod M.
        for (int idx = threadIdx.x; idx < L * hp; idx += NT) {
            const int l = idx / hp, dv = idx - l * hp;
            const int x = x0 + l;
            if (x >= n) continue;
            T v = T(0);
            if (dv < h) {
                const int jp = min(c + dv, n - 1), jm = max(c - dv, 0);
                v = tileT[2 * (((jp - c) & (M - 1)) * LP + l) + 1] + tileT[2 * (((jm - c) & (M - 1)) * LP + l) + 1];
            }
            Srow[(static_cast<size_t>(s) * n + x) * hp + dv] = v;
        }
        __syncthreads();
        tile_fft<T, M, L, LP, NT, -1>(tile, s_tw);

        // Split Z into the two real-input half spectra and store rows.
        for (int idx = threadIdx.x; idx < L * hp; idx += NT) {
            const int l = idx / hp, v = idx - l * hp;
            const int x = x0 + l;
            if (x >= n) continue;
            T Ar = T(0);
            cplx<T> B = mk<T>(T(0), T(0));
            if (v < h) {
                const cplx<T> Z = tile[v * LP + l];
                const cplx<T> Zc = cconj<T>(tile[((M - v) & (M - 1)) * LP + l]);
                if (v < n) Ar = dct_part<T>(Z, Zc, g_hs[v]);
                const T dx = Z.x - Zc.x, dy = Z.y - Zc.y;
                B = mk<T>(T(0.5) * dy, T(-0.5) * dx);
            }
            const size_t o = (static_cast<size_t>(s) * n + x) * hp + v;
            Areal[o] = Ar;
            Bspec[o] = B;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ pass 2
// Closed forms at one frequency (u, v): returns Y = F_det A and R = F_rand
// (greens.cpp:203-251) with one shared reciprocal; sets runaway flags.
template <typename T>
struct Vec4;
template <>
struct Vec4<float> {
    using type = float4;
};
template <>
struct Vec4<double> {
    using type = double4;
};

template <typename T, int M>
struct ClosedForm {
    using V4 = typename Vec4<T>::type;
    static constexpr int n = M / 2, c = n / 2, hp = MCGeom<T, M>::hp, W = MCGeom<T, M>::W;
    const V4* __restrict__ fg;  // {fk.re, fk.im, alpha g, D(u) D(v)} per (u, v) (fft2d.cu k_fg)
    T mug, mb;   // mu_g, mu_g beta
    T mus;       // sample mean leakage (F(p_var) = F(p_leak0) - mu K1)
    T bq4, bqs;  // beta / 4, beta qshift: beta q = bq4 (S[ip] + S[im]) + bqs
    T mn1, mn2;  // running minima of |den1|^2, |den2|^2 (runaway flags after the tile)

    __device__ __forceinline__ V4 table(int u, int v) const { return fg[static_cast<size_t>(u) * hp + v]; }
    // At frequency (u, v) (greens.cpp:203-251, one shared reciprocal):
    //   C: real 2-D DCT coefficient of the applied map, A_hat = ph C with
    //   ph = conj(w^{u/2} w^{v/2}); b: F(p_leak0) on entry, F_rand on return;
    //   ssum = S[ip] + S[im] (row-symmetrised leakage); returns Y = F_det A_hat.
    // den1 = 1 - alpha g - mu beta fk: F(mu) only touches the DC term, where
    // g(0,0) = g_sp0(c,c) - g_sp0(c,c) = 0 (greens.cpp:186-192), so it drops out.
    __device__ __forceinline__ cplx<T> eval(T C, cplx<T>& b, T ssum, cplx<T> ph, const V4& t4) {
        const T fx = t4.x, fy = t4.y, ag = t4.z, mk1 = mus * t4.w;
        const T a1 = T(1) - ag;
        const cplx<T> Bp = mk<T>(b.x - mk1 * ph.x, b.y - mk1 * ph.y);  // F(p_var) = F(p_leak0) - mu K1
        const T bq = bq4 * ssum + bqs;
        const cplx<T> den1 = mk<T>(a1 - mb * fx, -mb * fy);
        const cplx<T> t1 = mk<T>(bq * fx + ag * Bp.x, bq * fy + ag * Bp.y);
        const cplx<T> den2 = mk<T>(den1.x - t1.x, den1.y - t1.y);
        const T d1 = cabs2<T>(den1), d2 = cabs2<T>(den2);
        mn1 = fmin(mn1, d1);
        mn2 = fmin(mn2, d2);
        const cplx<T> fr = cscale<T>(cmul<T>(mk<T>(fx, fy), cconj<T>(den1)), fast_rcp(d1 * d2));
        b = cmul<T>(cmul<T>(fr, t1), cconj<T>(den2));
        return cscale<T>(cmul<T>(fr, ph), C * d2);
    }
    __device__ __forceinline__ int flags() const {
        return (mn1 < T(1e-12) ? GTD_ST_RUNAWAY_DET : 0) | (mn2 < T(1e-12) ? GTD_ST_RUNAWAY_RAND : 0);
    }
};

template <typename T, int GA, int M>
struct FwdLayout {
    static constexpr int ROWS = M + M / 8;
    static constexpr int PA_OFF = 2 * ROWS * GA;  // PB first (16-B aligned pairs), then PA
    static constexpr int SIZE = 3 * ROWS * GA;
    __device__ __forceinline__ static int pa(int prow_, int g) { return PA_OFF + prow_ * GA + g; }
    __device__ __forceinline__ static int pb(int prow_, int g) { return (prow_ * GA + g) * 2; }
};

// One forward Stockham stage over the (A, B, B') line groups of the tile.
template <typename T, int M, int GA, int NT, int S>
__device__ __forceinline__ void fwd_stage_ab(cplx<T>* tile, const cplx<T>* twf) {
    using FL = FwdLayout<T, GA, M>;
    using ST = StageTw<M, false>;
    constexpr int R = ST::R(S), NS = ST::NS(S);
    constexpr int NB = (M / R) * GA;
    constexpr int BPT = (NB + NT - 1) / NT;
    cplx<T> v[BPT][3][R];
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int id = threadIdx.x + b * NT;
        if (NB % NT != 0 && id >= NB) break;
        const int g = id % GA, j = id / GA;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int pr = prow<M / R>(j, r);
            v[b][0][r] = tile[FL::pa(pr, g)];
            const LinePair<T> q = ld_pair(&tile[FL::pb(pr, g)]);
            v[b][1][r] = q.a;
            v[b][2][r] = q.b;
        }
        stage_twiddle<T, M, false, S, 3>(v[b], j, twf);
#pragma unroll
        for (int l = 0; l < 3; ++l) dftR<R, -1, T>(v[b][l]);
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
        for (int r = 0; r < R; ++r) {
            const int pr = prow<NS>(base, r);
            tile[FL::pa(pr, g)] = v[b][0][r];
            st_pair(&tile[FL::pb(pr, g)], LinePair<T>{v[b][1][r], v[b][2][r]});
        }
    }
    __syncthreads();
}

template <typename T, int M, int GA, int NT, int S, int E>
struct FwdStagesAB {
    __device__ __forceinline__ static void run(cplx<T>* tile, const cplx<T>* twf) {
        if constexpr (S < E) {
            fwd_stage_ab<T, M, GA, NT, S>(tile, twf);
            FwdStagesAB<T, M, GA, NT, S + 1, E>::run(tile, twf);
        }
    }
};

// Persistent over (sample, tile of W half-spectrum columns).
//   forward: per column group one packed A line (two columns' real DCT parts:
//            the mirrored column of a real DCT row spectrum is again a DCT, so
//            the column transform of At_v + i At_v' separates locally:
//            C_v + i C_v' = w^{u/2} Z[u], A_hat_v = w^{-(u+v)/2} C_v) plus the
//            two B lines -- 3 lines per 2 columns instead of 4;
//   stage 0 reads straight from the row spectra (mirror / centre expansion in
//   the address; the centre embedding leaves half the B inputs zero), the last
//   forward stage, the closed forms and the first inverse stage run in
//   registers, and the last inverse stage writes the kept rows to global.
template <typename T, int M>
__global__ void __launch_bounds__(MCGeom<T, M>::NT2, MCGeom<T, M>::MINB2)
mc_pass2(const MCIn<T> in, int sample0, int count, const T* __restrict__ Areal,
         cplx<T>* __restrict__ Yspec, cplx<T>* __restrict__ Bspec, const T* __restrict__ Srow,
         gtd_sample_stats* __restrict__ stats, const cplx<T>* __restrict__ g_tw,
         const cplx<T>* __restrict__ g_hs, const T* __restrict__ fgtab, T alpha, T beta, int mu_per_sample,
         T mu_fixed) {
    using Gm = MCGeom<T, M>;
    using Pl = Plan<M>;
    constexpr int n = Gm::n, c = Gm::c, h = Gm::h, L = Gm::L, NT = Gm::NT2, W = Gm::W;
    constexpr int hp = Gm::hp;
    constexpr int CT = hp / W;
    constexpr int K = Pl::K;
    constexpr int GA = W >= 2 ? W / 2 : 1;  // column groups per tile
    constexpr int CG = W >= 2 ? 2 : 1;      // columns per group (v0 + g, v0 + g + GA)
    using FL = FwdLayout<T, GA, M>;
    using IL = InvLayout<W, M>;
    constexpr int U0 = (M / 8) * GA;
    constexpr int B0 = (U0 + NT - 1) / NT;
    constexpr int RL = Pl::RLAST_F;
    constexpr int UL = (M / RL) * GA;
    constexpr int BL = (UL + NT - 1) / NT;
    constexpr int RI = Pl::ir(K - 1);  // last inverse stage radix (8)
    constexpr int BPTI = (M / RI) * W / NT;
    constexpr int TWF = StageTw<M, false>::SIZE, TWI = StageTw<M, true>::SIZE;
    static_assert(K >= 2 && Pl::fr(0) == 8 && RI == 8, "plan");
    static_assert((M / 8) * W % NT == 0 && BPTI >= 1, "threads");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_twf = tile + (IL::SIZE > FL::SIZE ? IL::SIZE : FL::SIZE);
    cplx<T>* s_twi = s_twf + TWF;
    cplx<T>* s_hs = s_twi + TWI;
    T* s_srow = reinterpret_cast<T*>(s_hs + M);

    build_stage_tw<T, M, false, NT>(s_twf, g_tw);
    build_stage_tw<T, M, true, NT>(s_twi, g_tw);
    load_twiddles<T, M, NT>(s_hs, g_hs);
    for (int item = blockIdx.x; item < count * CT; item += gridDim.x) {
        // column-tile-major order: a CTA revisits the same column tile for
        // successive samples, so that tile's closed-form table stays in L1
#if GT_P2_TILE_MAJOR
        const int tI = item / count, s = item - tI * count;
#else
        const int s = item / CT, tI = item - s * CT;
#endif
        const int v0 = tI * W;
        const size_t sg = static_cast<size_t>(sample0) + s;
        const size_t sbase = static_cast<size_t>(s) * n * hp;
        __syncthreads();  // previous item's readers of tile / s_srow are done (and the tables are built)

        // ---- forward stage 0 (radix 8, NS = 1) straight from the row spectra
        cplx<T> v[B0][3][8];
#pragma unroll
        for (int b = 0; b < B0; ++b) {
            const int id = threadIdx.x + b * NT;
            if (U0 % NT != 0 && id >= U0) break;
            const int g = id % GA, j = id / GA;
            const int va = v0 + g;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int i = j + r * (M / 8);
                const int xa = i < n ? i : M - 1 - i;  // mirror_pad
                const int xb = (i + c) & (M - 1);      // centre_kernel: row i holds die row x
                const T* ar = Areal + sbase + static_cast<size_t>(xa) * hp + va;
                v[b][0][r] = mk<T>(ar[0], CG == 2 ? ar[GA] : T(0));
                // the centre embedding fills rows [0, M/4) u [3M/4, M): r in {0,1,6,7} only
                if (r < 2 || r >= 6) {
                    const cplx<T>* bp = Bspec + sbase + static_cast<size_t>(xb) * hp + va;
                    v[b][1][r] = bp[0];
                    v[b][2][r] = CG == 2 ? bp[GA] : mk<T>(T(0), T(0));
                }
            }
        }
#ifndef GT_P2_L2PF
#define GT_P2_L2PF 1
#endif
#if GT_P2_L2PF
        // The next item's row-spectrum tiles (A, B, S: one row segment per die row)
        // are pulled into L2 now, so its stage-0 loads hit L2 instead of HBM.
        {
            const int nx = item + gridDim.x;
            if (nx < count * CT) {
#if GT_P2_TILE_MAJOR
                const int tn = nx / count, sn = nx - tn * count;
#else
                const int sn = nx / CT, tn = nx - sn * CT;
#endif
                const size_t nb = static_cast<size_t>(sn) * n * hp + static_cast<size_t>(tn) * W;
                constexpr int LA = (W * int(sizeof(T)) + 127) / 128, LB = (W * int(sizeof(cplx<T>)) + 127) / 128;
                constexpr int PER = 2 * LA + LB;  // A and S segments, then B
#pragma unroll
                for (int t = threadIdx.x; t < n * PER; t += NT) {
                    const int k = t / n, x = t - k * n;  // n: power of two
                    const size_t o = nb + static_cast<size_t>(x) * hp;
                    if (k < LA)
                        prefetch_l2(reinterpret_cast<const char*>(Areal + o) + 128 * k);
                    else if (k < 2 * LA)
                        prefetch_l2(reinterpret_cast<const char*>(Srow + o) + 128 * (k - LA));
                    else
                        prefetch_l2(reinterpret_cast<const char*>(Bspec + o) + 128 * (k - 2 * LA));
                }
            }
        }
#endif
        // S rows into registers now, into shared memory after the stage-0 math (latency overlap)
        constexpr int ES = (n * W + NT - 1) / NT;
        T sv[ES];
#pragma unroll
        for (int k = 0; k < ES; ++k) {
            const int idx = threadIdx.x + k * NT;
            sv[k] = idx < n * W ? Srow[sbase + static_cast<size_t>(idx / W) * hp + v0 + idx % W] : T(0);
        }
#pragma unroll
        for (int b = 0; b < B0; ++b) {
            const int id = threadIdx.x + b * NT;
            if (U0 % NT != 0 && id >= U0) break;
            const int g = id % GA, j = id / GA;
            dftR<8, -1, T>(v[b][0]);
            dft8_outer_only<-1, T>(v[b][1]);
            dft8_outer_only<-1, T>(v[b][2]);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int pr = prow<1>(j * 8, r);
                tile[FL::pa(pr, g)] = v[b][0][r];
                st_pair(&tile[FL::pb(pr, g)], LinePair<T>{v[b][1][r], v[b][2][r]});
            }
        }
#pragma unroll
        for (int k = 0; k < ES; ++k) {
            const int idx = threadIdx.x + k * NT;
            if (idx < n * W) s_srow[(idx / W) * W + idx % W] = sv[k];
        }
        // Per-sample scalars (pass 1 has completed: kernel boundary).
        const double n2 = double(n) * double(n);
        const double mu_s = stats[sg].sum_leak / n2;
        const T* Nm = in.nn(sg);
        const T* Vm = in.v(sg);
        ClosedForm<T, M> cf;
        cf.fg = reinterpret_cast<const typename Vec4<T>::type*>(fgtab);
        cf.mug = mu_per_sample ? T(mu_s) : mu_fixed;
        cf.mb = cf.mug * beta;
        cf.mus = T(mu_s);
        cf.bq4 = T(0.25) * beta;
        {
            const T pl_cc = in.nom_scale * Nm[c * n + c] * Vm[c * n + c];
            const T pl_00 = in.nom_scale * Nm[0] * Vm[0];
            cf.bqs = beta * T(double(pl_cc) - double(pl_00) - mu_s);  // q shift, greens.cpp:177-184
        }
        cf.mn1 = cf.mn2 = Real<T>::max();
        __syncthreads();
        // ---- middle forward stages
        FwdStagesAB<T, M, GA, NT, 1, K - 1>::run(tile, s_twf);
        // ---- last forward stage + closed forms + first inverse stage, in registers.
        // All forward inputs are read before one barrier, so each column's (Y, R)
        // pair is stored as soon as it is transformed (two lines live, not four:
        // the registers this frees let the table loads issue ahead of their use).
        {
            cplx<T> z[BL][3][RL];
#pragma unroll
            for (int b = 0; b < BL; ++b) {
                const int id = threadIdx.x + b * NT;
                if (UL % NT != 0 && id >= UL) break;
                const int g = id % GA, j = id / GA;
#pragma unroll
                for (int q = 0; q < RL; ++q) {
                    const int pr = prow<M / RL>(j, q);
                    z[b][0][q] = tile[FL::pa(pr, g)];
                    const LinePair<T> p = ld_pair(&tile[FL::pb(pr, g)]);
                    z[b][1][q] = p.a;
                    z[b][2][q] = p.b;
                }
            }
            __syncthreads();
#pragma unroll
            for (int b = 0; b < BL; ++b) {
                const int id = threadIdx.x + b * NT;
                if (UL % NT != 0 && id >= UL) break;
                const int g = id % GA, j = id / GA;
                stage_twiddle<T, M, false, K - 1, 3>(z[b], j, s_twf);
#pragma unroll
                for (int l = 0; l < 3; ++l) dftR<RL, -1, T>(z[b][l]);
                // C_v + i C_v' = w^{u/2} Z[u]
#pragma unroll
                for (int q = 0; q < RL; ++q) z[b][0][q] = cmul<T>(s_hs[j + q * (M / RL)], z[b][0][q]);
#pragma unroll
                for (int col = 0; col < CG; ++col) {
                    const int w = g + col * GA, vv = v0 + w;
                    const cplx<T> hv = s_hs[vv];
                    cplx<T> yr[2][RL];  // Y, R of this column
#pragma unroll
                    for (int q = 0; q < RL; ++q) {
                        const int u = j + q * (M / RL);
                        // S rows ip = min(c + du, n - 1), im = max(c - du, 0). Padded columns
                        // (v > n) see an all-zero table entry and S = 0: they evaluate to 0.
                        const int du = u <= M - u ? u : M - u;
                        const int sp = min(c + du, n - 1) * W, sm = max(c - du, 0) * W;
                        const cplx<T> ph = cconj<T>(cmul<T>(s_hs[u], hv));
                        cplx<T> bb = z[b][1 + col][q];
                        yr[0][q] = cf.eval(col == 0 ? z[b][0][q].x : z[b][0][q].y, bb,
                                           s_srow[sp + w] + s_srow[sm + w], ph, cf.table(u, vv));
                        yr[1][q] = bb;
                    }
                    dftR<RL, +1, T>(yr[0]);
                    dftR<RL, +1, T>(yr[1]);
#pragma unroll
                    for (int r = 0; r < RL; ++r)
                        st_pair(&tile[IL::template off<1>(j * RL, r, w)], LinePair<T>{yr[0][r], yr[1][r]});
                }
            }
            __syncthreads();
        }
        or_flags(&stats[sg].status, cf.flags());
        // ---- middle inverse stages
        InvStagesPairs<T, M, W, NT, 1, K - 1>::run(tile, s_twi);
        // ---- last inverse stage (radix 8, NS = M/8): keep rows [0, n) of Y, rows rho(x) of R
        {
#pragma unroll
            for (int b = 0; b < BPTI; ++b) {
                const int id = threadIdx.x + b * NT;
                const int w = id % W, j = id / W;
                const int vv = v0 + w;
                cplx<T> o[2][8];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const LinePair<T> q = ld_pair(&tile[IL::template off<M / 8>(j, r, w)]);
                    o[0][r] = q.a;
                    o[1][r] = q.b;
                }
                stage_twiddle<T, M, true, K - 1, 2>(o, j, s_twi);
                dftR<8, +1, T>(o[0]);
                dftR<8, +1, T>(o[1]);
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int i = j + r * (M / 8);
                    if (i < n) Yspec[sbase + static_cast<size_t>(i) * hp + vv] = o[0][r];
                    const int x = (i + c) & (M - 1);
                    if (x < n) Bspec[sbase + static_cast<size_t>(x) * hp + vv] = o[1][r];
                }
            }
        }
    }
}

// ------------------------------------------------------------------ pass 3
template <typename T, int M>
__global__ void __launch_bounds__(TileGeom<T, M>::NT, TileGeom<T, M>::MINB)
mc_pass3(const MCIn<T> in, int sample0, int count, const cplx<T>* __restrict__ Aspec,
         const cplx<T>* __restrict__ Bspec, gtd_sample_stats* __restrict__ stats,
         const cplx<T>* __restrict__ g_tw, T* __restrict__ out, T rand_scale, int with_rand) {
    using Gm = MCGeom<T, M>;
    constexpr int n = Gm::n, c = Gm::c, h = Gm::h, L = Gm::L, LP = Gm::LP, NT = Gm::NT;
    constexpr int hp = Gm::hp;
    constexpr int RB = (n + L - 1) / L;
    constexpr int EPT = (L * h + NT - 1) / NT;
    constexpr int EPO = (L * n + NT - 1) / NT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_tw = tile + M * LP;
    double* red = reinterpret_cast<double*>(s_tw + M);

    load_twiddles<T, M, NT>(s_tw, g_tw);
    for (int item = blockIdx.x; item < count * RB; item += gridDim.x) {
        const int s = item / RB;
        const int x0 = (item - s * RB) * L;
        const size_t sg = static_cast<size_t>(sample0) + s;

        cplx<T> yv[EPT], rv[EPT];
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            const int idx = threadIdx.x + k * NT;
            const int l = idx / h, v = idx - l * h, x = x0 + l;
            yv[k] = rv[k] = mk<T>(T(0), T(0));
            if (idx < L * h && x < n) {
                const size_t o = (static_cast<size_t>(s) * n + x) * hp + v;
                yv[k] = Aspec[o];
                rv[k] = Bspec[o];
            }
        }
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            const int idx = threadIdx.x + k * NT;
            if (idx >= L * h) break;
            const int l = idx / h, v = idx - l * h;
            const cplx<T> y = yv[k], r = rv[k];
            if (v == 0 || v == n) {
                tile[v * LP + l] = mk<T>(y.x, r.x);
            } else {
                tile[v * LP + l] = mk<T>(y.x - r.y, y.y + r.x);
                tile[(M - v) * LP + l] = mk<T>(y.x + r.y, r.x - y.y);
            }
        }
        const double n2 = double(n) * double(n);
        const double mu_s = stats[sg].sum_leak / n2;
        const T scale = with_rand ? T(stats[sg].sum_applied * double(rand_scale)) : T(0);
        const T inv = T(1.0 / (double(M) * double(M)));
        const T* Nm = in.nn(sg);
        const T* V = in.v(sg);
        __syncthreads();
        tile_fft<T, M, L, LP, NT, +1>(tile, s_tw);
        T nv[EPO], vv[EPO];
#pragma unroll
        for (int k = 0; k < EPO; ++k) {
            const int idx = threadIdx.x + k * NT;
            const int l = idx / n, j = idx - l * n, x = x0 + l;
            nv[k] = vv[k] = T(0);
            if (idx < L * n && x < n) {
                nv[k] = Nm[x * n + j];
                vv[k] = V[x * n + j];
            }
        }

        T part_t = T(0), mxt = T(0);
        int bad = 0;
        const T mu_t = T(mu_s);
#pragma unroll
        for (int k = 0; k < EPO; ++k) {
            const int idx = threadIdx.x + k * NT;
            const int l = idx / n, j = idx - l * n, x = x0 + l;
            if (idx >= L * n || x >= n) continue;
            const T yd = tile[j * LP + l].x * inv;
            const int jr = (j - c) & (M - 1);
            const T rd = tile[jr * LP + l].y * inv;
            const T pvar = in.nom_scale * nv[k] * vv[k] - mu_t;
            T t = yd + rd * pvar * scale;
            if (!finite_(t)) bad = GTD_ST_NONFINITE;
            t = t > T(0) ? t : T(0);
            if (out) out[(sg * n + x) * n + j] = t;
            part_t += t;
            mxt = mxt > t ? mxt : t;
        }
        or_flags(&stats[sg].status, bad);
        const double ts = block_sum<NT>(double(part_t), red);
        const double tm = block_max<NT>(double(mxt), red);
        if (threadIdx.x == 0) {
            atomicAdd(&stats[sg].sum_rise, ts);
            atomicMax(&stats[sg].max_bits, static_cast<unsigned long long>(__double_as_longlong(tm)));
            if (x0 == 0) stats[sg].mu = mu_s;
        }
    }
}

// --------------------------------------------------- warp-per-row passes
// Row passes for M = 128 / 256 / 512: each warp owns one die row at a time,
// loads and stores it coalesced straight from / to registers and transforms it
// with the one-warp FFT (fft_warp.cuh): no CTA barriers, no transposing tile.
#ifndef GT_W1
#define GT_W1 16
#endif
#ifndef GT_W3
#define GT_W3 8
#endif
#ifndef GT_W1_CTAS
#define GT_W1_CTAS 2
#endif
#ifndef GT_W3_CTAS
#define GT_W3_CTAS 2
#endif
constexpr int WARPS = GT_W1;   // warps per CTA of the warp-per-row pass 1
constexpr int WARPS3 = GT_W3;  // pass 3 holds more live state: 8 warps x 2 CTAs at 128 registers
template <typename T, int CTAS>
struct WarpMinBlocks {
    static constexpr int value = sizeof(T) == 8 ? 1 : CTAS;  // fp64 lines need 128 registers
};

// Per-warp TMA staging of pass 1's row inputs (P row, V row; N = P).
template <typename T, int M>
struct P1Stage {
    static constexpr int n = M / 2;
    static constexpr unsigned NB = n * sizeof(T), BYTES = 2 * NB;
    static_assert(NB % 16 == 0, "bulk copy granularity");
    static constexpr unsigned OFF =
        ((M + n + WarpFFT<T, M>::TW1 + WARPS * WarpFFT<T, M>::SCRATCH) * sizeof(cplx<T>) + 127) / 128 * 128;
    static constexpr size_t SMEM = OFF + WARPS * (BYTES + 8);
};

template <typename T, int M, bool TMA>
__global__ void __launch_bounds__(WARPS * 32, WarpMinBlocks<T, GT_W1_CTAS>::value)
mc_pass1w(const MCIn<T> in, int sample0, int count, T* __restrict__ Areal,
          cplx<T>* __restrict__ Bspec, T* __restrict__ Srow, gtd_sample_stats* __restrict__ stats,
          const cplx<T>* __restrict__ g_tw, const cplx<T>* __restrict__ g_hs, T var_lo, T var_hi) {
    using Gm = MCGeom<T, M>;
    using WF = WarpFFT<T, M>;
    constexpr int n = Gm::n, c = Gm::c, h = Gm::h, hp = Gm::hp, P = WF::P;
    constexpr int E = n / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* s_tw = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_hs = s_tw + M;
    cplx<T>* s_tw1 = s_hs + n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    cplx<T>* scr = s_tw1 + WF::TW1 + warp * WF::SCRATCH;
    using SG = P1Stage<T, M>;
    unsigned char* stage = smem_raw + SG::OFF + warp * SG::BYTES;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem_raw + SG::OFF + WARPS * SG::BYTES) + warp;
    for (int t = threadIdx.x; t < M; t += WARPS * 32) s_tw[t] = g_tw[t];
    for (int t = threadIdx.x; t < n; t += WARPS * 32) s_hs[t] = g_hs[t];
    WF::build_tw1(s_tw1, g_tw, threadIdx.x, WARPS * 32);
    const int stride = gridDim.x * WARPS, total = count * n;
    auto request = [&](int item) {  // lane 0: the P and V rows of `item` into this warp's staging area
        const int s = item / n, x = item - s * n;
        const size_t sg = static_cast<size_t>(sample0) + s;
        mbar_expect_tx(mbar, SG::BYTES);
        bulk_g2s(stage, in.p(sg) + static_cast<size_t>(x) * n, SG::NB, mbar);
        bulk_g2s(stage + SG::NB, in.v(sg) + static_cast<size_t>(x) * n, SG::NB, mbar);
    };
    if constexpr (TMA) {
        if (lane == 0) {
            mbar_init(mbar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        const int first = blockIdx.x * WARPS + warp;
        if (lane == 0 && first < total) request(first);
    }
    __syncthreads();
    unsigned phase = 0;

    for (int item = blockIdx.x * WARPS + warp; item < total; item += stride) {
        const int s = item / n, x = item - s * n;
        const size_t sg = static_cast<size_t>(sample0) + s;
        const T* P_ = in.p(sg) + x * n;
        const T* N_ = in.nn(sg) + x * n;
        const T* V_ = in.v(sg) + x * n;
        bool n_is_p = in.N == in.P && in.sN == in.sP;
        if constexpr (TMA) {  // (the host selects TMA only when N = P)
            P_ = reinterpret_cast<const T*>(stage);
            V_ = reinterpret_cast<const T*>(stage + SG::NB);
            n_is_p = true;
            mbar_wait(mbar, phase);
            phase ^= 1u;
        }
        T pv[E], nv[E], vv[E];
#pragma unroll
        for (int t = 0; t < E; ++t) {
            const int y = lane + 32 * t;
            pv[t] = P_[y];
            vv[t] = V_[y];
            nv[t] = n_is_p ? pv[t] : N_[y];
        }
        T part_l = T(0), part_a = T(0);
        int bad = 0;
        T av[E], lv[E];  // applied / leakage row, element lane + 32 t
        // Input checks on bit patterns, one integer min / max per value: a finite
        // non-negative power has bits <= max-finite (-0.0 and anything else above
        // that take the exact check below); 0 < var_lo <= var <= var_hi is an
        // interval of bit patterns (negatives and NaNs fall outside it).
        using U = typename BitsOf<T>::U;
        U pmax = 0, vmin = ~U(0), vmax = 0;
#pragma unroll
        for (int t = 0; t < E; ++t) {
            pmax = max(pmax, BitsOf<T>::get(pv[t]));
            if (!n_is_p) pmax = max(pmax, BitsOf<T>::get(nv[t]));
            vmin = min(vmin, BitsOf<T>::get(vv[t]));
            vmax = max(vmax, BitsOf<T>::get(vv[t]));
            lv[t] = in.nom_scale * nv[t] * vv[t];
            av[t] = pv[t] + lv[t];
            part_l += lv[t];
            part_a += av[t];
        }
        if (pmax > BitsOf<T>::get(Real<T>::max())) {
#pragma unroll
            for (int t = 0; t < E; ++t)  // NaN fails both compares, +-inf one: !(x >= 0) || !isfinite(x)
                if (!(pv[t] >= T(0) && pv[t] <= Real<T>::max()) || !(nv[t] >= T(0) && nv[t] <= Real<T>::max()))
                    bad |= GTD_ST_BAD_POWER;
        }
        if (vmin < BitsOf<T>::get(var_lo) || vmax > BitsOf<T>::get(var_hi)) bad |= GTD_ST_BAD_VAR;
        if constexpr (TMA) {
            // the staged rows are consumed: request the warp's next row
            __syncwarp();
            if (lane == 0 && item + stride < total) {
                fence_proxy_async();
                request(item + stride);
            }
        }
        // Row-symmetrised leakage for q (symmetric_multiplier, spectral.cpp:167-185):
        // S[dv] = L[min(c + dv, n - 1)] + L[max(c - dv, 0)], c = 16 E. For dv = lane + 32 k < c,
        // L[c + dv] is this lane's lv[E/2 + k] and L[c - dv] is lane 32 - lane's lv[E/2 - 1 - k]
        // (lane 0: its own lv[E/2 - k]); for dv >= c both indices clamp: L[n - 1] + L[0].
        {
            T* Srow_x = Srow + (static_cast<size_t>(s) * n + x) * hp;
            const T cst = __shfl_sync(0xffffffffu, lv[E - 1], 31) + __shfl_sync(0xffffffffu, lv[0], 0);
#pragma unroll
            for (int k = 0; k < (hp + 31) / 32; ++k) {
                const int v = lane + 32 * k;
                T val;
                if (k < E / 2) {
                    const T mir = __shfl_sync(0xffffffffu, lv[k < E / 2 ? E / 2 - 1 - k : 0], (32 - lane) & 31);
                    val = lv[k < E / 2 ? E / 2 + k : 0] + (lane == 0 ? lv[k < E / 2 ? E / 2 - k : 0] : mir);
                } else {
                    val = v < h ? cst : T(0);
                }
                if (v < hp) Srow_x[v] = val;
            }
        }
        // z[i] = mirror(applied)[i] + i * centre-embedded(p_leak0)[i], i = lane + 32 k,
        // from registers: mirror(i) = M-1-i = (31 - lane) + 32 (P-1-k) for k >= E
        // (one shuffle); the centre embedding keeps the lane (t = k + E/2, k - 3E/2).
        cplx<T> z[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
            const T re = k < E ? av[k] : __shfl_xor_sync(0xffffffffu, av[P - 1 - k], 31);
            const T im = k < E / 2 ? lv[k + E / 2] : (k >= P - E / 2 ? lv[k - (P - E / 2)] : T(0));
            z[k] = mk<T>(re, im);
        }
        __syncwarp();
        WF::template run<-1>(z, scr, s_tw, s_tw1, lane);
        __syncwarp();
#pragma unroll
        for (int m1 = 0; m1 < P; ++m1) scr[WF::out_pos(lane, m1)] = z[m1];
        __syncwarp();
        // split into the two real-input half spectra (A as its real DCT part)
        T* A_x = Areal + (static_cast<size_t>(s) * n + x) * hp;
        cplx<T>* B_x = Bspec + (static_cast<size_t>(s) * n + x) * hp;
        for (int v = lane; v < hp; v += 32) {
            T Ar = T(0);
            cplx<T> B = mk<T>(T(0), T(0));
            if (v < h) {
                const cplx<T> Z = scr[v];
                const cplx<T> Zc = cconj<T>(scr[(M - v) & (M - 1)]);
                if (v < n) Ar = dct_part<T>(Z, Zc, s_hs[v]);
                B = mk<T>(T(0.5) * (Z.y - Zc.y), T(-0.5) * (Z.x - Zc.x));
            }
            A_x[v] = Ar;
            B_x[v] = B;
        }
        or_flags(&stats[sg].status, bad);
        const double tl = warp_sum(double(part_l)), ta = warp_sum(double(part_a));
        if (lane == 0) {
            atomicAdd(&stats[sg].sum_leak, tl);
            atomicAdd(&stats[sg].sum_applied, ta);
        }
        __syncwarp();
    }
}

// Per-warp TMA staging of pass 3's row inputs: Y row, R row (hp complex each),
// N row, V row (n reals each), contiguous in global memory per row.
template <typename T, int M>
struct P3Stage {
    static constexpr int n = M / 2, hp = MCGeom<T, M>::hp;
    static constexpr unsigned YB = hp * sizeof(cplx<T>), NB = n * sizeof(T);
    static constexpr unsigned BYTES = 2 * YB + 2 * NB;  // per warp; every segment a multiple of 16 B
    // staging offset in pass 3's shared memory: after the twiddles and the warps' scratch
    static constexpr unsigned OFF =
        ((M + WarpFFT<T, M>::TW1 + WARPS3 * WarpFFT<T, M>::SCRATCH) * sizeof(cplx<T>) + 127) / 128 * 128;
    static constexpr size_t SMEM = OFF + WARPS3 * (BYTES + 8);
    static_assert(YB % 16 == 0 && NB % 16 == 0, "bulk copy granularity");
};

template <typename T, int M, bool TMA>
__global__ void __launch_bounds__(WARPS3 * 32, WarpMinBlocks<T, GT_W3_CTAS>::value)
mc_pass3w(const MCIn<T> in, int sample0, int count, const cplx<T>* __restrict__ Aspec,
          const cplx<T>* __restrict__ Bspec, gtd_sample_stats* __restrict__ stats,
          const cplx<T>* __restrict__ g_tw, T* __restrict__ out, T rand_scale, int with_rand) {
    using Gm = MCGeom<T, M>;
    using WF = WarpFFT<T, M>;
    using SG = P3Stage<T, M>;
    constexpr int n = Gm::n, c = Gm::c, hp = Gm::hp, P = WF::P;
    constexpr int E = n / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* s_tw = reinterpret_cast<cplx<T>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    cplx<T>* s_tw1 = s_tw + M;
    cplx<T>* scr = s_tw1 + WF::TW1 + warp * WF::SCRATCH;
    // TMA: [WARPS3][SG::BYTES] staging after the scratch, then one mbarrier per warp
    unsigned char* stage = smem_raw + SG::OFF + warp * SG::BYTES;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(stage + (WARPS3 - warp) * SG::BYTES) + warp;
    for (int t = threadIdx.x; t < M; t += WARPS3 * 32) s_tw[t] = g_tw[t];
    WF::build_tw1(s_tw1, g_tw, threadIdx.x, WARPS3 * 32);
    const int stride = gridDim.x * WARPS3, total = count * n;
    // lane 0 requests the four row segments of `item` into this warp's staging area
    auto request = [&](int item) {
        const int s = item / n, x = item - s * n;
        const size_t sg = static_cast<size_t>(sample0) + s;
        const size_t so = (static_cast<size_t>(s) * n + x) * hp;
        mbar_expect_tx(mbar, SG::BYTES);
        bulk_g2s(stage, Aspec + so, SG::YB, mbar);
        bulk_g2s(stage + SG::YB, Bspec + so, SG::YB, mbar);
        bulk_g2s(stage + 2 * SG::YB, in.nn(sg) + static_cast<size_t>(x) * n, SG::NB, mbar);
        bulk_g2s(stage + 2 * SG::YB + SG::NB, in.v(sg) + static_cast<size_t>(x) * n, SG::NB, mbar);
    };
    if constexpr (TMA) {
        if (lane == 0) {
            mbar_init(mbar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        const int first = blockIdx.x * WARPS3 + warp;
        if (lane == 0 && first < total) request(first);
    }
    __syncthreads();
    const T inv = T(1.0 / (double(M) * double(M)));
    unsigned phase = 0;

    for (int item = blockIdx.x * WARPS3 + warp; item < total; item += stride) {
        const int s = item / n, x = item - s * n;
        const size_t sg = static_cast<size_t>(sample0) + s;
        const cplx<T>* Y_x;
        const cplx<T>* R_x;
        const T* N_;
        const T* V_;
        if constexpr (TMA) {
            Y_x = reinterpret_cast<const cplx<T>*>(stage);
            R_x = reinterpret_cast<const cplx<T>*>(stage + SG::YB);
            N_ = reinterpret_cast<const T*>(stage + 2 * SG::YB);
            V_ = reinterpret_cast<const T*>(stage + 2 * SG::YB + SG::NB);
            mbar_wait(mbar, phase);
            phase ^= 1u;
        } else {
            Y_x = Aspec + (static_cast<size_t>(s) * n + x) * hp;
            R_x = Bspec + (static_cast<size_t>(s) * n + x) * hp;
            N_ = in.nn(sg) + x * n;
            V_ = in.v(sg) + x * n;
        }
        // epilogue inputs requested up front (one exposed round trip per row)
        T nv[E], vv[E];
#pragma unroll
        for (int t = 0; t < E; ++t) {
            nv[t] = N_[lane + 32 * t];
            vv[t] = V_[lane + 32 * t];
        }
        // Z = Y + i R over the full line from the Hermitian half spectra
        cplx<T> z[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
            const int v = lane + 32 * k;
            const int w = v <= n ? v : M - v;
            const cplx<T> y = Y_x[w], r = R_x[w];
            if (v == 0 || v == n)
                z[k] = mk<T>(y.x, r.x);
            else if (v < n)
                z[k] = mk<T>(y.x - r.y, y.y + r.x);
            else
                z[k] = mk<T>(y.x + r.y, r.x - y.y);
        }
        const double n2 = double(n) * double(n);
        const double mu_s = stats[sg].sum_leak / n2;
        const T scale = with_rand ? T(stats[sg].sum_applied * double(rand_scale)) : T(0);
        const T mu_t = T(mu_s);
        T pvs[E];  // p_var * sum(applied) * rand_scale: consumes the staged N, V rows
#pragma unroll
        for (int t = 0; t < E; ++t) pvs[t] = (in.nom_scale * nv[t] * vv[t] - mu_t) * scale;
        if constexpr (TMA) {
            // the staging area is free once every lane has consumed it: request the next row
            __syncwarp();
            if (lane == 0 && item + stride < total) {
                fence_proxy_async();
                request(item + stride);
            }
        }
        WF::template run<+1>(z, scr, s_tw, s_tw1, lane);
        __syncwarp();
#pragma unroll
        for (int m1 = 0; m1 < P; ++m1) scr[WF::out_pos(lane, m1)] = z[m1];
        __syncwarp();
        T part = T(0), mxt = T(0);
        int bad = 0;
        T* O_x = out ? out + (sg * n + x) * n : nullptr;
#pragma unroll
        for (int t = 0; t < E; ++t) {
            const int f = lane + 32 * t;
            const T yd = scr[f].x * inv;
            const T rd = scr[(f - c) & (M - 1)].y * inv;
            T tt = yd + rd * pvs[t];
            if (!finite_(tt)) bad = GTD_ST_NONFINITE;
            tt = tt > T(0) ? tt : T(0);
            if (O_x) O_x[f] = tt;
            part += tt;
            mxt = mxt > tt ? mxt : tt;
        }
        or_flags(&stats[sg].status, bad);
        const double ts = warp_sum(double(part));
        const double tm = double(warp_max_t(mxt));  // max is exact in T
        if (lane == 0) {
            atomicAdd(&stats[sg].sum_rise, ts);
            atomicMax(&stats[sg].max_bits, static_cast<unsigned long long>(__double_as_longlong(tm)));
            if (x == 0) stats[sg].mu = mu_s;
        }
        __syncwarp();
    }
}

template <typename T, int M>
constexpr bool use_warp_rows() {
    return M == 128 || M == 256 || M == 512;
}

__global__ void mc_finalize(gtd_sample_stats* stats, int sample0, int count, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    gtd_sample_stats& st = stats[sample0 + i];
    st.max_rise = __longlong_as_double(static_cast<long long>(st.max_bits));
    st.mean_rise = st.sum_rise / (double(n) * double(n));
}

// ------------------------------------------------------------------ host side
template <typename T, int M>
struct MCLaunch {
    using Gm = MCGeom<T, M>;
    static size_t smem1() { return sizeof(cplx<T>) * (M * Gm::LP + M) + 64 * sizeof(double); }
    static constexpr int GA2 = Gm::W >= 2 ? Gm::W / 2 : 1;
    static size_t smem2() {
        constexpr int FS = FwdLayout<T, GA2, M>::SIZE, IS = InvLayout<Gm::W, M>::SIZE;
        return sizeof(cplx<T>) * ((FS > IS ? FS : IS) + StageTw<M, false>::SIZE + StageTw<M, true>::SIZE + M) +
               sizeof(T) * Gm::n * Gm::W;
    }
    static size_t smem3() { return sizeof(cplx<T>) * (M * Gm::LP + M) + 64 * sizeof(double); }
    static size_t smemw(bool tma) {
        if constexpr (use_warp_rows<T, M>())
            return tma ? P1Stage<T, M>::SMEM
                       : sizeof(cplx<T>) * (M + M / 2 + WarpFFT<T, M>::TW1 + WARPS * WarpFFT<T, M>::SCRATCH);
        else
            return 0;
    }
    static size_t smemw3(bool tma) {
        if constexpr (use_warp_rows<T, M>())
            return tma ? P3Stage<T, M>::SMEM
                       : sizeof(cplx<T>) * (M + WarpFFT<T, M>::TW1 + WARPS3 * WarpFFT<T, M>::SCRATCH);
        else
            return 0;
    }

    static int run(const gtd_greens* g, const MCIn<T>& in, int batch, const gtd_mc_opts* o,
                   T* out, gtd_sample_stats* stats, void* scratch, int chunk, cudaStream_t st,
                   gtd_mark_fn mark, void* ctx) {
        constexpr int n = Gm::n, hp = Gm::hp, L = Gm::L, NT = Gm::NT, W = Gm::W;
        constexpr int RB = (n + L - 1) / L, CT = hp / W;
        static int res[3] = {0, 0, 0};
        static int sms = 0;
        if (!sms) {
            cudaFuncSetAttribute(mc_pass1<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem1()));
            cudaFuncSetAttribute(mc_pass2<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2()));
            cudaFuncSetAttribute(mc_pass3<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem3()));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[0], mc_pass1<T, M>, NT, smem1());
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[1], mc_pass2<T, M>, Gm::NT2, smem2());
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[2], mc_pass3<T, M>, NT, smem3());
            if constexpr (use_warp_rows<T, M>()) {
                cudaFuncSetAttribute(mc_pass1w<T, M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smemw(false)));
                cudaFuncSetAttribute(mc_pass1w<T, M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smemw(true)));
                cudaFuncSetAttribute(mc_pass3w<T, M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smemw3(false)));
                cudaFuncSetAttribute(mc_pass3w<T, M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smemw3(true)));
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[0], mc_pass1w<T, M, true>, WARPS * 32,
                                                              smemw(true));
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[2], mc_pass3w<T, M, true>, WARPS3 * 32,
                                                              smemw3(true));
            }
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            for (int& r : res) r = r < 1 ? 1 : r;
        }
        const size_t per = static_cast<size_t>(n) * hp;
        const cplx<T>* hs = reinterpret_cast<const cplx<T>*>(g->hs);
        const cplx<T>* tw = reinterpret_cast<const cplx<T>*>(g->tw);
        const T var_lo = T(exp(-o->exponent_cap)), var_hi = T(exp(o->exponent_cap));
        // Overlap (GT_MC_OVERLAP=1): the chunk's scratch is split into two slots whose
        // sub-chunks run on two streams, every pass on a one-CTA-per-SM grid, so the
        // SM-issue-bound column pass of one slot shares the SMs with the HBM-bound row
        // passes of the other.
        static int ovl = -1;
        static cudaStream_t aux = nullptr;
        static cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
        if (ovl < 0) {
            const char* e = getenv("GT_MC_OVERLAP");
            ovl = e ? atoi(e) : 0;
            if (ovl) {
                cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking);
                cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming);
                cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming);
            }
        }
        const int slots = (ovl && chunk >= 2) ? 2 : 1;
        const int sub = chunk / slots;
        const int cpsm = slots == 2 ? ovl : 0;  // CTAs per SM per pass under overlap
        auto grid = [&](int items, int r) {
            const int rr = cpsm > 0 && cpsm < r ? cpsm : r;
            return items < sms * rr ? items : sms * rr;
        };
        // TMA row staging in pass 3 needs 16-byte aligned N / V rows (the spectra always are)
        auto al16 = [](const void* p, long long stride_elems) {
            return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && ((stride_elems * sizeof(T)) % 16 == 0);
        };
#ifndef GT_P3_TMA
#define GT_P3_TMA 1
#endif
        const bool tma3 = GT_P3_TMA && al16(in.N, in.sN) && al16(in.V, in.sV) && (n * sizeof(T)) % 16 == 0;
        // pass 1 stages P and V rows and takes N = P (the Monte-Carlo entries' nominal leakage map)
        const bool tma1 = GT_P3_TMA && in.N == in.P && in.sN == in.sP && al16(in.P, in.sP) && al16(in.V, in.sV) &&
                          (n * sizeof(T)) % 16 == 0;
        cudaMemsetAsync(stats, 0, sizeof(gtd_sample_stats) * batch, st);
        if (slots == 2) {
            cudaEventRecord(ev_fork, st);
            cudaStreamWaitEvent(aux, ev_fork, 0);
        }
        for (int s0 = 0, k = 0; s0 < batch; s0 += sub, ++k) {
            const int cnt = batch - s0 < sub ? batch - s0 : sub;
            const int slot = k % slots;
            cudaStream_t ss = slot == 0 ? st : aux;
            gtd_mark_fn mk_ = slot == 0 ? mark : nullptr;
            unsigned char* base = static_cast<unsigned char*>(scratch) +
                                  static_cast<size_t>(slot) * sub * gtd_mc_scratch_bytes_per_sample(n, sizeof(T) == 8);
            cplx<T>* A = reinterpret_cast<cplx<T>*>(base);  // Y (pass 2 -> pass 3)
            cplx<T>* B = A + per * sub;                     // B (pass 1 -> 2), R (pass 2 -> 3)
            T* S = reinterpret_cast<T*>(B + per * sub);      // row-symmetrised leakage
            T* Ar = S + per * sub;                           // real DCT part of A (pass 1 -> 2)
            if (mk_) mk_(ctx, 0, ss);
            if constexpr (use_warp_rows<T, M>())
            {
                if (tma1)
                    mc_pass1w<T, M, true><<<grid((cnt * n + WARPS - 1) / WARPS, res[0]), WARPS * 32, smemw(true), ss>>>(
                        in, s0, cnt, Ar, B, S, stats, tw, hs, var_lo, var_hi);
                else
                    mc_pass1w<T, M, false><<<grid((cnt * n + WARPS - 1) / WARPS, res[0]), WARPS * 32, smemw(false),
                                             ss>>>(in, s0, cnt, Ar, B, S, stats, tw, hs, var_lo, var_hi);
            }
            else
                mc_pass1<T, M><<<grid(cnt * RB, res[0]), NT, smem1(), ss>>>(in, s0, cnt, Ar, B, S, stats, tw, hs,
                                                                             var_lo, var_hi);
            if (mk_) mk_(ctx, 1, ss);
            mc_pass2<T, M><<<grid(cnt * CT, res[1]), Gm::NT2, smem2(), ss>>>(
                in, s0, cnt, Ar, A, B, S, stats, tw, hs, static_cast<const T*>(g->fg), T(g->alpha), T(g->beta),
                o->mu_per_sample, T(g->mu_fixed));
            if (mk_) mk_(ctx, 2, ss);
            if constexpr (use_warp_rows<T, M>())
            {
                if (tma3)
                    mc_pass3w<T, M, true><<<grid((cnt * n + WARPS3 - 1) / WARPS3, res[2]), WARPS3 * 32,
                                            smemw3(true), ss>>>(in, s0, cnt, A, B, stats, tw, out,
                                                                T(g->rand_scale), o->with_rand);
                else
                    mc_pass3w<T, M, false><<<grid((cnt * n + WARPS3 - 1) / WARPS3, res[2]), WARPS3 * 32,
                                             smemw3(false), ss>>>(in, s0, cnt, A, B, stats, tw, out,
                                                                  T(g->rand_scale), o->with_rand);
            }
            else
                mc_pass3<T, M><<<grid(cnt * RB, res[2]), NT, smem3(), ss>>>(in, s0, cnt, A, B, stats, tw, out,
                                                                             T(g->rand_scale), o->with_rand);
            if (mk_) mk_(ctx, 3, ss);
        }
        if (slots == 2) {
            cudaEventRecord(ev_join, aux);
            cudaStreamWaitEvent(st, ev_join, 0);
        }
        mc_finalize<<<(batch + 127) / 128, 128, 0, st>>>(stats, 0, batch, n);
        return static_cast<int>(cudaGetLastError());
    }
};

}  // namespace gtb

using namespace gtb;

template <typename T>
static int dispatch_mc(const gtd_greens* g, const gtd_mc_in* i, int batch, const gtd_mc_opts* o,
                       void* out, gtd_sample_stats* stats, void* scratch, int chunk,
                       cudaStream_t st, gtd_mark_fn mark, void* ctx) {
    MCIn<T> in;
    in.P = static_cast<const T*>(i->P);
    in.N = static_cast<const T*>(i->N);
    in.V = static_cast<const T*>(i->V);
    in.sP = i->sP;
    in.sN = i->sN;
    in.sV = i->sV;
    in.nom_scale = T(i->nom_scale);
    T* O = static_cast<T*>(out);
    switch (g->m) {
        case 32: return MCLaunch<T, 32>::run(g, in, batch, o, O, stats, scratch, chunk, st, mark, ctx);
        case 64: return MCLaunch<T, 64>::run(g, in, batch, o, O, stats, scratch, chunk, st, mark, ctx);
        case 128: return MCLaunch<T, 128>::run(g, in, batch, o, O, stats, scratch, chunk, st, mark, ctx);
        case 256: return MCLaunch<T, 256>::run(g, in, batch, o, O, stats, scratch, chunk, st, mark, ctx);
        case 512: return MCLaunch<T, 512>::run(g, in, batch, o, O, stats, scratch, chunk, st, mark, ctx);
        case 1024: return MCLaunch<T, 1024>::run(g, in, batch, o, O, stats, scratch, chunk, st, mark, ctx);
        case 2048: return MCLaunch<T, 2048>::run(g, in, batch, o, O, stats, scratch, chunk, st, mark, ctx);
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}

template <typename T>
static int geom_hp(int m) {
    switch (m) {
        case 32: return MCGeom<T, 32>::hp;
        case 64: return MCGeom<T, 64>::hp;
        case 128: return MCGeom<T, 128>::hp;
        case 256: return MCGeom<T, 256>::hp;
        case 512: return MCGeom<T, 512>::hp;
        case 1024: return MCGeom<T, 1024>::hp;
        case 2048: return MCGeom<T, 2048>::hp;
        default: return -1;
    }
}

extern "C" {

int gtd_padded_width(int n, int fp64) { return fp64 ? geom_hp<double>(2 * n) : geom_hp<float>(2 * n); }

size_t gtd_mc_scratch_bytes_per_sample(int n, int fp64) {
    const int hp = gtd_padded_width(n, fp64);
    if (hp < 0) return 0;
    const size_t cb = fp64 ? 16 : 8, rb = fp64 ? 8 : 4;
    return static_cast<size_t>(n) * hp * (2 * cb + 2 * rb);
}

int gtd_mc_launch_count(int batch, int chunk) {
    const int chunks = (batch + chunk - 1) / chunk;
    return chunks * 3 + 1;  // pass1, pass2, pass3 per chunk + one finalize (plus one memset node)
}

int gtd_mc_batch(const gtd_greens* g, const gtd_mc_in* in, int batch, const gtd_mc_opts* opts,
                 void* out, gtd_sample_stats* stats, void* scratch, int chunk,
                 cudaStream_t stream, gtd_mark_fn mark, void* ctx) {
    if (!g || !in || batch < 1 || chunk < 1) return static_cast<int>(cudaErrorInvalidValue);
    return g->fp64 ? dispatch_mc<double>(g, in, batch, opts, out, stats, scratch, chunk, stream, mark, ctx)
                   : dispatch_mc<float>(g, in, batch, opts, out, stats, scratch, chunk, stream, mark, ctx);
}

}  // extern "C"
