// fft_tile.cuh — shared-memory tile FFT engine for sm_100a.
//
// A "tile" is a block of L independent complex lines of power-of-two length M
// held in shared memory with the LINE index fastest: element j of line l lives
// at tile[j * LP + l] (LP >= L is the padded pitch). Warp lanes are mapped
// across lines, so every butterfly load/store of a warp touches 16 (fp32) or
// 8 (fp64) consecutive complex values per row: exactly the minimum number of
// shared-memory wavefronts whatever the Stockham index permutation, i.e. the
// engine is bank-conflict free by construction.
//
// The transform is a Stockham autosort FFT (natural order in and out) with
// radix-8 register butterflies and one trailing radix-2/4 stage when log2(M)
// is not a multiple of 3. Twiddles come from a per-CTA shared table
// tw[t] = exp(-2*pi*i*t/M) computed on the host in fp64.
//
// Convention (reference spectral.hpp:12-20): forward = unnormalised sum with
// exp(-2*pi*i*k*j/M); inverse = exp(+...) WITHOUT the 1/M factor (callers fold
// the 1/m^2 into their epilogue).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace gtb {

template <typename T>
struct V2;
template <>
struct V2<float> {
    using type = float2;
};
template <>
struct V2<double> {
    using type = double2;
};
template <typename T>
using cplx = typename V2<T>::type;

template <typename T>
__device__ __forceinline__ cplx<T> mk(T x, T y) {
    cplx<T> r;
    r.x = x;
    r.y = y;
    return r;
}
template <typename T>
__device__ __forceinline__ cplx<T> cadd(cplx<T> a, cplx<T> b) {
    return mk<T>(a.x + b.x, a.y + b.y);
}
template <typename T>
__device__ __forceinline__ cplx<T> csub(cplx<T> a, cplx<T> b) {
    return mk<T>(a.x - b.x, a.y - b.y);
}
template <typename T>
__device__ __forceinline__ cplx<T> cmul(cplx<T> a, cplx<T> b) {
    return mk<T>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
template <typename T>
__device__ __forceinline__ cplx<T> cconj(cplx<T> a) {
    return mk<T>(a.x, -a.y);
}
template <typename T>
__device__ __forceinline__ cplx<T> cscale(cplx<T> a, T s) {
    return mk<T>(a.x * s, a.y * s);
}
template <typename T>
__device__ __forceinline__ T cabs2(cplx<T> a) {
    return a.x * a.x + a.y * a.y;
}
// a / b for complex b
template <typename T>
__device__ __forceinline__ cplx<T> cdiv(cplx<T> a, cplx<T> b) {
    T d = T(1) / cabs2<T>(b);
    return mk<T>((a.x * b.x + a.y * b.y) * d, (a.y * b.x - a.x * b.y) * d);
}
// multiply by (SIGN * i): SIGN = -1 gives -i, +1 gives +i
template <int SIGN, typename T>
__device__ __forceinline__ cplx<T> mul_si(cplx<T> a) {
    return SIGN < 0 ? mk<T>(a.y, -a.x) : mk<T>(-a.y, a.x);
}

// ---- packed FP32 (sm_100 FADD2 / FMUL2 / FFMA2): a complex float is one
// register pair, so every complex add is ONE instruction and a complex multiply
// three; the SASS operand swizzle (.F32x2.LO_HI) and scalar broadcast (.F32)
// make the +-i rotations and the real scalings free inside an FFMA2. The
// arithmetic is the scalar one (IEEE round-to-nearest per lane); only the
// contraction of a complex multiply into FMA differs from the scalar path.
// Off by default; a translation unit opts in by defining GT_PACKED_F32 1 before
// including this header (mc_rows.cu: the warp row passes gain; the latency-bound
// column pass measured slower and stays scalar).
#ifndef GT_PACKED_F32
#define GT_PACKED_F32 0
#endif
#if GT_PACKED_F32
template <>
__device__ __forceinline__ float2 cadd<float>(float2 a, float2 b) {
    return __fadd2_rn(a, b);
}
template <>
__device__ __forceinline__ float2 csub<float>(float2 a, float2 b) {
    return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
// a b = (ax, ay) bx + (ay, ax) (-by, by): the pair (-by, by) is one FMUL2 of a
// broadcast, shared by every line a twiddle multiplies (common subexpression).
template <>
__device__ __forceinline__ float2 cmul<float>(float2 a, float2 b) {
    const float2 bn = __fmul2_rn(make_float2(b.y, b.y), make_float2(-1.0f, 1.0f));
    return __ffma2_rn(make_float2(a.y, a.x), bn, __fmul2_rn(a, make_float2(b.x, b.x)));
}
template <>
__device__ __forceinline__ float2 cscale<float>(float2 a, float s) {
    return __fmul2_rn(a, make_float2(s, s));
}
#endif

// a + s (SIGN i) d  (SIGN = -1: -i d = (d.y, -d.x); +1: i d = (-d.y, d.x))
template <int SIGN, typename T>
__device__ __forceinline__ cplx<T> add_rot(cplx<T> a, cplx<T> d, T s) {
#if GT_PACKED_F32
    if constexpr (sizeof(T) == 4)
        return __ffma2_rn(make_float2(d.y, d.x), SIGN < 0 ? make_float2(s, -s) : make_float2(-s, s), a);
    else
#endif
        return SIGN < 0 ? mk<T>(a.x + s * d.y, a.y - s * d.x) : mk<T>(a.x - s * d.y, a.y + s * d.x);
}
// p + s S (complex by real)
template <typename T>
__device__ __forceinline__ cplx<T> add_scaled(cplx<T> p, cplx<T> S, T s) {
#if GT_PACKED_F32
    if constexpr (sizeof(T) == 4)
        return __ffma2_rn(S, make_float2(s, s), p);
    else
#endif
        return mk<T>(fma(s, S.x, p.x), fma(s, S.y, p.y));
}

constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }

// ---------------------------------------------------------------- butterflies
template <int SIGN, typename T>
__device__ __forceinline__ void dft2(cplx<T>* v) {
    cplx<T> a = v[0], b = v[1];
    v[0] = cadd<T>(a, b);
    v[1] = csub<T>(a, b);
}

template <int SIGN, typename T>
__device__ __forceinline__ void dft4(cplx<T>* v) {
    cplx<T> a0 = cadd<T>(v[0], v[2]), a1 = csub<T>(v[0], v[2]);
    cplx<T> b0 = cadd<T>(v[1], v[3]), d = csub<T>(v[1], v[3]);
    v[0] = cadd<T>(a0, b0);
    v[2] = csub<T>(a0, b0);
    v[1] = add_rot<SIGN, T>(a1, d, T(1));   // a1 + (SIGN i) d
    v[3] = add_rot<SIGN, T>(a1, d, T(-1));  // a1 - (SIGN i) d
}

// Odd half of the radix-8 DIF butterfly: a4..a7 are the differences v[k] - v[k+4];
// a5 and a7 still owe their W8 factors (1 +- i)/sqrt2 and (-1 +- i)/sqrt2. The
// 1/sqrt2 is folded into FFMAs of the last layer instead of two FMULs each.
template <int SIGN, typename T>
__device__ __forceinline__ void dft8_odd(cplx<T> a4, cplx<T> a5, cplx<T> a6, cplx<T> a7, cplx<T>& o0, cplx<T>& o1,
                                         cplx<T>& o2, cplx<T>& o3) {
    const T r = T(0.70710678118654752440084436210485);
    // unscaled W8^1 a5 = (1 + SIGN i) a5 and W8^3 a7 = (-1 + SIGN i) a7
    const cplx<T> A5 = add_rot<SIGN, T>(a5, a5, T(1));
    const cplx<T> A7 = add_rot<SIGN, T>(mk<T>(-a7.x, -a7.y), a7, T(1));
    const cplx<T> p0 = add_rot<SIGN, T>(a4, a6, T(1)), p1 = add_rot<SIGN, T>(a4, a6, T(-1));  // a4 +- (SIGN i) a6
    const cplx<T> S = cadd<T>(A5, A7), Dd = csub<T>(A5, A7);  // D = (SIGN i) Dd
    o0 = add_scaled<T>(p0, S, r);
    o2 = add_scaled<T>(p0, S, -r);
    o1 = add_rot<SIGN, T>(p1, Dd, r);
    o3 = add_rot<SIGN, T>(p1, Dd, -r);
}

template <int SIGN, typename T>
__device__ __forceinline__ void dft8(cplx<T>* v) {
    // radix-2 DIF layer, then DFT4 of the sums (even outputs) and of the twiddled
    // differences (odd outputs)
    cplx<T> e[4] = {cadd<T>(v[0], v[4]), cadd<T>(v[1], v[5]), cadd<T>(v[2], v[6]), cadd<T>(v[3], v[7])};
    const cplx<T> a4 = csub<T>(v[0], v[4]), a5 = csub<T>(v[1], v[5]), a6 = csub<T>(v[2], v[6]),
                  a7 = csub<T>(v[3], v[7]);
    dft4<SIGN, T>(e);
    dft8_odd<SIGN, T>(a4, a5, a6, a7, v[1], v[3], v[5], v[7]);
    v[0] = e[0];
    v[2] = e[1];
    v[4] = e[2];
    v[6] = e[3];
}

// DFT8 of an input whose slots 2..5 are zero (never read): the first radix-2
// layer degenerates to copies / negations.
template <int SIGN, typename T>
__device__ __forceinline__ void dft8_outer_only(cplx<T>* v) {
    cplx<T> e[4] = {v[0], v[1], v[6], v[7]};
    const cplx<T> a4 = v[0], a5 = v[1], a6 = mk<T>(-v[6].x, -v[6].y), a7 = mk<T>(-v[7].x, -v[7].y);
    dft4<SIGN, T>(e);
    dft8_odd<SIGN, T>(a4, a5, a6, a7, v[1], v[3], v[5], v[7]);
    v[0] = e[0];
    v[2] = e[1];
    v[4] = e[2];
    v[6] = e[3];
}

template <int SIGN, typename T>
__device__ __forceinline__ void dft16(cplx<T>* v) {
    // radix-4 x radix-4 with w16 twiddles, in place: after the first layer slot
    // n2 + 4 k1 holds a[n2][k1]; the second layer leaves X[k1 + 4 k2] in slot
    // 4 k1 + k2, undone by a compile-time register permutation.
    const T c1 = T(0.92387953251128675613), s1 = T(0.38268343236508977173);  // cos/sin(pi/8)
    const T r2 = T(0.70710678118654752440);
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
        cplx<T> q[4] = {v[n2], v[4 + n2], v[8 + n2], v[12 + n2]};
        dft4<SIGN, T>(q);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) v[n2 + 4 * k1] = q[k1];
    }
    const T sg = SIGN < 0 ? T(-1) : T(1);
    v[5] = cmul<T>(v[5], mk<T>(c1, sg * s1));     // n2=1,k1=1: w^1
    v[9] = cmul<T>(v[9], mk<T>(r2, sg * r2));     // n2=1,k1=2: w^2
    v[13] = cmul<T>(v[13], mk<T>(s1, sg * c1));   // n2=1,k1=3: w^3
    v[6] = cmul<T>(v[6], mk<T>(r2, sg * r2));     // n2=2,k1=1: w^2
    v[10] = mul_si<SIGN, T>(v[10]);               // n2=2,k1=2: w^4
    v[14] = cmul<T>(v[14], mk<T>(-r2, sg * r2));  // n2=2,k1=3: w^6
    v[7] = cmul<T>(v[7], mk<T>(s1, sg * c1));     // n2=3,k1=1: w^3
    v[11] = cmul<T>(v[11], mk<T>(-r2, sg * r2));  // n2=3,k1=2: w^6
    v[15] = cmul<T>(v[15], mk<T>(-c1, -sg * s1)); // n2=3,k1=3: w^9
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
        cplx<T> q[4] = {v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]};
        dft4<SIGN, T>(q);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) v[4 * k1 + k2] = q[k2];
    }
    cplx<T> t[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = v[i];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = t[4 * k1 + k2];
}

template <int R, int SIGN, typename T>
__device__ __forceinline__ void dftR(cplx<T>* v) {
    if constexpr (R == 16)
        dft16<SIGN, T>(v);
    else if constexpr (R == 8)
        dft8<SIGN, T>(v);
    else if constexpr (R == 4)
        dft4<SIGN, T>(v);
    else if constexpr (R == 2)
        dft2<SIGN, T>(v);
}

// ------------------------------------------------------------- tile geometry
#ifndef GT_TILE_BYTES
#define GT_TILE_BYTES 65536
#endif
// Lines per tile: a tile of GT_TILE_BYTES so several CTAs share an SM and hide
// each other's barrier / load latency.
template <typename T, int M>
struct TileGeom {
    static constexpr int CB = int(sizeof(cplx<T>));
    static constexpr int Lraw = GT_TILE_BYTES / (M * CB);
    static constexpr int L = Lraw > 32 ? 32 : (Lraw < 2 ? 2 : Lraw);
    static constexpr int LOG2M = ilog2(M);
    static constexpr int N8 = LOG2M / 3;           // radix-8 stages
    static constexpr int RLAST = 1 << (LOG2M % 3); // 1, 2 or 4
    // threads: one radix-8 pair-butterfly (two lines) per thread in the widest stage
    static constexpr int NBMIN = (M / 8) * (L / 2);
    static constexpr int NT = NBMIN >= 512 ? 512 : (NBMIN < 32 ? 32 : NBMIN);
    // resident CTAs the register budget must allow: 64 regs/thread for fp32,
    // 128 for fp64 (a pair-butterfly holds 16 complex values)
    static constexpr int REGS = sizeof(T) == 8 ? 128 : 64;
    static constexpr int MINB = (65536 / REGS) / NT < 1 ? 1 : (65536 / REGS) / NT;
};

// One Stockham stage over a whole tile, in place (all loads, barrier, stores).
template <typename T, int M, int L, int LP, int NT, int SIGN, int R, int NS>
__device__ __forceinline__ void stockham_stage(cplx<T>* tile, const cplx<T>* tw) {
    constexpr int NB = (M / R) * L;
    static_assert(NB % NT == 0, "butterflies must divide evenly over threads");
    constexpr int BPT = NB / NT;
    cplx<T> v[BPT][R];
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int id = threadIdx.x + b * NT;
        const int l = id % L, j = id / L;
#pragma unroll
        for (int r = 0; r < R; ++r) v[b][r] = tile[(j + r * (M / R)) * LP + l];
        if constexpr (NS > 1) {
            const int k = j % NS;
#pragma unroll
            for (int r = 1; r < R; ++r) {
                cplx<T> w = tw[k * r * (M / (NS * R))];
                if (SIGN > 0) w.y = -w.y;
                v[b][r] = cmul<T>(v[b][r], w);
            }
        }
        dftR<R, SIGN, T>(v[b]);
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int id = threadIdx.x + b * NT;
        const int l = id % L, j = id / L;
        const int k = j % NS;
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) tile[(base + r * NS) * LP + l] = v[b][r];
    }
    __syncthreads();
}

// Two adjacent lines per thread: one vector shared-memory access moves both
// lines' elements and the twiddles are loaded once for the pair (halves the
// LDS count per point, the MIO pressure the single-line stage runs into).
template <typename T>
struct LinePair {
    cplx<T> a, b;
};
__device__ __forceinline__ LinePair<float> ld_pair(const float2* p) {
    const float4 q = *reinterpret_cast<const float4*>(p);
    return {make_float2(q.x, q.y), make_float2(q.z, q.w)};
}
__device__ __forceinline__ void st_pair(float2* p, const LinePair<float>& v) {
    *reinterpret_cast<float4*>(p) = make_float4(v.a.x, v.a.y, v.b.x, v.b.y);
}
__device__ __forceinline__ LinePair<double> ld_pair(const double2* p) { return {p[0], p[1]}; }
__device__ __forceinline__ void st_pair(double2* p, const LinePair<double>& v) {
    p[0] = v.a;
    p[1] = v.b;
}

template <typename T, int M, int L, int LP, int NT, int SIGN, int R, int NS>
__device__ __forceinline__ void stockham_stage_pairs(cplx<T>* tile, const cplx<T>* tw) {
    constexpr int L2 = L / 2;
    constexpr int NB = (M / R) * L2;
    static_assert(NB % NT == 0, "pair butterflies must divide evenly over threads");
    constexpr int BPT = NB / NT;
    cplx<T> va[BPT][R], vb[BPT][R];
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int id = threadIdx.x + b * NT;
        const int lp = id % L2, j = id / L2;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const LinePair<T> q = ld_pair(&tile[(j + r * (M / R)) * LP + 2 * lp]);
            va[b][r] = q.a;
            vb[b][r] = q.b;
        }
        if constexpr (NS > 1) {
            const int k = j % NS;
#pragma unroll
            for (int r = 1; r < R; ++r) {
                cplx<T> w = tw[k * r * (M / (NS * R))];
                if (SIGN > 0) w.y = -w.y;
                va[b][r] = cmul<T>(va[b][r], w);
                vb[b][r] = cmul<T>(vb[b][r], w);
            }
        }
        dftR<R, SIGN, T>(va[b]);
        dftR<R, SIGN, T>(vb[b]);
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int id = threadIdx.x + b * NT;
        const int lp = id % L2, j = id / L2;
        const int k = j % NS;
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) st_pair(&tile[(base + r * NS) * LP + 2 * lp], LinePair<T>{va[b][r], vb[b][r]});
    }
    __syncthreads();
}

template <typename T, int M, int L, int LP, int NT, int SIGN, int R, int NS>
__device__ __forceinline__ void stage(cplx<T>* tile, const cplx<T>* tw) {
    // pairs when the tile has enough pair-butterflies for every thread and the
    // pitch keeps pairs 16-byte aligned. fp32 only: a pair is one 16-byte access,
    // while an fp64 pair is two 16-byte accesses at a 32-byte thread stride (twice
    // the shared-memory wavefronts of the line-per-thread stage's contiguous ones)
    // Radix-16 stages run line-per-thread (a pair would hold 32 values).
    if constexpr (sizeof(T) == 4 && R <= 8 && LP % 2 == 0 && ((M / R) * (L / 2)) % NT == 0)
        stockham_stage_pairs<T, M, L, LP, NT, SIGN, R, NS>(tile, tw);
    else
        stockham_stage<T, M, L, LP, NT, SIGN, R, NS>(tile, tw);
}

// Tile plan: K = ceil(log2 M / 4) stages of radix <= 16, the larger radices first
// (M = 128: 16 x 8; 1024: 16 x 8 x 8; 2048: 16 x 16 x 8; 512: 8 x 8 x 8): one
// shared-memory round trip per stage, so fewer, wider stages move less data.
template <int M>
struct TilePlan {
    static constexpr int LOG2M = ilog2(M);
    static constexpr int K = (LOG2M + 3) / 4;
    static constexpr int bits(int s) { return LOG2M / K + (s < LOG2M % K ? 1 : 0); }
    static constexpr int R(int s) { return 1 << bits(s); }
    static constexpr int NS(int s) { return s == 0 ? 1 : NS(s - 1) * R(s - 1); }
};

template <typename T, int M, int L, int LP, int NT, int SIGN, int S>
struct StageRunner {
    __device__ __forceinline__ static void run(cplx<T>* tile, const cplx<T>* tw) {
        using TP = TilePlan<M>;
        if constexpr (S < TP::K) {
            stage<T, M, L, LP, NT, SIGN, TP::R(S), TP::NS(S)>(tile, tw);
            StageRunner<T, M, L, LP, NT, SIGN, S + 1>::run(tile, tw);
        }
    }
};

// --------------------------------------------------------------- stage plan
// Forward transforms run radices (8, ..., 8, RL); inverse transforms run the
// reverse (RL, 8, ..., 8). Then the last forward stage's outputs for butterfly
// j (positions j + q M/RL) are exactly the inputs of the first inverse stage's
// butterfly j, and the last inverse stage (radix 8, NS = M/8) outputs the
// positions j + r M/8 -- so kernels can fuse spectral algebra between the two
// transforms in registers and move the first/last stage data straight between
// registers and global memory.
template <int M>
struct Plan {
    static constexpr int LOG2M = ilog2(M);
    static constexpr int N8 = LOG2M / 3;
    static constexpr int RL = 1 << (LOG2M % 3);
    static constexpr int K = N8 + (RL > 1 ? 1 : 0);
    __host__ __device__ static constexpr int fr(int s) { return s < N8 ? 8 : RL; }
    __host__ __device__ static constexpr int fns(int s) { return s == 0 ? 1 : fns(s - 1) * fr(s - 1); }
    __host__ __device__ static constexpr int ir(int s) { return RL > 1 ? (s == 0 ? RL : 8) : 8; }
    __host__ __device__ static constexpr int ins(int s) { return s == 0 ? 1 : ins(s - 1) * ir(s - 1); }
    static constexpr int RLAST_F = fr(K - 1);  // radix of the last forward stage
};

template <int R, int NS, int M, int SIGN, typename T>
__device__ __forceinline__ void pair_twiddle_dft(cplx<T>* va, cplx<T>* vb, int j, const cplx<T>* tw) {
    if constexpr (NS > 1) {
        const int k = j % NS;
#pragma unroll
        for (int r = 1; r < R; ++r) {
            cplx<T> w = tw[k * r * (M / (NS * R))];
            if (SIGN > 0) w.y = -w.y;
            va[r] = cmul<T>(va[r], w);
            vb[r] = cmul<T>(vb[r], w);
        }
    }
    dftR<R, SIGN, T>(va);
    dftR<R, SIGN, T>(vb);
}

template <typename T, int M, int LP, int R>
__device__ __forceinline__ void pair_load(const cplx<T>* tile, int j, int lp, cplx<T>* va, cplx<T>* vb) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const LinePair<T> q = ld_pair(&tile[(j + r * (M / R)) * LP + 2 * lp]);
        va[r] = q.a;
        vb[r] = q.b;
    }
}

template <typename T, int M, int LP, int R, int NS>
__device__ __forceinline__ void pair_store(cplx<T>* tile, int j, int lp, const cplx<T>* va, const cplx<T>* vb) {
    const int k = j % NS;
    const int base = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) st_pair(&tile[(base + r * NS) * LP + 2 * lp], LinePair<T>{va[r], vb[r]});
}

// In-place pair stages s in [S, E) of the forward (INV=false) or inverse plan.
template <typename T, int M, int L, int LP, int NT, bool INV, int S, int E>
struct PlanStages {
    __device__ __forceinline__ static void run(cplx<T>* tile, const cplx<T>* tw) {
        if constexpr (S < E) {
            using Pl = Plan<M>;
            constexpr int R = INV ? Pl::ir(S) : Pl::fr(S);
            constexpr int NS = INV ? Pl::ins(S) : Pl::fns(S);
            stockham_stage_pairs<T, M, L, LP, NT, INV ? +1 : -1, R, NS>(tile, tw);
            PlanStages<T, M, L, LP, NT, INV, S + 1, E>::run(tile, tw);
        }
    }
};

// Full length-M transform of every line of the tile. Caller must
// __syncthreads() after filling the tile; on return the tile holds the
// natural-order spectrum and all threads are synchronised.
template <typename T, int M, int L, int LP, int NT, int SIGN>
__device__ __forceinline__ void tile_fft(cplx<T>* tile, const cplx<T>* tw) {
    StageRunner<T, M, L, LP, NT, SIGN, 0>::run(tile, tw);
}

// Cooperative copy of the M-entry twiddle table into shared memory.
template <typename T, int M, int NT>
__device__ __forceinline__ void load_twiddles(cplx<T>* s_tw, const cplx<T>* g_tw) {
    for (int t = threadIdx.x; t < M; t += NT) s_tw[t] = g_tw[t];
}

}  // namespace gtb
