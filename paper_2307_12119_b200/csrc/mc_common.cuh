// mc_common.cuh — definitions shared by the mode-A translation units:
// mc_rows.cu (passes 1 and 3: the row transforms, packed-FP32 arithmetic) and
// mc_modeA.cu (pass 2, the fused column pass, scalar FP32, and the host side).
// See mc_modeA.cu for the algorithm.
#pragma once
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
    static constexpr float min_pos() { return 1.175494351e-38f; }
};
template <>
struct Real<double> {
    static constexpr double max() { return 1.7976931348623157e308; }
    static constexpr double min_pos() { return 1e-300; }
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
    double nom64;     // nom_scale as the caller gave it (the fp64 re-solve must not inherit its fp32 rounding)
    const int* dcnt;  // optional device sample count (fp64 re-solve of selected pairs): min(*dcnt, count)
    __device__ __forceinline__ int eff_count(int count) const { return dcnt ? min(*dcnt, count) : count; }
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
#ifndef GT_P2_MINB64
#define GT_P2_MINB64 1  // fp64 column pass: resident CTAs the register budget targets (tuning)
#endif
#ifdef GT_P2_MINB
    static constexpr int MINB2 = sizeof(T) == 8 ? 1 : GT_P2_MINB;  // tuning override (occupancy sweeps)
#else
    static constexpr int MINB2 = sizeof(T) == 8 ? (M <= 512 ? GT_P2_MINB64 : 1) : ((512 / NT2) < 1 ? 1 : (512 / NT2));
#endif
};

// --------------------------------------------------- warp-per-row passes
// Row passes for M = 128 / 256 / 512: each warp owns one die row at a time,
// loads and stores it coalesced straight from / to registers and transforms it
// with the one-warp FFT (fft_warp.cuh): no CTA barriers, no transposing tile.
#ifndef GT_W1
#define GT_W1 12  // 12 warps x 2 CTAs at 80 registers: no spills (16 warps at 64 registers spilled 40 B;
                  // pass 1 1.51 -> 1.46 ms per 4096 pairs, profiles/r2s4_notes.md)
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

template <typename T, int M>
constexpr bool use_warp_rows() {
    return M == 128 || M == 256 || M == 512;
}

// Arguments of the row passes (pass 1: P, N, V -> Ar, B, S; pass 3: Y (A), R (B) -> out).
template <typename T>
struct MCRowArgs {
    MCIn<T> in;
    int s0, cnt;
    T* Ar;
    cplx<T>* A;
    cplx<T>* B;
    T* S;
    gtd_sample_stats* stats;
    const cplx<T>* tw;
    const cplx<T>* hs;
    T var_lo, var_hi;
    T* out;
    T rand_scale;
    int with_rand;
};
// Implemented in mc_rows.cu for every (T, M) the dispatcher uses.
// setup: kernel attributes; returns resident CTAs per SM of the pass's kernel.
template <typename T, int M>
int mc_rows_setup(int pass);
// launch on `st` with a grid of at most sms * ctas_per_sm persistent CTAs.
template <typename T, int M>
void mc_rows_launch(int pass, bool tma, int sms, int ctas_per_sm, cudaStream_t st, const MCRowArgs<T>& a);

}  // namespace gtb
