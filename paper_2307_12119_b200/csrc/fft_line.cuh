// fft_line.cuh — one whole FFT line in shared memory, transformed by a CTA: in-place
// Stockham stages (radix 8, then the remainder), one butterfly per thread per stage at
// NT = N / 8. Used where a line is too long for a warp's registers but fits one CTA:
// the large-grid one-pass row kernels (large.cu, n-point lines of the DCT-II / C2R
// factorisations of a 2n mirrored line) and the mode-B row pass at n = 1024 (fixed_point.cu).
#pragma once

#include "fft_tile.cuh"

#ifndef GT_LG_R16
#define GT_LG_R16 8  // radix of the line stages (the last stage takes the remainder)
#endif

namespace gtb {

// One 16-byte pad every 8 elements: the stride-R stores of the first Stockham stage (R x 16 B
// apart) land in different banks.
__device__ __forceinline__ int lpad(int i) { return i + (i >> 3); }

// Stage with radix R over the N-point line buf (padded), NS = product of the previous radices.
// Twiddles w_{NS R}^{k r} = w_m^{k r m / (NS R)} from the m-entry table tw (exp(-2 pi i t / m),
// m a multiple of N): fp64 takes one table load and forms the powers by products; fp32 loads
// every power (a product chain would add up to R-2 roundings).
template <typename T, int R, int NT, int N, int SIGN>
__device__ __forceinline__ void line_stage(cplx<T>* buf, int ns, const cplx<T>* __restrict__ tw, int m) {
    // butterfly j: inputs j + r N/R, outputs (j-k) R + k + r ns
    constexpr int nb = N / R;
    constexpr int BMAX = (nb + NT - 1) / NT;  // butterflies per thread
    const int tid = threadIdx.x;
    cplx<T> v[BMAX][R];
#pragma unroll
    for (int b = 0; b < BMAX; ++b) {
        const int j = tid + b * NT;
        if (j >= nb) break;
        const int k = j % ns;
#pragma unroll
        for (int r = 0; r < R; ++r) v[b][r] = buf[lpad(j + r * nb)];
        if (ns > 1) {
            const int step = (m / (ns * R)) * k;
            if constexpr (sizeof(T) == 8) {
                const cplx<T> w = tw[step & (m - 1)];
                const cplx<T> w1 = mk<T>(w.x, SIGN > 0 ? -w.y : w.y);
                cplx<T> wr = w1;
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    v[b][r] = cmul<T>(v[b][r], wr);
                    if (r + 1 < R) wr = cmul<T>(wr, w1);
                }
            } else {
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    const cplx<T> w = tw[(step * r) & (m - 1)];
                    v[b][r] = cmul<T>(v[b][r], mk<T>(w.x, SIGN > 0 ? -w.y : w.y));
                }
            }
        }
        dftR<R, SIGN, T>(v[b]);
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < BMAX; ++b) {
        const int j = tid + b * NT;
        if (j >= nb) break;
        const int k = j % ns;
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) buf[lpad(base + r * ns)] = v[b][r];
    }
    __syncthreads();
}

template <typename T, int NT, int N, int SIGN, int NS, int REM>
struct LineStages {
    __device__ __forceinline__ static void run(cplx<T>* buf, const cplx<T>* __restrict__ tw, int m) {
        if constexpr (REM > 1) {
            constexpr int R = REM % GT_LG_R16 == 0 ? GT_LG_R16 : REM;
            line_stage<T, R, NT, N, SIGN>(buf, NS, tw, m);
            LineStages<T, NT, N, SIGN, NS * R, REM / R>::run(buf, tw, m);
        }
    }
};

}  // namespace gtb
