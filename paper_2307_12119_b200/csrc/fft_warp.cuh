// fft_warp.cuh — one-warp FFT of a single length-M line, M = 32 P (P = 4, 8, 16).
//
// Used by the row passes, whose global data is contiguous along the line: a
// warp loads / stores a row coalesced straight from / to registers, and the
// only data exchange inside the transform is one warp-private shared-memory
// transpose plus a cross-lane step by shuffles -- no CTA barriers, no
// transposing staging tile (the tile engine needs both for rows).
//
// Four-step factorisation M = 32 x P, input index i = j + 32 k (lane j holds
// k = 0..P-1), output index f = k' + P m1 + P^2 h:
//   1. P-point DFT in registers over k, twiddle w_M^{j k'};
//   2. transpose through shared memory: lane (k', h) takes the decimated
//      sequence j = h + Q t (Q = 32 / P lanes per 32-point sub-transform);
//   3. P-point DFT over t, twiddle w_32^{h m1}, Q-point DFT across the Q lanes
//      sharing k' (shuffles).
// On return lane (k' + P h) holds X[k' + P m1 + P^2 h] in v[m1].
#pragma once

#include "fft_tile.cuh"

namespace gtb {

// 32-point DFT in registers: radix 8 over n1 (inputs n2 + 4 n1), twiddle
// w32^{n2 k1}, radix 4 over n2; X[k1 + 8 k2] lands in slot 4 k1 + k2 and a
// compile-time register permutation restores natural order.
template <int SIGN, typename T>
__device__ __forceinline__ void dft32(cplx<T>* v) {
    constexpr double C32[8] = {1.0, 0.98078528040323044913, 0.92387953251128675613, 0.83146961230254523708,
                               0.70710678118654752440, 0.55557023301960222474, 0.38268343236508977173,
                               0.19509032201612826785};  // cos(2 pi t / 32), t = 0..7
    cplx<T> a[4][8];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
#pragma unroll
        for (int n1 = 0; n1 < 8; ++n1) a[n2][n1] = v[n2 + 4 * n1];
        dft8<SIGN, T>(a[n2]);
    }
#pragma unroll
    for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
        for (int k1 = 1; k1 < 8; ++k1) {
            const int e = n2 * k1;  // w32^e, e < 32: cos / sin from the first octant table
            const int q = e & 7, oct = e >> 3;
            // cos / sin(2 pi e / 32) with e = 8 oct + q
            const double c0 = C32[q], s0 = C32[(8 - q) & 7] * (q == 0 ? 0.0 : 1.0);
            double c = c0, sn = s0;
            if (oct == 1) {
                c = -s0;
                sn = c0;
            } else if (oct == 2) {
                c = -c0;
                sn = -s0;
            } else if (oct == 3) {
                c = s0;
                sn = -c0;
            }
            a[n2][k1] = cmul<T>(a[n2][k1], mk<T>(T(c), T(SIGN < 0 ? -sn : sn)));
        }
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) {
        cplx<T> q[4] = {a[0][k1], a[1][k1], a[2][k1], a[3][k1]};
        dft4<SIGN, T>(q);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) v[k1 + 8 * k2] = q[k2];
    }
}

template <int P, int SIGN, typename T>
__device__ __forceinline__ void dftP(cplx<T>* v) {
    if constexpr (P == 32)
        dft32<SIGN, T>(v);
    else if constexpr (P == 16)
        dft16<SIGN, T>(v);
    else if constexpr (P == 8)
        dft8<SIGN, T>(v);
    else if constexpr (P == 4)
        dft4<SIGN, T>(v);
}

template <typename T>
__device__ __forceinline__ cplx<T> shfl_c(cplx<T> a, int src) {
    cplx<T> r;
    r.x = __shfl_sync(0xffffffffu, a.x, src);
    r.y = __shfl_sync(0xffffffffu, a.y, src);
    return r;
}

template <typename T, int M>
struct WarpFFT {
    static constexpr int P = M / 32;
    static constexpr int Q = 32 / P;
    static constexpr int SP = 33;  // scratch pitch (complex) of the P x 32 transpose
    static constexpr int SCRATCH = P * SP > M ? P * SP : M;  // complex elements per warp
    static_assert(P == 4 || P == 8 || P == 16 || P == 32, "warp FFT supports M = 128, 256, 512, 1024");

    // Step-1 twiddles lane-major: tw1[(k - 1) 32 + j] = w_M^{j k}, so a warp's
    // loads for one k are 32 consecutive entries (the flat table's j k stride is
    // a k-way bank conflict).
    static constexpr int TW1 = (P - 1) * 32;
    __device__ __forceinline__ static void build_tw1(cplx<T>* tw1, const cplx<T>* tw, int tid, int nthr) {
        for (int i = tid; i < TW1; i += nthr) tw1[i] = tw[(i & 31) * (1 + (i >> 5))];
    }

    // tw: M-entry table exp(-2 pi i t / M), tw1 (above), both shared; scratch: SCRATCH complex per warp.
    template <int SIGN>
    __device__ __forceinline__ static void run(cplx<T>* v, cplx<T>* scratch, const cplx<T>* tw,
                                               const cplx<T>* tw1, int lane) {
        dftP<P, SIGN, T>(v);
#pragma unroll
        for (int k = 1; k < P; ++k) {
            cplx<T> w = tw1[(k - 1) * 32 + lane];  // w_M^{j k'}
            if (SIGN > 0) w.y = -w.y;
            v[k] = cmul<T>(v[k], w);
        }
#pragma unroll
        for (int k = 0; k < P; ++k) scratch[k * SP + lane] = v[k];
        __syncwarp();
        const int kq = lane % P, h = lane / P;
#pragma unroll
        for (int t = 0; t < P; ++t) v[t] = scratch[kq * SP + h + Q * t];
        __syncwarp();
        dftP<P, SIGN, T>(v);
        if constexpr (Q == 2) {
            // w_32^{h m1} with h in {0, 1}: compile-time constants selected per lane (the
            // shared-memory twiddle loads were ~13% of the row passes' shared wavefronts)
#pragma unroll
            for (int m1 = 1; m1 < P; ++m1) {
                constexpr double C8[9] = {1.0, 0.98078528040323044913, 0.92387953251128675613,
                                          0.83146961230254523708, 0.70710678118654752440, 0.55557023301960222474,
                                          0.38268343236508977173, 0.19509032201612826785, 0.0};
                // cos / sin(2 pi m1 / 32), m1 < 16: second quadrant for m1 > 8
                const double cw = m1 <= 8 ? C8[m1] : -C8[16 - m1];
                const double sw = m1 <= 8 ? C8[8 - m1] : C8[m1 - 8];
                const T wc = h ? T(cw) : T(1), ws = h ? T(SIGN < 0 ? -sw : sw) : T(0);
                v[m1] = cmul<T>(v[m1], mk<T>(wc, ws));
            }
        } else if constexpr (Q > 2) {
#pragma unroll
            for (int m1 = 1; m1 < P; ++m1) {
                cplx<T> w = tw[h * m1 * P];  // w_32^{h m1} = w_M^{h m1 P}
                if (SIGN > 0) w.y = -w.y;
                v[m1] = cmul<T>(v[m1], w);
            }
        }  // Q == 1 (M = 1024): h = 0, all factors are 1
        // Q-point DFT across the lanes kq + P h' (lane h keeps output g = h)
        if constexpr (Q == 2) {
            // radix-2 butterfly with the partner lane: g = 0 -> v0 + v1, g = 1 -> v0 - v1
            const T sg = h ? T(-1) : T(1);
#pragma unroll
            for (int m1 = 0; m1 < P; ++m1) {
                const cplx<T> z = shfl_c<T>(v[m1], lane ^ P);
                v[m1] = mk<T>(fma(sg, v[m1].x, z.x), fma(sg, v[m1].y, z.y));
            }
        } else if constexpr (Q > 1) {
            // direct form
#pragma unroll
            for (int m1 = 0; m1 < P; ++m1) {
                // own term h' = h carries w_Q^{h h}
                cplx<T> w0 = tw[((h * h) % Q) * (M / Q)];
                if (SIGN > 0) w0.y = -w0.y;
                cplx<T> acc = cmul<T>(v[m1], w0);
#pragma unroll
                for (int d = 1; d < Q; ++d) {
                    const int hs = (h + d) % Q;  // source h'
                    const cplx<T> z = shfl_c<T>(v[m1], kq + P * hs);
                    // w_Q^{h' g}, g = h: exponent (hs * h) mod Q, table index * (M / Q)
                    cplx<T> w = tw[((hs * h) % Q) * (M / Q)];
                    if (SIGN > 0) w.y = -w.y;
                    acc = cadd<T>(acc, cmul<T>(z, w));
                }
                v[m1] = acc;
            }
        }
    }

    // position of v[m1] held by `lane` on return
    __device__ __forceinline__ static int out_pos(int lane, int m1) {
        return (lane % P) + P * m1 + P * P * (lane / P);
    }
};

}  // namespace gtb
