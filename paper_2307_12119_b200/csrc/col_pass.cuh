// col_pass.cuh — building blocks of the fused column passes (mode A pass 2,
// mode B column pass): per-stage r-major twiddle tables, padded row layouts
// with folded addressing, and the inverse pair stages.
#pragma once

#include "fft_tile.cuh"

namespace gtb {

// Real DCT part of the half spectrum of a mirrored real row: with
// A = (Z[v] + conj Z[M-v]) / 2 (the real part's spectrum of a packed line),
// A = w^{-v/2} At, At real; returns At = Re(hs[v] A), hs[v] = w^{v/2}.
template <typename T>
__device__ __forceinline__ T dct_part(cplx<T> Z, cplx<T> Zc, cplx<T> hs) {
    return T(0.5) * ((Z.x + Zc.x) * hs.x - (Z.y + Zc.y) * hs.y);
}
// Same for the imaginary part's spectrum B = (Z[v] - conj Z[M-v]) / (2i).
template <typename T>
__device__ __forceinline__ T dct_part_im(cplx<T> Z, cplx<T> Zc, cplx<T> hs) {
    return T(0.5) * ((Z.y - Zc.y) * hs.x + (Z.x - Zc.x) * hs.y);
}

// Per-stage twiddle tables, r-major: entry off(s) + (r-1) NS + k holds the
// stage-s twiddle w_M^{k r M/(NS R)} (conjugated for the inverse plan). The
// k = j mod NS of a warp's butterflies are consecutive, so a warp's twiddle
// loads for one r hit consecutive words -- the flat table's k*r stride makes
// them bank conflicts.
template <int M, bool INV>
struct StageTw {
    using Pl = Plan<M>;
    __host__ __device__ static constexpr int R(int s) { return INV ? Pl::ir(s) : Pl::fr(s); }
    __host__ __device__ static constexpr int NS(int s) { return INV ? Pl::ins(s) : Pl::fns(s); }
    __host__ __device__ static constexpr int off(int s) { return s == 0 ? 0 : off(s - 1) + (R(s - 1) - 1) * NS(s - 1); }
    static constexpr int SIZE = off(Pl::K);
};

template <typename T, int M, bool INV, int NT>
__device__ __forceinline__ void build_stage_tw(cplx<T>* dst, const cplx<T>* tw) {
    using ST = StageTw<M, INV>;
    for (int idx = threadIdx.x; idx < ST::SIZE; idx += NT) {
        int s = 0;
#pragma unroll
        for (int t = 1; t < Plan<M>::K; ++t)
            if (idx >= ST::off(t)) s = t;
        const int R = ST::R(s), NS = ST::NS(s);
        const int rel = idx - ST::off(s);
        const int r = 1 + rel / NS, k = rel % NS;
        cplx<T> w = tw[(k * r * (M / (NS * R))) & (M - 1)];
        if (INV) w.y = -w.y;
        dst[idx] = w;
    }
}

// Stage twiddles for butterfly j of stage S: v[r] *= tws[off + (r-1) NS + j mod NS].
template <typename T, int M, bool INV, int S, int NL>
__device__ __forceinline__ void stage_twiddle(cplx<T> (*v)[StageTw<M, INV>::R(S)], int j, const cplx<T>* tws) {
    using ST = StageTw<M, INV>;
    constexpr int R = ST::R(S), NS = ST::NS(S);
    if constexpr (NS > 1) {
        const int k = j % NS;
#pragma unroll
        for (int r = 1; r < R; ++r) {
            const cplx<T> w = tws[ST::off(S) + (r - 1) * NS + k];
#pragma unroll
            for (int l = 0; l < NL; ++l) v[l][r] = cmul<T>(v[l][r], w);
        }
    }
}

// Column-pass tile layouts. Both insert padding every 8 rows so that a warp's
// stride-8 row accesses (the Stockham stores, the fused stage's first inverse
// stores) land in different banks; the padding is a function of row >> 3, so
// for row = base + r S (S a multiple of 8, or S = 1 inside one 8-row block)
// the physical offset is base_offset + r * const and folds into immediates.
//
// Forward phase: the tile's W columns form GA = max(1, W/2) groups; group g
// holds columns v0 + g and v0 + g + GA and three lines: the packed A line
// z = At_v + i At_{v+GA} (both columns' real DCT parts, pass 1) in plane PA,
// and the two B lines as one LinePair in plane PB; one pad row per 8 rows.
// S == 1 requires base and base + r in one 8-row block (the callers' rows j RL + r, RL | 8).
template <int S>
__device__ __forceinline__ int prow(int base, int r) {
    if constexpr (S % 8 == 0 || S == 1) {
        return base + (base >> 3) + r * (S % 8 == 0 ? S + S / 8 : 1);
    } else {
        const int row = base + r * S;
        return row + (row >> 3);
    }
}
// Inverse phase: pairs (Y_w, R_w) of column v0 + w, W pairs per row, half a
// row of padding per 8 rows (the fused stage writes half-rows at stride 8).
template <int W, int M>
struct InvLayout {
    static constexpr int PITCH = 2 * W;
    static constexpr int PADI = W >= 2 ? W : 2;
    static constexpr int SIZE = M * PITCH + (M / 8) * PADI;
    template <int S>
    __device__ __forceinline__ static int off(int base, int r, int w) {
        if constexpr (S % 8 == 0 || S == 1) {
            return base * PITCH + (base >> 3) * PADI + 2 * w + r * (S * PITCH + (S % 8 == 0 ? (S / 8) * PADI : 0));
        } else {
            const int row = base + r * S;
            return row * PITCH + (row >> 3) * PADI + 2 * w;
        }
    }
};

// One Stockham stage (forward plan if !INV, inverse plan if INV) over the
// line pairs of an InvLayout tile (W pairs per row).
template <typename T, int M, int W, int NT, int S, bool INV>
__device__ __forceinline__ void pair_stage(cplx<T>* tile, const cplx<T>* tws) {
    using ST = StageTw<M, INV>;
    constexpr int R = ST::R(S), NS = ST::NS(S);
    constexpr int NB = (M / R) * W;
    static_assert(NB % NT == 0, "pair butterflies must divide evenly over threads");
    constexpr int BPT = NB / NT;
    cplx<T> v[BPT][2][R];
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int id = threadIdx.x + b * NT;
        const int w = id % W, j = id / W;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const LinePair<T> q = ld_pair(&tile[InvLayout<W, M>::template off<M / R>(j, r, w)]);
            v[b][0][r] = q.a;
            v[b][1][r] = q.b;
        }
        stage_twiddle<T, M, INV, S, 2>(v[b], j, tws);
        dftR<R, INV ? +1 : -1, T>(v[b][0]);
        dftR<R, INV ? +1 : -1, T>(v[b][1]);
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int id = threadIdx.x + b * NT;
        const int w = id % W, j = id / W;
        const int k = j % NS;
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r)
            st_pair(&tile[InvLayout<W, M>::template off<NS>(base, r, w)], LinePair<T>{v[b][0][r], v[b][1][r]});
    }
    __syncthreads();
}

template <typename T, int M, int W, int NT, int S, int E, bool INV = true>
struct InvStagesPairs {
    __device__ __forceinline__ static void run(cplx<T>* tile, const cplx<T>* tws) {
        if constexpr (S < E) {
            pair_stage<T, M, W, NT, S, INV>(tile, tws);
            InvStagesPairs<T, M, W, NT, S + 1, E, INV>::run(tile, tws);
        }
    }
};

}  // namespace gtb
