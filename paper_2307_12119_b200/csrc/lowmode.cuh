// lowmode.cuh — Anderson(m) mixing on the LMK x LMK lowest cosine modes of a die field: the
// per-field state and the mixing step shared by the batched path (fixed_point.cu fp_lowmode)
// and the large-grid path (large.cu lg_lowmode_*). See fixed_point.cu for the method.
#pragma once
#include <cuda_runtime.h>

namespace gtb {

constexpr int LMK = 16, LMN = LMK * LMK, LMD = 4;
struct LMState {
    int calls;      // mixing steps on this field so far
    int nd;         // residual differences pushed so far
    int have_x;     // xlow valid (cold start: x_0 = 0; warm start: from the second call on)
    int have_prev;  // gprev / fprev valid
    double rprev;   // Picard residual seen at the previous call (growth guard)
    double xlow[LMN], gprev[LMN], fprev[LMN];
    double dG[LMD][LMN], dF[LMD][LMN];
};

__device__ __forceinline__ double lm_warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One mixing step by a CTA of LMN threads: thread tid holds coefficient g of G(x_k); rnow is the
// Picard residual of the previous iteration. Returns this coefficient's correction (x_{k+1} =
// G(x_k) + corr) and updates the state; *applied tells whether any correction was formed.
__device__ __forceinline__ double lowmode_mix(LMState& L, double g, double rnow, int depth, int tid, bool* applied) {
    __shared__ double red[LMD * (LMD + 1) / 2 + LMD][LMN / 32];
    __shared__ double s_gamma[LMD];
    __shared__ int s_k;
    const int calls = L.calls, have_x = L.have_x, have_prev = L.have_prev;
    int nd = L.nd;
    // growth guard: a Picard residual that doubled since the last call drops the history
    const double rprev = L.rprev;
    const bool reset = calls > 1 && rprev > 0.0 && rnow > 2.0 * rprev;
    if (reset) nd = 0;
    __syncthreads();  // every thread has read the header before thread 0 rewrites it
    const double f = g - L.xlow[tid];
    if (have_x && have_prev && !reset) {
        const int slot = nd % depth;
        L.dG[slot][tid] = g - L.gprev[tid];
        L.dF[slot][tid] = f - L.fprev[tid];
        nd += 1;
    }
    L.gprev[tid] = g;
    L.fprev[tid] = f;
    const int k = have_x ? (nd < depth ? nd : depth) : 0;
    double corr = 0.0;
    if (k > 0) {
        double df[LMD], dg[LMD];
#pragma unroll
        for (int i = 0; i < LMD; ++i) {
            df[i] = i < k ? L.dF[i][tid] : 0.0;
            dg[i] = i < k ? L.dG[i][tid] : 0.0;
        }
        // Gram entries (upper triangle) and right-hand side
        int e = 0;
#pragma unroll
        for (int i = 0; i < LMD; ++i) {
#pragma unroll
            for (int j = i; j < LMD; ++j) {
                const double v = lm_warp_sum(df[i] * df[j]);
                if ((tid & 31) == 0) red[e][tid >> 5] = v;
                ++e;
            }
        }
#pragma unroll
        for (int i = 0; i < LMD; ++i) {
            const double v = lm_warp_sum(df[i] * f);
            if ((tid & 31) == 0) red[e][tid >> 5] = v;
            ++e;
        }
        __syncthreads();
        if (tid == 0) {
            double A[LMD][LMD], b[LMD];
            int e2 = 0;
            for (int i = 0; i < LMD; ++i)
                for (int j = i; j < LMD; ++j) {
                    double v = 0.0;
                    for (int w = 0; w < LMN / 32; ++w) v += red[e2][w];
                    A[i][j] = A[j][i] = v;
                    ++e2;
                }
            for (int i = 0; i < LMD; ++i) {
                double v = 0.0;
                for (int w = 0; w < LMN / 32; ++w) v += red[e2][w];
                b[i] = v;
                ++e2;
            }
            double tr = 0.0;
            for (int i = 0; i < k; ++i) tr += A[i][i];
            const double lam = 1e-10 * tr;
            for (int i = 0; i < k; ++i) A[i][i] += lam;
            // Gaussian elimination with partial pivoting on the k x k system
            int ok = tr > 0.0;
            double gm[LMD] = {0.0, 0.0, 0.0, 0.0};
            if (ok) {
                int perm[LMD] = {0, 1, 2, 3};
                for (int c = 0; c < k && ok; ++c) {
                    int piv = c;
                    for (int r = c + 1; r < k; ++r)
                        if (fabs(A[perm[r]][c]) > fabs(A[perm[piv]][c])) piv = r;
                    const int tmp = perm[c];
                    perm[c] = perm[piv];
                    perm[piv] = tmp;
                    const double d = A[perm[c]][c];
                    if (!(fabs(d) > 1e-300)) {
                        ok = 0;
                        break;
                    }
                    for (int r = c + 1; r < k; ++r) {
                        const double m_ = A[perm[r]][c] / d;
                        for (int cc = c; cc < k; ++cc) A[perm[r]][cc] -= m_ * A[perm[c]][cc];
                        b[perm[r]] -= m_ * b[perm[c]];
                    }
                }
                if (ok)
                    for (int c = k - 1; c >= 0; --c) {
                        double v = b[perm[c]];
                        for (int cc = c + 1; cc < k; ++cc) v -= A[perm[c]][cc] * gm[cc];
                        gm[c] = v / A[perm[c]][c];
                    }
                for (int i = 0; i < k; ++i)
                    if (!isfinite(gm[i]) || fabs(gm[i]) > 1e3) ok = 0;
            }
            for (int i = 0; i < LMD; ++i) s_gamma[i] = ok ? gm[i] : 0.0;
            s_k = ok;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < LMD; ++i) corr -= s_gamma[i] * dg[i];
        if (!s_k) nd = 0;  // unusable history: start over from plain iterations
    }
    if (!isfinite(corr)) corr = 0.0;
    L.xlow[tid] = g + corr;
    if (tid == 0) {
        L.calls = calls + 1;
        L.nd = nd;
        L.have_prev = have_x;
        L.have_x = 1;
        L.rprev = rnow;
    }
    *applied = k > 0;
    return corr;
}

}  // namespace gtb
