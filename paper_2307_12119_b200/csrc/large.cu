// large.cu — config 4: the mode-B leakage fixed point on a single large grid
// (n up to 8192, m = 16384), fp64, as seven four-step FFT passes per iteration,
// each usable on a slab of rows or columns so that a multi-GPU driver can put an
// all-to-all transpose between the row and the column phases.
//
// Same math as fixed_point.cu (oracle: oracle/restate.cpp ref_fixed_point_batch):
//   theta - T0 = crop(IFFT(fk . FFT(mirror(P + L0 f(T)))))
// A length-m line transform is split four-step, m = M1 M2, i = i1 + M1 i2,
// k = k2 + M2 k1:
//   forward : FFT_M2 over i2 (per i1) x W_m^{i1 k2}, then FFT_M1 over i1 (per k2)
//   inverse : IFFT_M1 over k1 (per k2) x W_m^{-i_a k2}, then IFFT_M2 over k2 (per
//             i_a), output i = i_a + M1 i_b
// and every sub-transform runs in the shared-memory tile engine (fft_tile.cuh)
// on L lines at a time, with the passes' loads and stores coalesced across the
// L lines. Passes per iteration (p = die-row pair, v = half-spectrum column):
//   rows   : FwdA (applied rows, mirrored, two rows per line) -> S1 -> FwdB -> Z
//   columns: ColA (split Z into the rows' half spectra, mirror) -> C1 -> ColB
//            (forward, x fk, inverse) -> C2 -> ColC (rows [0, n)) -> Y
//   rows   : RinvA (Hermitian merge of two rows) -> S1 -> RinvB (theta -> T,
//            residual, next applied rows)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#ifndef GT_LG_RINV_NT
#define GT_LG_RINV_NT 1024
#endif

#include "launch_once.cuh"
#include "fft_line.cuh"
#include "fft_tile.cuh"
#include "gt_device.h"
#include "kirchhoff.cuh"
#include "lowmode.cuh"

namespace gtb {
namespace {

template <typename T>
__device__ __forceinline__ cplx<T> twm(const double2* __restrict__ tw, int M, long long e, bool inv) {
    const double2 w = tw[e & (M - 1)];
    return mk<T>(T(w.x), T(inv ? -w.y : w.y));
}

__device__ __forceinline__ void pf_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// ------------------------------------------------------------------ pass ops
// Every op: load(g, line, j) -> the element; pf(g, line, j) issues an L2 prefetch of the
// same address(es) (lg_pass pulls the NEXT item's lines into L2 while it transforms this one).
template <typename T>
struct FwdA {
    static constexpr bool REDUCE = false;  // group p (row pair), line i1, j = i2
    static constexpr int SIGN = -1;
    static constexpr bool LINE_FAST = true;
    const T* app;  // [rows][n] applied power, rows of this slab
    cplx<T>* S1;   // [pairs][m]
    const double2* tw;
    int n, M, M1;
    int embed = 0;  // 0: mirror_pad (spectral.cpp:105-114); 1: center_kernel of (app - shift) (spectral.cpp:126-141)
    T shift = T(0);
    __device__ cplx<T> load(int p, int i1, int j) const {
        const int i = i1 + M1 * j;
        int y;
        if (embed) {
            y = (i + n / 2) & (M - 1);
            if (y >= n) return mk<T>(T(0), T(0));
        } else {
            y = i < n ? i : M - 1 - i;
        }
        return mk<T>(app[static_cast<size_t>(2 * p) * n + y] - shift, app[static_cast<size_t>(2 * p + 1) * n + y] - shift);
    }
    __device__ void pf(int p, int i1, int j) const {
        const int i = i1 + M1 * j;
        int y;
        if (embed) {
            y = (i + n / 2) & (M - 1);
            if (y >= n) return;
        } else {
            y = i < n ? i : M - 1 - i;
        }
        pf_l2(app + static_cast<size_t>(2 * p) * n + y);
        pf_l2(app + static_cast<size_t>(2 * p + 1) * n + y);
    }
    using Pre = cplx<T>;  // the four-step twiddle, issued ahead of the stores
    __device__ Pre pre(int, int i1, int k2) const { return twm<T>(tw, M, static_cast<long long>(i1) * k2, false); }
    __device__ void store(int p, int i1, int k2, cplx<T> v, const Pre& w) const {
        S1[static_cast<size_t>(p) * M + i1 + static_cast<size_t>(M1) * k2] = cmul<T>(v, w);
    }
};

template <typename T>
struct FwdB {
    static constexpr bool REDUCE = false;  // group p, line k2, j = i1
    static constexpr int SIGN = -1;
    static constexpr bool LINE_FAST = false;
    const cplx<T>* S1;
    cplx<T>* Z;  // [pairs][m] natural order spectra of (row 2p) + i (row 2p+1), mirrored
    int M, M1, M2;
    __device__ cplx<T> load(int p, int k2, int j) const {
        return S1[static_cast<size_t>(p) * M + j + static_cast<size_t>(M1) * k2];
    }
    __device__ void pf(int p, int k2, int j) const { pf_l2(S1 + static_cast<size_t>(p) * M + j + static_cast<size_t>(M1) * k2); }
    struct Pre {};
    __device__ Pre pre(int, int, int) const { return {}; }
    __device__ void store(int p, int k2, int k1, cplx<T> v, const Pre&) const {
        Z[static_cast<size_t>(p) * M + k2 + static_cast<size_t>(M2) * k1] = v;
    }
};

template <typename T>
struct ColA {
    static constexpr bool REDUCE = false;  // group i1, line = local column c (v = c0 + c), j = i2
    static constexpr int SIGN = -1;
    static constexpr bool LINE_FAST = true;
    // Spectra of ALL row pairs: Z[p zs + oa + c] = Z_p[v], Z[p zs + ((ob + sb c) & mask)] = Z_p[m - v].
    // Full layout (one GPU): zs = m, oa = c0, ob = m - c0, sb = -1, mask = m - 1.
    // Compact layout (after the all-to-all): zs = 2 hc, oa = 0, ob = hc, sb = +1, mask = ~0.
    // Peer layout (multi-GPU without an all-to-all, gtd_lg_cols_peer): row pair p lives in
    // rank p / Pr's full [Pr][m] spectra, read in place through its mapped pointer Zr[p / Pr]
    // (NVLink peer loads, one rank's row block per pointer); Z is unused then.
    const cplx<T>* Z;
    cplx<T>* C1;  // [m][hc] (row i1 + M1 k2)
    const double2* tw;
    int n, M, M1, c0, hc;
    long long zs;
    int oa, ob, sb, mask;
    int embed = 0;  // rows: 0 mirror_pad, 1 center_kernel
    const cplx<T>* const* Zr = nullptr;
    int Pr = 0;
    // Real-DCT row layout (rows written by lg_rfwd_dct, n <= 8192): At[x][aoff + c] = C_x[v],
    // the row's spectrum U_x[v] = conj(hs[v]) C_x[v] -- one 8-byte load per element. With a
    // peer table (Zr set) rank r holds rows [2 Pr r, 2 Pr (r+1)) of At.
    const T* At = nullptr;
    int hA = 0, aoff = 0;
    const double2* hs = nullptr;
    // pack = 1 (DCT rows): line c carries the two real columns 2c, 2c+1 of the block (< hcols)
    // as C[., 2c] + i C[., 2c+1]; their column transforms separate locally in ColB
    int pack = 0, hcols = 0;
    __device__ T atv(int x, int c) const {
        if (Zr) {
            const int rpr = 2 * Pr, r = x / rpr;
            return reinterpret_cast<const T*>(Zr[r])[static_cast<size_t>(x - r * rpr) * hA + aoff + c];
        }
        return At[static_cast<size_t>(x) * hA + aoff + c];
    }
    __device__ const cplx<T>* zrow(int p) const {
        if (Zr) {
            const int r = p / Pr;
            return Zr[r] + static_cast<size_t>(p - r * Pr) * zs;
        }
        return Z + static_cast<size_t>(p) * zs;
    }
    __device__ cplx<T> load(int i1, int c, int j) const {
        const int i = i1 + M1 * j;
        int x;
        if (embed) {
            x = (i + n / 2) & (M - 1);
            if (x >= n) return mk<T>(T(0), T(0));
        } else {
            x = i < n ? i : M - 1 - i;
        }
        if (pack) {
            const T a0 = atv(x, 2 * c);
            const T a1 = 2 * c + 1 < hcols ? atv(x, 2 * c + 1) : T(0);
            return mk<T>(a0, a1);
        }
        if (hs) {
            const T a = atv(x, c);
            const double2 h = hs[c0 + c];
            return mk<T>(T(h.x) * a, -T(h.y) * a);
        }
        const cplx<T>* Zp = zrow(x >> 1);
        const cplx<T> a = Zp[oa + c], b = cconj<T>(Zp[(ob + sb * c) & mask]);
        // half spectra of the two real rows packed in Zp (x even: real part's, odd: imaginary part's)
        return (x & 1) ? mk<T>(T(0.5) * (a.y - b.y), T(-0.5) * (a.x - b.x))
                       : mk<T>(T(0.5) * (a.x + b.x), T(0.5) * (a.y + b.y));
    }
    __device__ void pf(int i1, int c, int j) const {
        const int i = i1 + M1 * j;
        int x;
        if (embed) {
            x = (i + n / 2) & (M - 1);
            if (x >= n) return;
        } else {
            x = i < n ? i : M - 1 - i;
        }
        if (hs) {
            if (!Zr) pf_l2(At + static_cast<size_t>(x) * hA + aoff + (pack ? 2 * c : c));
            return;
        }
        const cplx<T>* Zp = zrow(x >> 1);
        pf_l2(Zp + oa + c);
        pf_l2(Zp + ((ob + sb * c) & mask));
    }
    using Pre = cplx<T>;
    __device__ Pre pre(int i1, int, int k2) const { return twm<T>(tw, M, static_cast<long long>(i1) * k2, false); }
    __device__ void store(int i1, int c, int k2, cplx<T> v, const Pre& w) const {
        C1[(static_cast<size_t>(i1) + static_cast<size_t>(M1) * k2) * hc + c] = cmul<T>(v, w);
    }
};

template <typename T>
struct ColB {
    static constexpr bool REDUCE = false;  // group k2, line c, j = i1; forward -> x fk -> inverse over k1
    static constexpr int SIGN = -1;
    static constexpr bool LINE_FAST = true;
    const cplx<T>* C1;
    cplx<T>* C2;  // [m][hc] (row k2 + M2 i_a)
    const cplx<T>* fk;
    int fkp;
    const double2* tw;
    int h, M, M1, M2, c0, hc;
    // pack = 1: C1 holds packed lines [m][hcp] (ColA pack); a 32-line item is the 16 packed
    // lines of its 32 columns in slots 0..15 (slots 16..31 start empty), unpacked after the
    // forward transform into column 2 cp (slot s) and 2 cp + 1 (slot s + 16):
    //   D_a + i D_b = hs[u] Z[u] (both real: DCT-II of the mirrored columns), and the column
    //   spectrum of U_x[v] = conj(hs[v]) C_x[v] is conj(hs[u] hs[v]) D[u].
    int pack = 0, hcp = 0;
    const double2* hs = nullptr;
    __device__ int slot_col(int c) const { return 32 * (c >> 5) + 2 * (c & 15) + ((c >> 4) & 1); }
    __device__ cplx<T> load(int k2, int c, int j) const {
        if (pack) {
            const int s = c & 31, cp = 16 * (c >> 5) + s;
            if (s >= 16 || cp >= hcp) return mk<T>(T(0), T(0));
            return C1[(static_cast<size_t>(j) + static_cast<size_t>(M1) * k2) * hcp + cp];
        }
        return C1[(static_cast<size_t>(j) + static_cast<size_t>(M1) * k2) * hc + c];
    }
    __device__ void pf(int k2, int c, int j) const {
        if (pack) {
            const int s = c & 31, cp = 16 * (c >> 5) + s;
            if (s < 16 && cp < hcp) pf_l2(C1 + (static_cast<size_t>(j) + static_cast<size_t>(M1) * k2) * hcp + cp);
            return;
        }
        pf_l2(C1 + (static_cast<size_t>(j) + static_cast<size_t>(M1) * k2) * hc + c);
    }
    // unpack slot s < 16 of frequency row k1 in place (slots s, s + 16), times the spectral factor
    __device__ void unpack(cplx<T>* tile, int LP, int k2, int l0, int s, int k1) const {
        const int u = k2 + M2 * k1;
        const int cp = (l0 >> 1) + s;
        const cplx<T> z = tile[k1 * LP + s];
        const double2 hu = hs[u];
        const cplx<T> d = cmul<T>(mk<T>(T(hu.x), T(hu.y)), z);  // D_a + i D_b
        cplx<T> y0 = mk<T>(T(0), T(0)), y1 = mk<T>(T(0), T(0));
        const int va = 2 * cp, vb = va + 1;  // local columns
        if (va < hc && c0 + va < h) {
            const double2 hv = hs[c0 + va];
            const cplx<T> ph = cconj<T>(cmul<T>(mk<T>(T(hu.x), T(hu.y)), mk<T>(T(hv.x), T(hv.y))));
            y0 = cscale<T>(cmul<T>(fk[static_cast<size_t>(u) * fkp + c0 + va], ph), d.x);
        }
        if (vb < hc && c0 + vb < h) {
            const double2 hv = hs[c0 + vb];
            const cplx<T> ph = cconj<T>(cmul<T>(mk<T>(T(hu.x), T(hu.y)), mk<T>(T(hv.x), T(hv.y))));
            y1 = cscale<T>(cmul<T>(fk[static_cast<size_t>(u) * fkp + c0 + vb], ph), d.y);
        }
        tile[k1 * LP + s] = y0;
        tile[k1 * LP + s + 16] = y1;
    }
    // the spectral factor at (u, v); zero for the padded columns v > n
    __device__ cplx<T> midw(int k2, int c, int k1) const {
        const int u = k2 + M2 * k1, vv = c0 + c;
        return vv < h ? fk[static_cast<size_t>(u) * fkp + vv] : mk<T>(T(0), T(0));
    }
    using Pre = cplx<T>;
    __device__ Pre pre(int k2, int, int ia) const { return twm<T>(tw, M, static_cast<long long>(ia) * k2, true); }
    __device__ void store(int k2, int c, int ia, cplx<T> v, const Pre& w) const {
        if (pack) {
            c = slot_col(c);
            if (c >= hc) return;
        }
        C2[(static_cast<size_t>(k2) + static_cast<size_t>(M2) * ia) * hc + c] = cmul<T>(v, w);
    }
};

template <typename T>
struct KColB {  // group k2, line c, j = i1: forward only; fk[u][v] natural order (+ DC term)
    static constexpr bool REDUCE = false;
    static constexpr int SIGN = -1;
    static constexpr bool LINE_FAST = true;
    const cplx<T>* C1;
    cplx<T>* fk;
    int fkp, M, M1, M2, hc;
    T dc;
    __device__ cplx<T> load(int k2, int c, int j) const {
        return C1[(static_cast<size_t>(j) + static_cast<size_t>(M1) * k2) * hc + c];
    }
    __device__ void pf(int, int, int) const {}
    struct Pre {};
    __device__ Pre pre(int, int, int) const { return {}; }
    __device__ void store(int k2, int c, int k1, cplx<T> v, const Pre&) const {
        const int u = k2 + M2 * k1;
        if (u == 0 && c == 0) v.x += dc;  // baseline_kernel_spectrum: fk[0] += phi m^2 / 4 (greens.cpp:194-201)
        fk[static_cast<size_t>(u) * fkp + c] = v;
    }
};

template <typename T>
struct ColC {
    static constexpr bool REDUCE = false;  // group i_a, line c, j = k2; output rows i = i_a + M1 i_b < n
    static constexpr int SIGN = +1;
    static constexpr bool LINE_FAST = true;
    const cplx<T>* C2;
    cplx<T>* Y;  // [n][hc]
    int n, M, M1, M2, hc;
    // Peer layout: die row i goes straight into its owner's row buffer Yr[i / rpr]
    // [rpr][hy] at column c0 + c (NVLink peer stores), in place of the second all-to-all.
    cplx<T>* const* Yr = nullptr;
    int rpr = 0, hy = 0, c0 = 0;
    __device__ cplx<T> load(int ia, int c, int j) const {
        return C2[(static_cast<size_t>(j) + static_cast<size_t>(M2) * ia) * hc + c];
    }
    __device__ void pf(int ia, int c, int j) const {
        pf_l2(C2 + (static_cast<size_t>(j) + static_cast<size_t>(M2) * ia) * hc + c);
    }
    struct Pre {};
    __device__ Pre pre(int, int, int) const { return {}; }
    __device__ void store(int ia, int c, int ib, cplx<T> v, const Pre&) const {
        const int i = ia + M1 * ib;
        if (i >= n) return;
        if (Yr) {
            const int r = i / rpr;
            Yr[r][static_cast<size_t>(i - r * rpr) * hy + c0 + c] = v;
        } else {
            Y[static_cast<size_t>(i) * hc + c] = v;
        }
    }
};

template <typename T>
struct RinvA {
    static constexpr bool REDUCE = false;  // group p, line k2, j = k1: Hermitian merge of rows 2p, 2p+1
    static constexpr int SIGN = +1;
    static constexpr bool LINE_FAST = true;
    const cplx<T>* Y;  // [rows][hy] all columns of this slab's rows (after the transpose back)
    cplx<T>* S1;
    const double2* tw;
    int n, M, M2, hy;
    __device__ cplx<T> load(int p, int k2, int j) const {
        const int f = k2 + M2 * j, w = f <= n ? f : M - f;
        const cplx<T> y = Y[static_cast<size_t>(2 * p) * hy + w], r = Y[static_cast<size_t>(2 * p + 1) * hy + w];
        if (f == 0 || f == n) return mk<T>(y.x, r.x);
        return f < n ? mk<T>(y.x - r.y, y.y + r.x) : mk<T>(y.x + r.y, r.x - y.y);
    }
    __device__ void pf(int p, int k2, int j) const {
        const int f = k2 + M2 * j, w = f <= n ? f : M - f;
        pf_l2(Y + static_cast<size_t>(2 * p) * hy + w);
        pf_l2(Y + static_cast<size_t>(2 * p + 1) * hy + w);
    }
    using Pre = cplx<T>;
    __device__ Pre pre(int, int k2, int ia) const { return twm<T>(tw, M, static_cast<long long>(ia) * k2, true); }
    __device__ void store(int p, int k2, int ia, cplx<T> v, const Pre& w) const {
        S1[static_cast<size_t>(p) * M + k2 + static_cast<size_t>(M2) * ia] = cmul<T>(v, w);
    }
};

template <typename T>
struct RinvB {  // group p, line i_a, j = k2: theta -> T, residual, next applied
    static constexpr bool REDUCE = true;
    static constexpr int SIGN = +1;
    static constexpr bool LINE_FAST = false;
    const cplx<T>* S1;
    T* Tst;        // [rows][n] rise state
    T* app;        // [rows][n] next applied
    const T* P;    // [rows][n]
    const T* L0;   // [rows][n]
    // Chebyshev semi-iteration (slab.py, accel > 0): Q holds x_{k-1} on entry and x_k on exit,
    // G receives G(x_k) (the result once the stop rule holds); om > 0 stores
    // x_{k+1} = om (gm G(x_k) + (1 - gm) x_k - x_{k-1}) + x_{k-1} as the state
    T* Q = nullptr;
    T* G = nullptr;
    T om = T(0), gm = T(1);
    unsigned long long* res_bits;
    int* status;
    int n, M, M1, M2, law, kirchhoff;
    T beta, ka, kb, kexp, t_ambient, inv;
    __device__ cplx<T> load(int p, int ia, int j) const {
        return S1[static_cast<size_t>(p) * M + j + static_cast<size_t>(M2) * ia];
    }
    __device__ void pf(int p, int ia, int j) const { pf_l2(S1 + static_cast<size_t>(p) * M + j + static_cast<size_t>(M2) * ia); }
    struct Pre {
        T told[2], p[2], l0[2], q[2];
    };
    // the epilogue's global inputs, issued ahead of the stores (lg_pass batches 4 elements)
    __device__ Pre pre(int p, int ia, int ib) const {
        Pre r{};
        const int i = ia + M1 * ib;
        if (i >= n) return r;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const size_t o = static_cast<size_t>(2 * p + half) * n + i;
            r.told[half] = Tst[o];
            r.p[half] = P[o];
            r.l0[half] = L0[o];
            r.q[half] = om > T(0) ? Q[o] : T(0);
        }
        return r;
    }
    __device__ void store(int p, int ia, int ib, cplx<T> v, const Pre& q, double& dmax, int& bad) const {
        const int i = ia + M1 * ib;
        if (i >= n) return;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const size_t o = static_cast<size_t>(2 * p + half) * n + i;
            T t = (half ? v.y : v.x) * inv;
            if (kirchhoff) t = kirchhoff_rise(t, kb / ka, kexp, t_ambient, bad);
            if (!isfinite(t)) bad |= GTD_ST_NONFINITE;
            dmax = fmax(dmax, double(fabs(t - q.told[half])));
            if (G) G[o] = t;
            if (Q) Q[o] = q.told[half];
            if (om > T(0)) t = om * (gm * t + (T(1) - gm) * q.told[half] - q.q[half]) + q.q[half];
            Tst[o] = t;
            const T f = law ? T(exp(beta * t)) : T(1) + beta * t;
            app[o] = q.p[half] + q.l0[half] * f;
        }
    }
};

// ------------------------------------------------------------------ generic pass
template <typename T, int N>
constexpr int lg_pitch() {
    return sizeof(T) == 8 ? TileGeom<T, N>::L + 1 : TileGeom<T, N>::L + 2;
}

// L lines of N points per work item; items = groups x ceil(nlines / L).
template <typename T, int N, class Op, bool TWO>
__global__ void __launch_bounds__(TileGeom<T, N>::NT, TileGeom<T, N>::MINB)
lg_pass(Op op, const double2* __restrict__ twm_g, int M, int groups, int nlines) {
    using G = TileGeom<T, N>;
    // odd pitch (fp64 stages are line-per-thread, no pair alignment): the j-fast
    // tile fills of the row ops hit distinct banks
    constexpr int L = G::L, LP = lg_pitch<T, N>(), NT = G::NT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_tw = tile + N * LP;
    for (int t = threadIdx.x; t < N; t += NT) {
        const double2 w = twm_g[static_cast<size_t>(t) * (M / N)];
        s_tw[t] = mk<T>(T(w.x), T(w.y));
    }
    const int bpg = (nlines + L - 1) / L;
    double r_dmax = 0.0;  // REDUCE ops: per-thread residual / status over all of the CTA's items
    int r_bad = 0;
    for (int item = blockIdx.x; item < groups * bpg; item += gridDim.x) {
        const int g = item / bpg, l0 = (item - g * bpg) * L;
        __syncthreads();
        // loads in groups of U elements, all issued before the shared-memory stores
        // (the whole item at once up to 16: one exposed HBM latency per item)
        constexpr int EPT = (N * L + NT - 1) / NT;
#ifndef GT_LG_U
#define GT_LG_U 16
#endif
        constexpr int U = EPT < GT_LG_U ? EPT : GT_LG_U;
        for (int base = threadIdx.x; base < N * L; base += NT * U) {
            cplx<T> vals[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int idx = base + u * NT;
                const int l = Op::LINE_FAST ? idx % L : idx / N, j = Op::LINE_FAST ? idx / L : idx % N;
                vals[u] = (idx < N * L && l0 + l < nlines) ? op.load(g, l0 + l, j) : mk<T>(T(0), T(0));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int idx = base + u * NT;
                const int l = Op::LINE_FAST ? idx % L : idx / N, j = Op::LINE_FAST ? idx / L : idx % N;
                if (idx < N * L) tile[j * LP + l] = vals[u];
            }
        }
#ifndef GT_LG_PF
#define GT_LG_PF 1
#endif
        if (GT_LG_PF && L >= 8) {
            // the next item's lines into L2 while this one is transformed: one prefetch per
            // 128 bytes (8 consecutive 16-byte elements: 8 lines of a line-fast op, 8 j's otherwise)
            const int nx = item + gridDim.x;
            if (nx < groups * bpg) {
                const int gn = nx / bpg, ln0 = (nx - gn * bpg) * L;
                constexpr int LP8 = L / 8 > 0 ? L / 8 : 1, NP8 = N / 8;
                for (int t = threadIdx.x; t < (Op::LINE_FAST ? LP8 * N : L * NP8); t += NT) {
                    int l, j;
                    if constexpr (Op::LINE_FAST) {
                        l = (t % LP8) * 8;
                        j = t / LP8;
                    } else {
                        l = t / NP8;
                        j = (t % NP8) * 8;
                    }
                    if (ln0 + l < nlines) op.pf(gn, ln0 + l, j);
                }
            }
        }
        __syncthreads();
        tile_fft<T, N, L, LP, NT, Op::SIGN>(tile, s_tw);
        if constexpr (TWO) {
          if (op.pack) {
            // packed ColB: unpack the 16 packed lines into the 32 columns (in place), times fk
            // (32-column items: every column transform length the DCT-row path uses, M1 <= 128)
            if constexpr (L == 32)
                for (int idx = threadIdx.x; idx < N * 16; idx += NT) op.unpack(tile, LP, g, l0, idx % 16, idx / 16);
            else
                __trap();
          } else {
            // spectral factors issued in batches ahead of their use (global / L2 latency)
            constexpr int UM = EPT < 8 ? EPT : 8;
            for (int base = threadIdx.x; base < N * L; base += NT * UM) {
                cplx<T> f[UM];
#pragma unroll
                for (int u = 0; u < UM; ++u) {
                    const int idx = base + u * NT, l = idx % L, k = idx / L;
                    f[u] = (idx < N * L && l0 + l < nlines) ? op.midw(g, l0 + l, k) : mk<T>(T(0), T(0));
                }
#pragma unroll
                for (int u = 0; u < UM; ++u) {
                    const int idx = base + u * NT, l = idx % L, k = idx / L;
                    if (idx < N * L && l0 + l < nlines) tile[k * LP + l] = cmul<T>(tile[k * LP + l], f[u]);
                }
            }
          }
            __syncthreads();
            tile_fft<T, N, L, LP, NT, -Op::SIGN>(tile, s_tw);
        }
        {
            // the store side's global inputs (twiddles, epilogue operands) in batches of US
            constexpr int US = sizeof(typename Op::Pre) > 16 ? 4 : (EPT < 8 ? EPT : 8);
            for (int base = threadIdx.x; base < N * L; base += NT * US) {
                typename Op::Pre q[US];
#pragma unroll
                for (int u = 0; u < US; ++u) {
                    const int idx = base + u * NT, l = idx % L, k = idx / L;
                    if (idx < N * L && l0 + l < nlines) q[u] = op.pre(g, l0 + l, k);
                }
#pragma unroll
                for (int u = 0; u < US; ++u) {
                    const int idx = base + u * NT, l = idx % L, k = idx / L;
                    if (idx < N * L && l0 + l < nlines) {
                        if constexpr (Op::REDUCE)
                            op.store(g, l0 + l, k, tile[k * LP + l], q[u], r_dmax, r_bad);
                        else
                            op.store(g, l0 + l, k, tile[k * LP + l], q[u]);
                    }
                }
            }
        }
    }
    if constexpr (Op::REDUCE) {
        // one atomic per CTA (a per-warp atomic on one address serialised the pass)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r_dmax = fmax(r_dmax, __shfl_xor_sync(0xffffffffu, r_dmax, o));
        r_bad = __reduce_or_sync(0xffffffffu, r_bad);
        __shared__ double s_m[NT / 32];
        __shared__ int s_b[NT / 32];
        if ((threadIdx.x & 31) == 0) {
            s_m[threadIdx.x >> 5] = r_dmax;
            s_b[threadIdx.x >> 5] = r_bad;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < NT / 32; ++w) {
                r_dmax = fmax(r_dmax, s_m[w]);
                r_bad |= s_b[w];
            }
            atomicMax(op.res_bits, static_cast<unsigned long long>(__double_as_longlong(r_dmax)));
            if (r_bad) atomicOr(op.status, r_bad);
        }
    }
}

// ------------------------------------------------ low-mode Anderson mixing on the row buffer
// The large-grid twin of fixed_point.cu's fp_lowmode (method and state: lowmode.cuh), split in
// three launches so that a multi-GPU driver (slab.py) can all-reduce the 256 coefficients
// between the projection of its row slab and the mixing step: every rank then takes the same
// step. Y: this rank's rows [rows][hy] of the row buffer (die rows row0 ..), columns q < LMK.
constexpr int LM_ROWS = 64;  // die rows per CTA of the projection / application kernels

__device__ __forceinline__ double lm_cos(int p, int x, int n) { return cospi(double(p) * (2.0 * x + 1.0) / (2.0 * n)); }

__global__ void __launch_bounds__(LMN)
lg_lowmode_project(const double2* __restrict__ Y, int hy, int rows, int row0, int n, const double2* __restrict__ hs,
                   double* __restrict__ partial) {
    const int tid = threadIdx.x, p = tid / LMK, q = tid % LMK;
    const int x0 = blockIdx.x * LM_ROWS;
    const double2 hq = hs[q];
    double acc = 0.0;
#pragma unroll 8
    for (int t = 0; t < LM_ROWS; ++t) {
        const int x = x0 + t;
        if (x < rows) {
            const double2 y = Y[static_cast<size_t>(x) * hy + q];
            acc += (hq.x * y.x - hq.y * y.y) * lm_cos(p, row0 + x, n);  // Re(hs_q Y[x][q]) cos(pi p (X + 1/2) / n)
        }
    }
    partial[static_cast<size_t>(blockIdx.x) * LMN + tid] = acc;
}

// coef[p][q] = (sum over the CTAs' partial sums, in order) / (M^2 eps_q n eps_p)
__global__ void __launch_bounds__(LMN) lg_lowmode_reduce(const double* __restrict__ partial, int nblocks, int n,
                                                         double* __restrict__ coef) {
    const int tid = threadIdx.x, p = tid / LMK, q = tid % LMK;
    double acc = 0.0;
    for (int b = 0; b < nblocks; ++b) acc += partial[static_cast<size_t>(b) * LMN + tid];
    const double M = 2.0 * n;
    coef[tid] = acc / (M * M * (q == 0 ? 1.0 : 0.5) * double(n) * (p == 0 ? 1.0 : 0.5));
}

__global__ void __launch_bounds__(LMN) lg_lowmode_init(LMState* st) {
    const int tid = threadIdx.x;
    st->xlow[tid] = 0.0;
    if (tid == 0) {
        st->calls = 0;
        st->nd = 0;
        st->have_x = 1;  // cold start: x_0 = 0
        st->have_prev = 0;
        st->rprev = 0.0;
    }
}

__global__ void __launch_bounds__(LMN) lg_lowmode_mix(LMState* st, const double* __restrict__ coef, int depth,
                                                      double res_prev, double* __restrict__ corr) {
    bool applied = false;
    corr[threadIdx.x] = lowmode_mix(*st, coef[threadIdx.x], res_prev, depth, threadIdx.x, &applied);
}

// Y[x][q] += conj(hs_q) M^2 eps_q sum_p corr_pq cos(pi p (X + 1/2) / n)
__global__ void __launch_bounds__(LMN)
lg_lowmode_apply(double2* __restrict__ Y, int hy, int rows, int row0, int n, const double2* __restrict__ hs,
                 const double* __restrict__ corr) {
    __shared__ double s_corr[LMN];
    const int tid = threadIdx.x, rg = tid / LMK, q = tid % LMK;
    s_corr[tid] = corr[tid];
    __syncthreads();
    double cq[LMK];
#pragma unroll
    for (int pp = 0; pp < LMK; ++pp) cq[pp] = s_corr[pp * LMK + q];
    const double2 hq = hs[q];
    const double M = 2.0 * n, sc = M * M * (q == 0 ? 1.0 : 0.5);
    const int x1 = min(rows, (blockIdx.x + 1) * LM_ROWS);
    for (int x = blockIdx.x * LM_ROWS + rg; x < x1; x += LMK) {
        double v = 0.0;
#pragma unroll
        for (int pp = 0; pp < LMK; ++pp) v += cq[pp] * lm_cos(pp, row0 + x, n);
        v *= sc;
        double2 y = Y[static_cast<size_t>(x) * hy + q];
        y.x += v * hq.x;  // conj(hs_q) v
        y.y -= v * hq.y;
        Y[static_cast<size_t>(x) * hy + q] = y;
    }
}

template <typename T, int N>
size_t lg_smem() {
    return sizeof(cplx<T>) * (N * lg_pitch<T, N>() + N);
}

// Packed ColB with 64-column items: the 32 packed lines (two real columns each) of the item
// fill the whole tile for the forward sub-pass (no empty slots), then the item is finished in
// two rounds of 32 columns -- packed lines 0..15 unpacked in place while 16..31 wait in
// registers, inverse sub-pass, store; then 16..31 the same way.
template <int N>
__global__ void __launch_bounds__(TileGeom<double, N>::NT, TileGeom<double, N>::MINB)
lg_colb64(ColB<double> op, const double2* __restrict__ twm_g, int M, int groups, int blocks) {
    using T = double;
    using G = TileGeom<T, N>;
    constexpr int L = G::L, LP = lg_pitch<T, N>(), NT = G::NT;
    static_assert(L == 32, "64-column items: 32 packed lines per tile");
    constexpr int EPT = (N * L + NT - 1) / NT;
    constexpr int ES = (N * 16 + NT - 1) / NT;  // stashed elements per thread
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_tw = tile + N * LP;
    for (int t = threadIdx.x; t < N; t += NT) {
        const double2 w = twm_g[static_cast<size_t>(t) * (M / N)];
        s_tw[t] = mk<T>(T(w.x), T(w.y));
    }
    for (int item = blockIdx.x; item < groups * blocks; item += gridDim.x) {
        const int b = item / groups, k2 = item - b * groups;  // block-major: items of one block run together
        const int cp0 = 32 * b;                                 // first packed line of the item
        __syncthreads();
        for (int base = threadIdx.x; base < N * L; base += NT * 16) {
            cplx<T> vals[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int idx = base + u * NT, l = idx % L, j = idx / L;
                vals[u] = (idx < N * L && cp0 + l < op.hcp)
                              ? op.C1[(static_cast<size_t>(j) + static_cast<size_t>(op.M1) * k2) * op.hcp + cp0 + l]
                              : mk<T>(T(0), T(0));
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int idx = base + u * NT, l = idx % L, j = idx / L;
                if (idx < N * L) tile[j * LP + l] = vals[u];
            }
        }
#ifndef GT_LG_CB_PF
#define GT_LG_CB_PF 0  // measured: 4.86 vs 4.57 ms per 8192^2 iteration with the prefetch on (profiles/r2s4_notes.md)
#endif
#if GT_LG_CB_PF
        // The next item's packed lines (N rows x 512 B) and its spectral factors fk (N rows x
        // 64 columns) are pulled into L2 now, so its tile loads and unpack gathers hit L2.
        {
            const int nx = item + gridDim.x;
            if (nx < groups * blocks) {
                const int nb = nx / groups, nk2 = nx - nb * groups;
                const int ncp0 = 32 * nb;
                for (int t = threadIdx.x; t < N * 4; t += NT) {
                    const int j = t >> 2, q = t & 3;
                    if (ncp0 + 8 * q < op.hcp)
                        pf_l2(op.C1 + (static_cast<size_t>(j) + static_cast<size_t>(op.M1) * nk2) * op.hcp + ncp0 + 8 * q);
                }
                for (int t = threadIdx.x; t < N * 8; t += NT) {
                    const int k1 = t >> 3, q = t & 7;
                    const int col = op.c0 + 2 * ncp0 + 8 * q;
                    if (col < op.h) pf_l2(op.fk + static_cast<size_t>(nk2 + op.M2 * k1) * op.fkp + col);
                }
            }
        }
#endif
        __syncthreads();
        tile_fft<T, N, L, LP, NT, -1>(tile, s_tw);
        cplx<T> stash[ES];
#pragma unroll
        for (int q = 0; q < ES; ++q) {
            const int idx = threadIdx.x + q * NT;
            if (idx < N * 16) stash[q] = tile[(idx / 16) * LP + 16 + idx % 16];
        }
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
            if (half == 1) {
                __syncthreads();  // round 0's stores have read the tile
#pragma unroll
                for (int q = 0; q < ES; ++q) {
                    const int idx = threadIdx.x + q * NT;
                    if (idx < N * 16) tile[(idx / 16) * LP + idx % 16] = stash[q];
                }
                __syncthreads();
            }
            // unpack packed lines cp0 + 16 half + s (slot s < 16) into slots s, s + 16 (in place)
            for (int idx = threadIdx.x; idx < N * 16; idx += NT)
                op.unpack(tile, LP, k2, 2 * (cp0 + 16 * half), idx % 16, idx / 16);
            __syncthreads();
            tile_fft<T, N, L, LP, NT, +1>(tile, s_tw);
            // store: slot s -> local column 2 (cp0 + 16 half) + 2 (s mod 16) + (s >= 16)
            constexpr int US = EPT < 8 ? EPT : 8;
            for (int base = threadIdx.x; base < N * L; base += NT * US) {
                cplx<T> w[US];
#pragma unroll
                for (int u = 0; u < US; ++u) {
                    const int idx = base + u * NT, k = idx / L;
                    w[u] = idx < N * L ? op.pre(k2, 0, k) : mk<T>(T(0), T(0));
                }
#pragma unroll
                for (int u = 0; u < US; ++u) {
                    const int idx = base + u * NT, l = idx % L, ia = idx / L;
                    if (idx >= N * L) continue;
                    const int c = 2 * (cp0 + 16 * half) + 2 * (l & 15) + (l >> 4);
                    if (c < op.hc)
                        op.C2[(static_cast<size_t>(k2) + static_cast<size_t>(op.M2) * ia) * op.hc + c] =
                            cmul<T>(tile[ia * LP + l], w[u]);
                }
            }
        }
    }
}

template <int N>
int launch_colb64_n(const ColB<double>& b, const double2* tw, int M, int groups, int blocks, cudaStream_t st) {
    const size_t smem = lg_smem<double, N>();
    static int res = 0, sms = 0;  // per N: each instantiation sets its own shared-memory attribute
    static DeviceOnce once_;
    once_([&] {
        cudaFuncSetAttribute(lg_colb64<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, lg_colb64<N>, TileGeom<double, N>::NT, smem);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        res = res < 1 ? 1 : res;
    });
    const int items = groups * blocks;
    const int grid = items < sms * res ? items : sms * res;
    if (grid > 0) lg_colb64<N><<<grid, TileGeom<double, N>::NT, smem, st>>>(b, tw, M, groups, blocks);
    return static_cast<int>(cudaGetLastError());
}

int launch_colb64(const ColB<double>& b, const double2* tw, int M, int groups, int hcp, cudaStream_t st) {
    const int blocks = (hcp + 31) / 32;
    switch (b.M1) {
        case 32: return launch_colb64_n<32>(b, tw, M, groups, blocks, st);
        case 64: return launch_colb64_n<64>(b, tw, M, groups, blocks, st);
        case 128: return launch_colb64_n<128>(b, tw, M, groups, blocks, st);
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}

template <typename T, int N, class Op, bool TWO>
int launch_n(const Op& op, const double2* tw, int M, int groups, int nlines, cudaStream_t st) {
    static int res = 0, sms = 0;
    auto k = lg_pass<T, N, Op, TWO>;
    static DeviceOnce once_;
    once_([&] {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(lg_smem<T, N>()));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, k, TileGeom<T, N>::NT, lg_smem<T, N>());
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        res = res < 1 ? 1 : res;
    });
    const int items = groups * ((nlines + TileGeom<T, N>::L - 1) / TileGeom<T, N>::L);
    const int grid = items < sms * res ? items : sms * res;
    if (grid > 0) k<<<grid, TileGeom<T, N>::NT, lg_smem<T, N>(), st>>>(op, tw, M, groups, nlines);
    return static_cast<int>(cudaGetLastError());
}

template <typename T, class Op, bool TWO = false>
int launch(int N, const Op& op, const double2* tw, int M, int groups, int nlines, cudaStream_t st) {
    switch (N) {
        case 32: return launch_n<T, 32, Op, TWO>(op, tw, M, groups, nlines, st);
        case 64: return launch_n<T, 64, Op, TWO>(op, tw, M, groups, nlines, st);
        case 128: return launch_n<T, 128, Op, TWO>(op, tw, M, groups, nlines, st);
        case 256: return launch_n<T, 256, Op, TWO>(op, tw, M, groups, nlines, st);
        case 512: return launch_n<T, 512, Op, TWO>(op, tw, M, groups, nlines, st);
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}


// ------------------------------------------------------------------ one-pass inverse rows
// The inverse row phase of one die row in ONE pass (replaces RinvA + RinvB for n <= 8192):
// the real inverse of the Hermitian half spectrum Y[0..n] at length m = 2n is an n-point
// complex inverse FFT of Z[k] = E[k] + i O[k], E = Y[k] + conj Y[n-k],
// O = (Y[k] - conj Y[n-k]) w_m^{-k}, whose output z[j] = theta[2j] + i theta[2j+1] (only
// j < n/2 is kept: the die's n samples). The whole n-point line lives in shared memory
// (128 KB at n = 8192, one CTA per SM), the Stockham stages run in place, and the epilogue
// (theta -> T, Kirchhoff inverse, residual, Chebyshev step, next applied row) is RinvB's.
template <int NT, int N>
__global__ void __launch_bounds__(NT, 1)
lg_rinv_c2r(const double2* __restrict__ Y, int hy, int rows, const double2* __restrict__ tw, int m,
            RinvB<double> op) {
    constexpr int n = N;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* buf = reinterpret_cast<double2*>(smem_raw);
    __shared__ double s_m[NT / 32];
    __shared__ int s_b[NT / 32];
    double r_dmax = 0.0;
    int r_bad = 0;
    for (int x = blockIdx.x; x < rows; x += gridDim.x) {
        const double2* Yx = Y + static_cast<size_t>(x) * hy;
        __syncthreads();  // the previous row's epilogue reads of buf are done
#pragma unroll 4
        for (int k = threadIdx.x; k < n; k += NT) {
            const double2 a = Yx[k], bq = Yx[n - k];  // k = 0 pairs with the Nyquist term Y[n]
            const double2 w = tw[k];                    // w_m^{k} -> w_m^{-k} = conj
            const double ex = a.x + bq.x, ey = a.y - bq.y;  // E = Y[k] + conj Y[n-k]
            const double dx = a.x - bq.x, dy = a.y + bq.y;  // Y[k] - conj Y[n-k]
            const double ox = dx * w.x + dy * w.y, oy = dy * w.x - dx * w.y;  // (..) w^{-k}
            buf[lpad(k)] = make_double2(ex - oy, ey + ox);  // E + i O
        }
        __syncthreads();
        // Stockham stages: radix 16 while 16 | the rest, then one radix-2/4/8 stage
        LineStages<double, NT, N, +1, 1, N>::run(buf, tw, m);
        // epilogue: theta[t], t < n, from z[t / 2]; every global input of EB elements is
        // requested before the first store (the stores may alias them for the compiler)
        const double* th = reinterpret_cast<const double*>(buf);  // (re, im) pairs = theta[2j], theta[2j+1]
        constexpr int EB = 4;
        const bool acc = op.Q != nullptr && op.om > 0.0;
#pragma unroll 1
        for (int t0 = threadIdx.x; t0 < n; t0 += NT * EB) {
            double told[EB], pv[EB], lv[EB], qv[EB];
#pragma unroll
            for (int e = 0; e < EB; ++e) {
                const int t = t0 + e * NT;
                if (t >= n) break;
                const size_t o = static_cast<size_t>(x) * n + t;
                told[e] = op.Tst[o];
                pv[e] = op.P[o];
                lv[e] = op.L0[o];
                qv[e] = acc ? op.Q[o] : 0.0;
            }
#pragma unroll
            for (int e = 0; e < EB; ++e) {
                const int t = t0 + e * NT;
                if (t >= n) break;
                const size_t o = static_cast<size_t>(x) * n + t;
                double tv = th[2 * lpad(t >> 1) + (t & 1)] * op.inv;
                if (op.kirchhoff) tv = kirchhoff_rise(tv, op.kb / op.ka, op.kexp, op.t_ambient, r_bad);
                if (!isfinite(tv)) r_bad |= GTD_ST_NONFINITE;
                r_dmax = fmax(r_dmax, fabs(tv - told[e]));
                if (op.G) op.G[o] = tv;
                if (op.Q) op.Q[o] = told[e];
                if (acc) tv = op.om * (op.gm * tv + (1.0 - op.gm) * told[e] - qv[e]) + qv[e];
                op.Tst[o] = tv;
                const double f = op.law ? exp(op.beta * tv) : 1.0 + op.beta * tv;
                op.app[o] = pv[e] + lv[e] * f;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r_dmax = fmax(r_dmax, __shfl_xor_sync(0xffffffffu, r_dmax, o));
    r_bad = __reduce_or_sync(0xffffffffu, r_bad);
    if ((threadIdx.x & 31) == 0) {
        s_m[threadIdx.x >> 5] = r_dmax;
        s_b[threadIdx.x >> 5] = r_bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < NT / 32; ++w) {
            r_dmax = fmax(r_dmax, s_m[w]);
            r_bad |= s_b[w];
        }
        atomicMax(op.res_bits, static_cast<unsigned long long>(__double_as_longlong(r_dmax)));
        if (r_bad) atomicOr(op.status, r_bad);
    }
}

// One-pass forward row phase (replaces FwdA + FwdB for n <= 8192): the spectra of the
// mirrored rows 2p, 2p+1 are their DCT-IIs, U_x[k] = conj(hs[k]) C_x[k] (hs[k] = w_m^{k/2}),
// and the DCT-II of a real length-n row is Makhoul's n-point FFT of the reordered row
// v[j] = x[2j], v[n-1-j] = x[2j+1]: C[k] = 2 Re(hs[k] V[k]). Both rows ride one complex line
// (z = v_a + i v_b, separated by Hermitian symmetry), so one n-point FFT in shared memory
// gives both rows' DCT-II coefficients, stored as the real row layout At [rows][n + 1] the
// column phase reads (ColA: U_x[v] = conj(hs[v]) At[x][v], one 8-byte load per element; the
// packed complex spectra of the four-step path were 4x the bytes and read 4 times).
template <int NT, int N>
__global__ void __launch_bounds__(NT, 1)
lg_rfwd_dct(const double* __restrict__ app, int pairs, const double2* __restrict__ tw,
            const double2* __restrict__ hs, double* __restrict__ At, int m) {
    constexpr int n = N;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* buf = reinterpret_cast<double2*>(smem_raw);
    for (int p = blockIdx.x; p < pairs; p += gridDim.x) {
        const double* xa = app + static_cast<size_t>(2 * p) * n;
        const double* xb = xa + n;
        __syncthreads();  // the previous pair's readers of buf are done
#pragma unroll 4
        for (int t = threadIdx.x; t < n; t += NT) {
            const int j = (t & 1) ? n - 1 - (t >> 1) : (t >> 1);
            buf[lpad(j)] = make_double2(xa[t], xb[t]);
        }
        __syncthreads();
        LineStages<double, NT, N, -1, 1, N>::run(buf, tw, m);
#pragma unroll 2
        for (int k = threadIdx.x; k < n; k += NT) {
            const double2 a = buf[lpad(k)], b = buf[lpad((n - k) & (n - 1))];  // Z[k], Z[n-k]
            // V_a = (Z[k] + conj Z[n-k]) / 2, V_b = (Z[k] - conj Z[n-k]) / (2i)
            const double vax = 0.5 * (a.x + b.x), vay = 0.5 * (a.y - b.y);
            const double vbx = 0.5 * (a.y + b.y), vby = -0.5 * (a.x - b.x);
            const double2 h = hs[k];
            const double ca = 2.0 * (h.x * vax - h.y * vay), cb = 2.0 * (h.x * vbx - h.y * vby);
            // the rows' real DCT-II coefficients At [2 pairs][n + 1] (C[n] = 0)
            double* Ar = At + static_cast<size_t>(2 * p) * (n + 1);
            Ar[k] = ca;
            Ar[n + 1 + k] = cb;
            if (k == 0) {
                Ar[n] = 0.0;
                Ar[2 * n + 1] = 0.0;
            }
        }
    }
}

template <int N>
int rows_fwd_dct_n(const gtd_lg* g, const double* app, int pairs, const void* hs, void* Z, cudaStream_t st) {
    constexpr int NT = N / 8 < GT_LG_RINV_NT ? N / 8 : GT_LG_RINV_NT;
    constexpr size_t smem = sizeof(double2) * (N + N / 8);
    static int res = 0, sms = 0;
    static DeviceOnce once_;
    once_([&] {
        cudaFuncSetAttribute(lg_rfwd_dct<NT, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, lg_rfwd_dct<NT, N>, NT, smem);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        res = res < 1 ? 1 : res;
    });
    const int grid = pairs < sms * res ? pairs : sms * res;
    lg_rfwd_dct<NT, N><<<grid, NT, smem, st>>>(app, pairs, static_cast<const double2*>(g->tw),
                                              static_cast<const double2*>(hs), static_cast<double*>(Z), g->m);
    return static_cast<int>(cudaGetLastError());
}

// n <= 8192 with the half-step table: the one-pass row kernels and the real DCT row layout
bool dct_rows(const gtd_lg* g) {
    static const int two_pass = getenv("GT_LG_RFWD_2PASS") ? atoi(getenv("GT_LG_RFWD_2PASS")) : 0;  // A/B switch
    return g->hs && g->n >= 512 && g->n <= 8192 && !two_pass;
}

int rows_fwd_dct(const gtd_lg* g, const double* app, int pairs, const void* hs, void* Z, cudaStream_t st) {
    switch (g->n) {
        case 512: return rows_fwd_dct_n<512>(g, app, pairs, hs, Z, st);
        case 1024: return rows_fwd_dct_n<1024>(g, app, pairs, hs, Z, st);
        case 2048: return rows_fwd_dct_n<2048>(g, app, pairs, hs, Z, st);
        case 4096: return rows_fwd_dct_n<4096>(g, app, pairs, hs, Z, st);
        case 8192: return rows_fwd_dct_n<8192>(g, app, pairs, hs, Z, st);
        default: return -1;
    }
}

template <int N>
int rows_inv_c2r_n(const gtd_lg* g, const void* Y, int hy, int pairs, const RinvB<double>& b, cudaStream_t st) {
    constexpr int NT = N / 8 < GT_LG_RINV_NT ? N / 8 : GT_LG_RINV_NT;  // one radix-8 butterfly per thread
    constexpr size_t smem = sizeof(double2) * (N + N / 8);
    static int res = 0, sms = 0;
    static DeviceOnce once_;
    once_([&] {
        cudaFuncSetAttribute(lg_rinv_c2r<NT, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, lg_rinv_c2r<NT, N>, NT, smem);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        res = res < 1 ? 1 : res;
    });
    const int rows = 2 * pairs;
    const int grid = rows < sms * res ? rows : sms * res;
    lg_rinv_c2r<NT, N><<<grid, NT, smem, st>>>(static_cast<const double2*>(Y), hy, rows,
                                              static_cast<const double2*>(g->tw), g->m, b);
    return static_cast<int>(cudaGetLastError());
}

int rows_inv_c2r(const gtd_lg* g, const void* Y, int hy, int pairs, const RinvB<double>& b, cudaStream_t st) {
    switch (g->n) {
        case 512: return rows_inv_c2r_n<512>(g, Y, hy, pairs, b, st);
        case 1024: return rows_inv_c2r_n<1024>(g, Y, hy, pairs, b, st);
        case 2048: return rows_inv_c2r_n<2048>(g, Y, hy, pairs, b, st);
        case 4096: return rows_inv_c2r_n<4096>(g, Y, hy, pairs, b, st);
        case 8192: return rows_inv_c2r_n<8192>(g, Y, hy, pairs, b, st);
        default: return -1;
    }
return static_cast<int>(cudaGetLastError());
}

}  // namespace
}  // namespace gtb

using namespace gtb;

extern "C" {

int gtd_lg_row_layout(const gtd_lg* g) { return dct_rows(g) ? 1 : 0; }

size_t gtd_lg_lowmode_state_bytes(void) { return sizeof(LMState); }
int gtd_lg_lowmode_partial_blocks(int rows) { return (rows + LM_ROWS - 1) / LM_ROWS; }
int gtd_lg_lowmode_init(void* state, cudaStream_t st) {
    lg_lowmode_init<<<1, LMN, 0, st>>>(static_cast<LMState*>(state));
    return static_cast<int>(cudaGetLastError());
}
int gtd_lg_lowmode_project(const gtd_lg* g, const void* y, int hy, int rows, int row0, double* partial, double* coef,
                           cudaStream_t st) {
    if (!g->hs || g->n < LMK) return static_cast<int>(cudaErrorInvalidValue);
    const int nb = (rows + LM_ROWS - 1) / LM_ROWS;
    lg_lowmode_project<<<nb, LMN, 0, st>>>(static_cast<const double2*>(y), hy, rows, row0, g->n,
                                           static_cast<const double2*>(g->hs), partial);
    lg_lowmode_reduce<<<1, LMN, 0, st>>>(partial, nb, g->n, coef);
    return static_cast<int>(cudaGetLastError());
}
int gtd_lg_lowmode_mix(void* state, const double* coef, int depth, double res_prev, double* corr, cudaStream_t st) {
    if (depth < 1 || depth > LMD) return static_cast<int>(cudaErrorInvalidValue);
    lg_lowmode_mix<<<1, LMN, 0, st>>>(static_cast<LMState*>(state), coef, depth, res_prev, corr);
    return static_cast<int>(cudaGetLastError());
}
int gtd_lg_lowmode_apply(const gtd_lg* g, void* y, int hy, int rows, int row0, const double* corr, cudaStream_t st) {
    if (!g->hs || g->n < LMK) return static_cast<int>(cudaErrorInvalidValue);
    const int nb = (rows + LM_ROWS - 1) / LM_ROWS;
    lg_lowmode_apply<<<nb, LMN, 0, st>>>(static_cast<double2*>(y), hy, rows, row0, g->n,
                                         static_cast<const double2*>(g->hs), corr);
    return static_cast<int>(cudaGetLastError());
}


int gtd_lg_split(int m, int* M1, int* M2) {
    int lg = 0;
    while ((1 << lg) < m) ++lg;
    if ((1 << lg) != m || m < 1024 || m > 262144) return static_cast<int>(cudaErrorInvalidValue);
    *M1 = 1 << ((lg + 1) / 2);
    *M2 = 1 << (lg / 2);
    return 0;
}

int gtd_lg_rows_fwd(const gtd_lg* g, const double* app, int pairs, void* S1, void* Z, cudaStream_t st) {
    if (dct_rows(g)) return rows_fwd_dct(g, app, pairs, g->hs, Z, st);
    FwdA<double> a{app, static_cast<double2*>(S1), static_cast<const double2*>(g->tw), g->n, g->m, g->M1};
    int e = launch<double>(g->M2, a, static_cast<const double2*>(g->tw), g->m, pairs, g->M1, st);
    if (e) return e;
    FwdB<double> b{static_cast<const double2*>(S1), static_cast<double2*>(Z), g->m, g->M1, g->M2};
    return launch<double>(g->M1, b, static_cast<const double2*>(g->tw), g->m, pairs, g->M2, st);
}

// ColA + ColB of the column phase; with DCT rows two real columns share a line through the
// first two sub-passes (half the ColA items and the C1 bytes), unpacked inside ColB.
static int cols_ab(const gtd_lg* g, ColA<double>& a, int c0, int hc, void* C1, void* C2, cudaStream_t st) {
    const bool pk = dct_rows(g) && !getenv("GT_LG_NOPACK");
    const int hcp = (hc + 1) / 2;
    if (pk) {
        a.pack = 1;
        a.hcols = hc;
        a.hc = hcp;  // C1 pitch: packed lines
    }
    int e = launch<double>(g->M2, a, static_cast<const double2*>(g->tw), g->m, g->M1, pk ? hcp : hc, st);
    if (e) return e;
    ColB<double> b{static_cast<const double2*>(C1), static_cast<double2*>(C2), static_cast<const double2*>(g->fk),
                   g->fkp, static_cast<const double2*>(g->tw), g->n + 1, g->m, g->M1, g->M2, c0, hc};
    if (pk) {
        b.pack = 1;
        b.hcp = hcp;
        b.hs = static_cast<const double2*>(g->hs);
    }
    if (pk && !getenv("GT_LG_COLB32")) return launch_colb64(b, static_cast<const double2*>(g->tw), g->m, g->M2, hcp, st);
    return launch<double, ColB<double>, true>(g->M1, b, static_cast<const double2*>(g->tw), g->m, g->M2,
                                              pk ? (hc + 31) / 32 * 32 : hc, st);
}

int gtd_lg_cols(const gtd_lg* g, const void* Z, int compact, int c0, int hc, void* C1, void* C2, void* Y,
                cudaStream_t st) {
    ColA<double> a{static_cast<const double2*>(Z), static_cast<double2*>(C1), static_cast<const double2*>(g->tw),
                   g->n, g->m, g->M1, c0, hc};
    if (compact) {
        a.zs = 2LL * hc;
        a.oa = 0;
        a.ob = hc;
        a.sb = 1;
        a.mask = 0x7fffffff;
    } else {
        a.zs = g->m;
        a.oa = c0;
        a.ob = g->m - c0;
        a.sb = -1;
        a.mask = g->m - 1;
    }
    if (dct_rows(g)) {  // real DCT rows: full [n][n + 1] or compact [n][hc] (columns c0.. of every row)
        a.At = static_cast<const double*>(Z);
        a.hA = compact ? hc : g->n + 1;
        a.aoff = compact ? 0 : c0;
        a.hs = static_cast<const double2*>(g->hs);
    }
    int e = cols_ab(g, a, c0, hc, C1, C2, st);
    if (e) return e;
    ColC<double> c{static_cast<const double2*>(C2), static_cast<double2*>(Y), g->n, g->m, g->M1, g->M2, hc};
    return launch<double>(g->M2, c, static_cast<const double2*>(g->tw), g->m, g->M1, hc, st);
}

int gtd_lg_cols_peer(const gtd_lg* g, const void* const* Zr, int pairs_per_rank, int c0, int hc, void* C1, void* C2,
                     void* const* Yr, int hy, cudaStream_t st) {
    ColA<double> a{nullptr, static_cast<double2*>(C1), static_cast<const double2*>(g->tw), g->n, g->m, g->M1, c0, hc};
    a.zs = g->m;
    a.oa = c0;
    a.ob = g->m - c0;
    a.sb = -1;
    a.mask = g->m - 1;
    a.Zr = reinterpret_cast<const double2* const*>(Zr);
    a.Pr = pairs_per_rank;
    if (dct_rows(g)) {  // each rank's real DCT rows [2 pairs][n + 1]
        a.hA = g->n + 1;
        a.aoff = c0;
        a.hs = static_cast<const double2*>(g->hs);
    }
    int e = cols_ab(g, a, c0, hc, C1, C2, st);
    if (e) return e;
    ColC<double> c{static_cast<const double2*>(C2), nullptr, g->n, g->m, g->M1, g->M2, hc};
    c.Yr = reinterpret_cast<double2* const*>(Yr);
    c.rpr = 2 * pairs_per_rank;
    c.hy = hy;
    c.c0 = c0;
    return launch<double>(g->M2, c, static_cast<const double2*>(g->tw), g->m, g->M1, hc, st);
}

int gtd_lg_rows_inv(const gtd_lg* g, const void* Y, int hy, int pairs, void* S1, double* Tst, double* app,
                    const double* P, const double* L0, const gtd_fp_opts* o, unsigned long long* res_bits,
                    int* status, double* Q, double* G, double omega, double gamma, cudaStream_t st) {
    RinvB<double> b{};
    b.S1 = static_cast<const double2*>(S1);
    b.Tst = Tst;
    b.app = app;
    b.P = P;
    b.L0 = L0;
    b.Q = Q;
    b.G = G;
    b.om = omega;
    b.gm = gamma;
    b.res_bits = res_bits;
    b.status = status;
    b.n = g->n;
    b.M = g->m;
    b.M1 = g->M1;
    b.M2 = g->M2;
    b.law = o->law;
    b.kirchhoff = o->kirchhoff;
    b.beta = o->beta;
    b.kexp = 1.0 / (1.0 - o->eta);
    b.ka = pow(o->t_ambient, 1.0 - o->eta);
    b.kb = (1.0 - o->eta) * pow(o->t_ambient, -o->eta);
    b.t_ambient = o->t_ambient;
    b.inv = 1.0 / (double(g->m) * double(g->m));
    static const int two_pass = getenv("GT_LG_RINV_2PASS") ? atoi(getenv("GT_LG_RINV_2PASS")) : 0;  // A/B switch
    if (g->n >= 512 && g->n <= 8192 && !two_pass) return rows_inv_c2r(g, Y, hy, pairs, b, st);
    RinvA<double> a{static_cast<const double2*>(Y), static_cast<double2*>(S1), static_cast<const double2*>(g->tw), g->n, g->m, g->M2, hy};
    int e = launch<double>(g->M1, a, static_cast<const double2*>(g->tw), g->m, pairs, g->M2, st);
    if (e) return e;
    return launch<double>(g->M2, b, static_cast<const double2*>(g->tw), g->m, pairs, g->M1, st);
}



// fk = FFT2(center_kernel(f_sp0 - phi)) with fk[0] += phi m^2 / 4, half width [m][fkp]
// (baseline_kernel_spectrum, greens.cpp:194-201), by the same four-step passes.
int gtd_lg_kernel_spectrum(const gtd_lg* g, const double* f_sp0, double phi, void* S1, void* Z, void* C1,
                           void* fk_out, cudaStream_t st) {
    const int n = g->n, M = g->m, pairs = n / 2;
    const double2* tw = static_cast<const double2*>(g->tw);
    FwdA<double> a{f_sp0, static_cast<double2*>(S1), tw, n, M, g->M1};
    a.embed = 1;
    a.shift = phi;
    int e = launch<double>(g->M2, a, tw, M, pairs, g->M1, st);
    if (e) return e;
    FwdB<double> b{static_cast<const double2*>(S1), static_cast<double2*>(Z), M, g->M1, g->M2};
    e = launch<double>(g->M1, b, tw, M, pairs, g->M2, st);
    if (e) return e;
    const int hc = g->fkp;  // every stored column (v >= n+1 are harmless extras)
    ColA<double> ca{static_cast<const double2*>(Z), static_cast<double2*>(C1), tw, n, M, g->M1, 0, hc};
    ca.zs = M;
    ca.oa = 0;
    ca.ob = M;
    ca.sb = -1;
    ca.mask = M - 1;
    ca.embed = 1;
    e = launch<double>(g->M2, ca, tw, M, g->M1, hc, st);
    if (e) return e;
    KColB<double> kb{static_cast<const double2*>(C1), static_cast<double2*>(fk_out), g->fkp, M, g->M1, g->M2, hc,
                     phi * double(M) * double(M) / 4.0};
    return launch<double>(g->M1, kb, tw, M, g->M2, hc, st);
}

}  // extern "C"
