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
#include <type_traits>

#include "launch_once.cuh"
#include "mc_common.cuh"

#ifndef GT_P2_ABL
#define GT_P2_ABL 0  // timing ablations of the column pass (tools/var_time.sh); 0 = the product
#endif

namespace gtb {

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

// Closed forms at a fixed mu (mu_per_sample = 0: the reference monte_carlo,
// solver.cpp:350-351,361). F_det is a table (k_fgm), so per frequency only the
// random part remains: with t1 = beta fk q + alpha g F(p_var) and
// den2 = den1 - t1, F_rand = F_det t1 / den2 (greens.cpp:241-248), one
// reciprocal; Y = F_det A_hat. F(p_var) arrives complete (the mu K1
// correction is applied to the B row spectra in stage 0).
template <typename T, int M>
struct ClosedFormMF {
    using V4 = typename Vec4<T>::type;
    static constexpr int hp = MCGeom<T, M>::hp;
    const V4* __restrict__ fg;  // [m][hp] {F_det, fk}
    const T* __restrict__ gt;   // [n+1][hp] g(du, v) (alpha multiplier, zero-padded)
    T alpha, mb;                // alpha, mu beta
    T bq4, bqs;                 // beta q = bq4 (S[ip] + S[im]) + bqs
    T mn2;                      // running minimum of |den2|^2
    __device__ __forceinline__ V4 table(int u, int v) const { return fg[static_cast<size_t>(u) * hp + v]; }
    __device__ __forceinline__ T g(int du, int v) const { return gt[du * hp + v]; }
    // C: real DCT coefficient of the applied map (A_hat = ph C); b: F(p_var) in, F_rand out.
    __device__ __forceinline__ cplx<T> eval(T C, cplx<T>& b, T ssum, cplx<T> ph, const V4& t, T gv) {
        const T ag = alpha * gv;
        const T bq = bq4 * ssum + bqs;
        const cplx<T> t1 = mk<T>(fma(bq, t.z, ag * b.x), fma(bq, t.w, ag * b.y));
        const cplx<T> den2 = mk<T>(fma(-mb, t.z, T(1) - ag) - t1.x, fma(-mb, t.w, -t1.y));
        const T d2 = cabs2<T>(den2);
        mn2 = fmin(mn2, d2);
        const cplx<T> fd = mk<T>(t.x, t.y);
        const cplx<T> num = cscale<T>(cmul<T>(t1, cconj<T>(den2)), fast_rcp(d2));
        b = cmul<T>(fd, num);
        return cscale<T>(cmul<T>(fd, ph), C);
    }
    __device__ __forceinline__ int flags() const { return mn2 < T(1e-12) ? GTD_ST_RUNAWAY_RAND : 0; }
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
template <typename T, int M, bool MF>
__global__ void __launch_bounds__(MCGeom<T, M>::NT2, MCGeom<T, M>::MINB2)
mc_pass2(const MCIn<T> in, int sample0, int count, const T* __restrict__ Areal,
         cplx<T>* __restrict__ Yspec, cplx<T>* __restrict__ Bspec, const T* __restrict__ Srow,
         gtd_sample_stats* __restrict__ stats, const cplx<T>* __restrict__ g_tw,
         const cplx<T>* __restrict__ g_hs, const T* __restrict__ fgtab, T alpha, T beta, int mu_per_sample,
         T mu_fixed, const cplx<T>* __restrict__ g_k1, const T* __restrict__ g_gtab) {
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
    static_assert(NT % GA == 0, "a thread's column group is the same in every stage-0 butterfly");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_twf = tile + (IL::SIZE > FL::SIZE ? IL::SIZE : FL::SIZE);
    cplx<T>* s_twi = s_twf + TWF;
    cplx<T>* s_hs = s_twi + TWI;
    T* s_srow = reinterpret_cast<T*>(s_hs + M);

    build_stage_tw<T, M, false, NT>(s_twf, g_tw);
    build_stage_tw<T, M, true, NT>(s_twi, g_tw);
    load_twiddles<T, M, NT>(s_hs, g_hs);
    count = in.eff_count(count);
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

        // mu K1 correction of the B rows (fixed-mu closed forms): the row spectrum
        // of the centred p_var row is B - mu k1(v) (p_var = p_leak0 - mu on the die)
        const double n2 = double(n) * double(n);
        const double mu_s = stats[sg].sum_leak / n2;
        cplx<T> k1m[CG];
        if constexpr (MF) {
#pragma unroll
            for (int col = 0; col < CG; ++col) {
                const cplx<T> k = g_k1[v0 + (threadIdx.x % GA) + col * GA];
                k1m[col] = mk<T>(T(mu_s) * k.x, T(mu_s) * k.y);
            }
        }
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
#if GT_P2_ABL == 5  // timing ablation: no stage-0 global loads
                v[b][0][r] = mk<T>(T(xa), T(va));
                if (r < 2 || r >= 6) {
                    v[b][1][r] = mk<T>(T(xb), T(r));
                    v[b][2][r] = mk<T>(T(r), T(xb));
                }
                continue;
#endif
                // columns va and va + GA are adjacent in A's rows (a_col): one 8-byte load
                const T* ar = Areal + sbase + static_cast<size_t>(xa) * hp + va;
                v[b][0][r] = mk<T>(ar[0], CG == 2 ? ar[GA] : T(0));
                // the centre embedding fills rows [0, M/4) u [3M/4, M): r in {0,1,6,7} only
                if (r < 2 || r >= 6) {
                    const cplx<T>* bp = Bspec + sbase + static_cast<size_t>(xb) * hp + va;
                    v[b][1][r] = bp[0];
                    v[b][2][r] = CG == 2 ? bp[GA] : mk<T>(T(0), T(0));
                    if constexpr (MF) {
                        v[b][1][r] = csub<T>(v[b][1][r], k1m[0]);
                        if (CG == 2) v[b][2][r] = csub<T>(v[b][2][r], k1m[CG - 1]);
                    }
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
                // S: tiles beyond column c read column c's segment (see the S loads below)
                const size_t nbS = static_cast<size_t>(sn) * n * hp + static_cast<size_t>(min(tn * W, (c / W) * W));
                constexpr int LA = (W * int(sizeof(T)) + 127) / 128, LB = (W * int(sizeof(cplx<T>)) + 127) / 128;
                constexpr int PER = 2 * LA + LB;  // A and S segments, then B
#pragma unroll
                for (int t = threadIdx.x; t < n * PER; t += NT) {
                    const int k = t / n, x = t - k * n;  // n: power of two
                    const size_t o = nb + static_cast<size_t>(x) * hp;
                    if (k < LA)
                        prefetch_l2(reinterpret_cast<const char*>(Areal + o) + 128 * k);
                    else if (k < 2 * LA)
                        prefetch_l2(reinterpret_cast<const char*>(Srow + nbS + static_cast<size_t>(x) * hp) +
                                    128 * (k - LA));
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
            // S columns beyond c are all equal to column c (pass 1 writes [0, c] only)
            sv[k] = idx < n * W ? Srow[sbase + static_cast<size_t>(idx / W) * hp + min(v0 + idx % W, c)] : T(0);
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
        const T* Nm = in.nn(sg);
        const T* Vm = in.v(sg);
        using CF = std::conditional_t<MF, ClosedFormMF<T, M>, ClosedForm<T, M>>;
        CF cf;
        cf.fg = reinterpret_cast<const typename Vec4<T>::type*>(fgtab);
        if constexpr (MF) {
            cf.mb = mu_fixed * beta;
            cf.alpha = alpha;
            cf.gt = g_gtab;
        } else {
            cf.mug = mu_per_sample ? T(mu_s) : mu_fixed;
            cf.mb = cf.mug * beta;
            cf.mus = T(mu_s);
            cf.mn1 = Real<T>::max();
        }
        cf.bq4 = T(0.25) * beta;
        {
            const T pl_cc = in.nom_scale * Nm[c * n + c] * Vm[c * n + c];
            const T pl_00 = in.nom_scale * Nm[0] * Vm[0];
            cf.bqs = beta * T(double(pl_cc) - double(pl_00) - mu_s);  // q shift, greens.cpp:177-184
        }
        cf.mn2 = Real<T>::max();
        __syncthreads();
        // ---- middle forward stages
#if GT_P2_ABL != 4  // timing ablation 4: without the middle forward stage
        FwdStagesAB<T, M, GA, NT, 1, K - 1>::run(tile, s_twf);
#endif
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
                        cplx<T> bb = z[b][1 + col][q];
                        const cplx<T> ph = cconj<T>(cmul<T>(s_hs[u], hv));
#if GT_P2_ABL == 1  // timing ablation: table load, no closed form
                        if constexpr (MF) {
                            const auto t4 = cf.table(u, vv);
                            const T C = col == 0 ? z[b][0][q].x : z[b][0][q].y;
                            yr[0][q] = mk<T>(C * t4.x, C * t4.y);
                        } else
#elif GT_P2_ABL == 2  // timing ablation: no table, no closed form
                        if constexpr (MF) {
                            const T C = col == 0 ? z[b][0][q].x : z[b][0][q].y;
                            yr[0][q] = mk<T>(C * ph.x, C * ph.y);
                        } else
#endif
                        if constexpr (MF)
                            yr[0][q] = cf.eval(col == 0 ? z[b][0][q].x : z[b][0][q].y, bb,
                                               s_srow[sp + w] + s_srow[sm + w], ph, cf.table(u, vv), cf.g(du, vv));
                        else
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
        {   // conditioning: max 1/|den2|^2 (positive floats order like their bit patterns)
            const float rd = float(T(1) / fmax(cf.mn2, Real<T>::min_pos()));
            const float wm = warp_max_t<float>(rd);
            if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(&stats[sg].max_rden2), __float_as_int(wm));
        }
        // ---- middle inverse stages
#if GT_P2_ABL != 3  // timing ablation 3: without the middle inverse stage
        InvStagesPairs<T, M, W, NT, 1, K - 1>::run(tile, s_twi);
#endif
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
#if GT_P2_ABL == 6  // timing ablation: no global stores (kept alive by an impossible condition)
                    if (o[0][r].x == T(1.2345e-30) && o[1][r].y == T(-7.5e-31)) Yspec[0] = o[0][r];
                    continue;
#endif
                    if (i < n) Yspec[sbase + static_cast<size_t>(i) * hp + vv] = o[0][r];
                    const int x = (i + c) & (M - 1);
                    if (x < n) Bspec[sbase + static_cast<size_t>(x) * hp + vv] = o[1][r];
                }
            }
        }
    }
}

__global__ void mc_finalize(gtd_sample_stats* stats, int sample0, int count, int n, int det_flags,
                            const int* dcnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (dcnt) count = min(*dcnt, count);
    if (i >= count) return;
    gtd_sample_stats& st = stats[sample0 + i];
    st.status |= det_flags;  // fixed-mu den1 runaway (checked once when the table was built)
    st.max_rise = __longlong_as_double(static_cast<long long>(st.max_bits));
    st.mean_rise = st.sum_rise / (double(n) * double(n));
}

// ------------------------------------------------- fp64 re-solve of ill-conditioned pairs
// Pairs whose fp32 closed forms met a near-singular random_greens denominator
// (max 1/|den2|^2 > thr) amplify the fp32 rounding of their inputs beyond the
// 1e-3 K bar; they are solved again in fp64 (BASELINE config 1: "fp32 with fp64
// residual check"). sel[0] counts, sel[1..cap] lists the selected samples.
__global__ void mc_resolve_select(gtd_sample_stats* __restrict__ stats, int batch, float thr, int* __restrict__ sel,
                                  int cap) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= batch) return;
    gtd_sample_stats& st = stats[i];
    if (st.status != 0 || !(st.max_rden2 > thr)) return;  // failed pairs stay failed
    const int slot = atomicAdd(sel, 1);
    if (slot < cap)
        sel[1 + slot] = i;
    else
        st.status |= GTD_ST_ILLCOND;
}

// fp32 inputs of the selected pairs -> fp64 [slot][P, N, V] (exact widening).
template <typename T>
__global__ void mc_resolve_gather(const MCIn<T> in, const int* __restrict__ sel, int cap, int n,
                                  double* __restrict__ in64) {
    const int slot = blockIdx.y;
    if (slot >= min(sel[0], cap)) return;
    const size_t s = static_cast<size_t>(sel[1 + slot]), nn = static_cast<size_t>(n) * n;
    const T* P = in.p(s);
    const T* N = in.nn(s);
    const T* V = in.v(s);
    double* o = in64 + slot * 3 * nn;
    for (size_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nn; k += gridDim.x * blockDim.x) {
        o[k] = double(P[k]);
        o[nn + k] = double(N[k]);
        o[2 * nn + k] = double(V[k]);
    }
}

// fp64 results -> the fp32 outputs and stats of the selected pairs; a negative
// max_rden2 marks a pair as re-solved in fp64.
template <typename T>
__global__ void mc_resolve_scatter(const int* __restrict__ sel, int cap, int n, const double* __restrict__ out64,
                                   const gtd_sample_stats* __restrict__ stats64, T* __restrict__ out,
                                   gtd_sample_stats* __restrict__ stats) {
    const int slot = blockIdx.y;
    if (slot >= min(sel[0], cap)) return;
    const size_t s = static_cast<size_t>(sel[1 + slot]), nn = static_cast<size_t>(n) * n;
    if (out)
        for (size_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nn; k += gridDim.x * blockDim.x)
            out[s * nn + k] = T(out64[slot * nn + k]);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const float rd = stats[s].max_rden2;
        stats[s] = stats64[slot];
        stats[s].max_rden2 = -rd;
    }
}

// ------------------------------------------------------------------ host side
template <typename T, int M>
struct MCLaunch {
    using Gm = MCGeom<T, M>;
    static constexpr int GA2 = Gm::W >= 2 ? Gm::W / 2 : 1;
    static size_t smem2() {
        constexpr int FS = FwdLayout<T, GA2, M>::SIZE, IS = InvLayout<Gm::W, M>::SIZE;
        return sizeof(cplx<T>) * ((FS > IS ? FS : IS) + StageTw<M, false>::SIZE + StageTw<M, true>::SIZE + M) +
               sizeof(T) * Gm::n * Gm::W;
    }

    static int run(const gtd_greens* g, const MCIn<T>& in, int batch, const gtd_mc_opts* o,
                   T* out, gtd_sample_stats* stats, void* scratch, int chunk, cudaStream_t st,
                   gtd_mark_fn mark, void* ctx) {
        constexpr int n = Gm::n, hp = Gm::hp, W = Gm::W;
        constexpr int CT = hp / W;
        // Kernel attributes and resident CTAs per SM, set up once per (T, M) and device
        // (launch_once.cuh; every device of a node is the same sm_100a part).
        struct Occ {
            int res[3];
            int sms;
        };
        static Occ occ{{1, 1, 1}, 1};
        static DeviceOnce once_;
        once_([] { occ = [] {
            Occ r{{0, 0, 0}, 0};
            r.res[0] = mc_rows_setup<T, M>(1);
            r.res[2] = mc_rows_setup<T, M>(3);
            cudaFuncSetAttribute(mc_pass2<T, M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2()));
            cudaFuncSetAttribute(mc_pass2<T, M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2()));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r.res[1], mc_pass2<T, M, false>, Gm::NT2, smem2());
            int r2 = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r2, mc_pass2<T, M, true>, Gm::NT2, smem2());
            r.res[1] = r2 < r.res[1] ? r2 : r.res[1];
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&r.sms, cudaDevAttrMultiProcessorCount, dev);
            for (int& x : r.res) x = x < 1 ? 1 : x;
            return r;
        }(); });
        const int* res = occ.res;
        const int sms = occ.sms;
        const size_t per = static_cast<size_t>(n) * hp;
        const cplx<T>* hs = reinterpret_cast<const cplx<T>*>(g->hs);
        const cplx<T>* tw = reinterpret_cast<const cplx<T>*>(g->tw);
        const T var_lo = T(exp(-o->exponent_cap)), var_hi = T(exp(o->exponent_cap));
        auto grid = [&](int items, int r) { return items < sms * r ? items : sms * r; };
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
        // fixed-mu closed forms (the reference monte_carlo's gs.mu) read the k_fgm table
        static const int no_fgm = getenv("GT_MC_NO_FGM") ? atoi(getenv("GT_MC_NO_FGM")) : 0;  // A/B switch
        const bool mf = !o->mu_per_sample && g->fgm != nullptr && !no_fgm;
        cudaMemsetAsync(stats, 0, sizeof(gtd_sample_stats) * batch, st);
        for (int s0 = 0; s0 < batch; s0 += chunk) {
            const int cnt = batch - s0 < chunk ? batch - s0 : chunk;
            cudaStream_t ss = st;
            gtd_mark_fn mk_ = mark;
            cplx<T>* A = static_cast<cplx<T>*>(scratch);  // Y (pass 2 -> pass 3)
            cplx<T>* B = A + per * chunk;                  // B (pass 1 -> 2), R (pass 2 -> 3)
            T* S = reinterpret_cast<T*>(B + per * chunk);   // row-symmetrised leakage
            T* Ar = S + per * chunk;                        // real DCT part of A (pass 1 -> 2)
            MCRowArgs<T> ra{in, s0, cnt, Ar, A, B, S, stats, tw, hs, var_lo, var_hi, out, T(g->rand_scale), o->with_rand};
            if (mk_) mk_(ctx, 0, ss);
            mc_rows_launch<T, M>(1, tma1, sms, res[0], ss, ra);
            if (mk_) mk_(ctx, 1, ss);
            const cplx<T>* k1 = static_cast<const cplx<T>*>(g->k1);
            if (mf)
                mc_pass2<T, M, true><<<grid(cnt * CT, res[1]), Gm::NT2, smem2(), ss>>>(
                    in, s0, cnt, Ar, A, B, S, stats, tw, hs, static_cast<const T*>(g->fgm), T(g->alpha),
                    T(g->beta), 0, T(g->mu_fixed), k1, static_cast<const T*>(g->gtab));
            else
                mc_pass2<T, M, false><<<grid(cnt * CT, res[1]), Gm::NT2, smem2(), ss>>>(
                    in, s0, cnt, Ar, A, B, S, stats, tw, hs, static_cast<const T*>(g->fg), T(g->alpha),
                    T(g->beta), o->mu_per_sample, T(g->mu_fixed), k1, nullptr);
            if (mk_) mk_(ctx, 2, ss);
            mc_rows_launch<T, M>(3, tma3, sms, res[2], ss, ra);
            if (mk_) mk_(ctx, 3, ss);
        }
        mc_finalize<<<(batch + 127) / 128, 128, 0, st>>>(stats, 0, batch, n, mf ? g->det_flags : 0, in.dcnt);
        if constexpr (sizeof(T) == 4) {
            if (o->resolve) {
                const gtd_mc_resolve* r = o->resolve;
                const size_t nn = static_cast<size_t>(n) * n;
                cudaMemsetAsync(r->sel, 0, sizeof(int), st);
                mc_resolve_select<<<(batch + 255) / 256, 256, 0, st>>>(stats, batch, r->thr, r->sel, r->cap);
                mc_resolve_gather<T><<<dim3(32, r->cap), 256, 0, st>>>(in, r->sel, r->cap, n,
                                                                         static_cast<double*>(r->in64));
                MCIn<double> i64;
                i64.P = static_cast<const double*>(r->in64);
                i64.N = i64.P + nn;
                i64.V = i64.P + 2 * nn;
                i64.sP = i64.sN = i64.sV = static_cast<long long>(3 * nn);
                i64.nom_scale = in.nom64;
                i64.nom64 = in.nom64;
                i64.dcnt = r->sel;
                gtd_mc_opts o64 = *o;
                o64.resolve = nullptr;
                const int e = MCLaunch<double, M>::run(r->g64, i64, r->cap, &o64, static_cast<double*>(r->out64),
                                                       r->stats64, r->scratch64, r->cap, st, nullptr, nullptr);
                if (e) return e;
                mc_resolve_scatter<T><<<dim3(32, r->cap), 256, 0, st>>>(r->sel, r->cap, n,
                                                                          static_cast<const double*>(r->out64),
                                                                          r->stats64, out, stats);
            }
        }
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
    in.nom64 = i->nom_scale;
    in.dcnt = nullptr;
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

int gtd_mc_resolve_launch_count(void) { return 3 + 4 + 1; }  // select, gather, 3 passes, finalize, scatter

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
