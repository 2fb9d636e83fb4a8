// trace_batch.cu — config 3: batched transient traces with the leakage
// update applied every step (north-star subsystem 5 + subsystem 4).
//
// Per trace (oracle: oracle/restate.cpp ref_trace_leak_batch, which drives the
// reference's own time_varying_profile, solver.cpp:212-287, step by step):
//   P_n = P_dyn,n + L0 o f(T_{n-1})       f = 1 + beta dT (variation.cpp:213-222) or exp
//   T_n = max(0, crop(IFFT(acc_n)))      acc_n = windowed superposition, window k
// The window sum is carried by the per-mode recursion of SURVEY §8a D10 in the
// form that needs ONE spectral state Z = F (P^_n - E_n) per trace:
//   Z_n = (1 - r) F P^_n + r Z_{n-1} + [n > k] r^{k+1} F Delta^_{n-k}
// with r = exp(-dt / tau) per mode (solver.cpp:129-149), P^_n = FFT(mirror(P_n))
// and Delta^_{n-k} = FFT(mirror(P_{n-k} - P_{n-k-1})). Both inputs are mirrored
// real maps, so one packed complex line per row / column carries both, and the
// column transform separates them locally through their real DCT parts.
//
// Kernels per step (batched over traces):
//   tr_rows_fwd : rows of P_n and d_{n-k} from the per-trace power ring -> packed
//                 row FFT -> the two rows' real DCT parts (complex pair per cell)
//   tr_cols     : column FFT of the pairs, the Z update in registers against the
//                 L2-resident tables {(1-r)F, r, r^{k+1} F}, inverse column FFT
//   tr_rows_inv : inverse rows (two rows per line) -> T_n -> stored frame ->
//                 P_{n+1} = P_dyn(blocks, schedule) + L0 f(T_n) into the ring
#include <cuda_runtime.h>

#include <cstdint>

#include "launch_once.cuh"
#include "col_pass.cuh"
#include "fft_tile.cuh"
#include "fft_warp.cuh"
#include "gt_device.h"

namespace gtb {
namespace {

template <typename T, int M>
struct TRGeom {
    using G = TileGeom<T, M>;
    static constexpr int n = M / 2, h = n + 1;
    static constexpr int L = G::L, LP = L + 2, NT = G::NT;
    static constexpr int GA = L / 2 > 0 ? L / 2 : 1;  // column pairs per column tile
    static constexpr int W = 2 * GA;
    static constexpr int hp = ((h + W - 1) / W) * W;
    static constexpr int CT = hp / W;
    static constexpr int RB = (n + L - 1) / L;        // row blocks (forward rows)
    static constexpr int RPB = (n / 2 + L - 1) / L;   // row-pair blocks (inverse rows)
    static constexpr int U8 = (M / 8) * GA;
    static constexpr int NTC = U8 >= 256 ? 256 : (U8 < 32 ? 32 : U8);
    static constexpr int MINBC = sizeof(T) == 8 ? 1 : ((512 / NTC) < 1 ? 1 : 512 / NTC);
    static constexpr int TILEC = InvLayout<GA, M>::SIZE;
};

struct TRStep {
    int step;       // 1-based step n
    int slot_n;     // ring slot of P_n
    int slot_k;     // ring slot of P_{n-k} (valid if has_k)
    int slot_k1;    // ring slot of P_{n-k-1}, -1 for P_0 = 0
    int has_k;      // n > k
    int slot_next;  // ring slot for P_{n+1}; -1 on the last step
    int frame;      // output frame index of T_n, -1 if not stored
};

template <typename T>
struct TRBuf {
    T* ring;            // [B][k+2][n*n]
    size_t ring_stride; // per trace, elements
    cplx<T>* D;         // [B][n][hp] packed DCT pairs, then Y rows
    cplx<T>* Z;         // [B][M][hp] spectral state
    const int* blk;
    long long blk_stride;
    const T* sched;     // [B][steps][nblk]
    int nblk, steps;
    const T* leak0;
    long long leak_stride;
};

// ---------------------------------------------------------------- rows forward
template <typename T, int M>
__global__ void __launch_bounds__(TileGeom<T, M>::NT, TileGeom<T, M>::MINB)
tr_rows_fwd(int b0, int count, TRBuf<T> bf, TRStep sp, const cplx<T>* __restrict__ g_tw,
            const cplx<T>* __restrict__ g_hs) {
    using Gm = TRGeom<T, M>;
    constexpr int n = Gm::n, L = Gm::L, LP = Gm::LP, NT = Gm::NT, hp = Gm::hp, RB = Gm::RB;
    constexpr size_t nn = size_t(n) * n;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_tw = tile + M * LP;
    cplx<T>* s_hs = s_tw + M;
    load_twiddles<T, M, NT>(s_tw, g_tw);
    for (int t = threadIdx.x; t < n; t += NT) s_hs[t] = g_hs[t];
    for (int item = blockIdx.x; item < count * RB; item += gridDim.x) {
        const int b = item / RB, x0 = (item - b * RB) * L;
        const T* ring = bf.ring + static_cast<size_t>(b0 + b) * bf.ring_stride;
        const T* Pn = ring + sp.slot_n * nn;
        const T* Pk = ring + sp.slot_k * nn;
        const T* Pk1 = sp.slot_k1 >= 0 ? ring + sp.slot_k1 * nn : nullptr;
        __syncthreads();
        // z = mirror(P_n row) + i mirror(d_{n-k} row): every tile row is written
        for (int idx = threadIdx.x; idx < L * n; idx += NT) {
            const int l = idx / n, y = idx - l * n, x = x0 + l;
            cplx<T> z = mk<T>(T(0), T(0));
            if (x < n) {
                const size_t o = static_cast<size_t>(x) * n + y;
                T d = T(0);
                if (sp.has_k) d = Pk[o] - (Pk1 ? Pk1[o] : T(0));
                z = mk<T>(Pn[o], d);
            }
            tile[y * LP + l] = z;
            tile[(M - 1 - y) * LP + l] = z;
        }
        __syncthreads();
        tile_fft<T, M, L, LP, NT, -1>(tile, s_tw);
        cplx<T>* Db = bf.D + static_cast<size_t>(b0 + b) * n * hp;
        for (int idx = threadIdx.x; idx < L * hp; idx += NT) {
            const int l = idx / hp, v = idx - l * hp, x = x0 + l;
            if (x >= n) continue;
            cplx<T> o = mk<T>(T(0), T(0));
            if (v < n) {
                const cplx<T> Zv = tile[v * LP + l];
                const cplx<T> Zc = cconj<T>(tile[((M - v) & (M - 1)) * LP + l]);
                o = mk<T>(dct_part<T>(Zv, Zc, s_hs[v]), dct_part_im<T>(Zv, Zc, s_hs[v]));
            }
            Db[static_cast<size_t>(x) * hp + v] = o;
        }
    }
}

// ---------------------------------------------------------------- columns
// Tile of W = 2 GA columns, lines paired (v0 + g, v0 + g + GA) in InvLayout for
// both the forward and the inverse phase. Line of column v: P~_v + i d~_v
// (real DCT parts); forward FFT gives Z[u] with C_P + i C_d = w^{u/2} Z[u].
template <typename T, int M>
__global__ void __launch_bounds__(TRGeom<T, M>::NTC, TRGeom<T, M>::MINBC)
tr_cols(int b0, int count, TRBuf<T> bf, TRStep sp, const cplx<T>* __restrict__ g_tw,
        const cplx<T>* __restrict__ g_hs, const cplx<T>* __restrict__ tab) {
    using Gm = TRGeom<T, M>;
    using Pl = Plan<M>;
    using IL = InvLayout<Gm::GA, M>;
    constexpr int n = Gm::n, GA = Gm::GA, W = Gm::W, hp = Gm::hp, CT = Gm::CT, NT = Gm::NTC;
    constexpr int K = Pl::K, RL = Pl::RLAST_F;
    constexpr int U0 = (M / 8) * GA, B0 = U0 / NT;
    constexpr int UL = (M / RL) * GA, BL = UL / NT;
    constexpr int TWF = StageTw<M, false>::SIZE, TWI = StageTw<M, true>::SIZE;
    constexpr size_t plane = size_t(M) * hp;
    static_assert(K >= 2 && Pl::fr(0) == 8 && Pl::ir(K - 1) == 8, "plan");
    static_assert(U0 % NT == 0 && UL % NT == 0 && B0 >= 1, "threads");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_twf = tile + Gm::TILEC;
    cplx<T>* s_twi = s_twf + TWF;
    cplx<T>* s_hs = s_twi + TWI;
    build_stage_tw<T, M, false, NT>(s_twf, g_tw);
    build_stage_tw<T, M, true, NT>(s_twi, g_tw);
    for (int t = threadIdx.x; t < M; t += NT) s_hs[t] = g_hs[t];

    for (int item = blockIdx.x; item < count * CT; item += gridDim.x) {
        const int b = item / CT, v0 = (item - b * CT) * W;
        cplx<T>* Db = bf.D + static_cast<size_t>(b0 + b) * n * hp;
        cplx<T>* Zb = bf.Z + static_cast<size_t>(b0 + b) * plane;
        __syncthreads();
        // ---- stage 0 straight from the packed DCT rows (mirror in the address)
#pragma unroll
        for (int bb = 0; bb < B0; ++bb) {
            const int id = threadIdx.x + bb * NT;
            const int g = id % GA, j = id / GA;
            cplx<T> va[8], vb[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int i = j + r * (M / 8);
                const int xa = i < n ? i : M - 1 - i;
                const cplx<T>* dp = Db + static_cast<size_t>(xa) * hp + v0 + g;
                va[r] = dp[0];
                vb[r] = dp[GA];
            }
            dftR<8, -1, T>(va);
            dftR<8, -1, T>(vb);
#pragma unroll
            for (int r = 0; r < 8; ++r) st_pair(&tile[IL::template off<1>(j * 8, r, g)], LinePair<T>{va[r], vb[r]});
        }
        __syncthreads();
        InvStagesPairs<T, M, GA, NT, 1, K - 1, false>::run(tile, s_twf);
        // ---- last forward stage + state update + first inverse stage
        {
            cplx<T> y[BL][2][RL];
#pragma unroll
            for (int bb = 0; bb < BL; ++bb) {
                const int id = threadIdx.x + bb * NT;
                const int g = id % GA, j = id / GA;
#pragma unroll
                for (int q = 0; q < RL; ++q) {
                    const LinePair<T> p = ld_pair(&tile[IL::template off<M / RL>(j, q, g)]);
                    y[bb][0][q] = p.a;
                    y[bb][1][q] = p.b;
                }
                stage_twiddle<T, M, false, K - 1, 2>(y[bb], j, s_twf);
                dftR<RL, -1, T>(y[bb][0]);
                dftR<RL, -1, T>(y[bb][1]);
                // the state and table entries of this butterfly's 2 RL points, all issued
                // before any state store (the stores to Zb would otherwise pin each load
                // behind the previous point's store: one L2/HBM round trip per point).
                // Each state entry is read and written by this thread only, once per
                // launch, so the read-only path is safe.
                // (RL > 2: 8 RL operands would not fit the register budget; per point.)
                constexpr bool BATCH = RL <= 2;
                constexpr int RB = BATCH ? RL : 1;
                cplx<T> zo[2][RB], ta[2][RB], tr[2][RB], tb[2][RB];
                if constexpr (BATCH) {
#pragma unroll
                    for (int col = 0; col < 2; ++col)
#pragma unroll
                        for (int q = 0; q < RB; ++q) {
                            const size_t o = static_cast<size_t>(j + q * (M / RL)) * hp + v0 + g + col * GA;
                            zo[col][q] = __ldg(&Zb[o]);
                            ta[col][q] = tab[o];
                            tr[col][q] = tab[plane + o];
                            tb[col][q] = sp.has_k ? tab[2 * plane + o] : mk<T>(T(0), T(0));
                        }
                }
#pragma unroll
                for (int col = 0; col < 2; ++col) {
                    const int vv = v0 + g + col * GA;
                    const cplx<T> hv = s_hs[vv];
#pragma unroll
                    for (int q = 0; q < RL; ++q) {
                        const int u = j + q * (M / RL);
                        const cplx<T> hu = s_hs[u];
                        const cplx<T> Cz = cmul<T>(hu, y[bb][col][q]);  // C_P + i C_d
                        const cplx<T> ph = cconj<T>(cmul<T>(hu, hv));
                        const size_t o = static_cast<size_t>(u) * hp + vv;
                        const int qb = BATCH ? q : 0;
                        if constexpr (!BATCH) {
                            zo[col][0] = __ldg(&Zb[o]);
                            ta[col][0] = tab[o];
                            tr[col][0] = tab[plane + o];
                            tb[col][0] = sp.has_k ? tab[2 * plane + o] : mk<T>(T(0), T(0));
                        }
                        const cplx<T> a = ta[col][qb], r = tr[col][qb], bk = tb[col][qb];
                        cplx<T> zs = cmul<T>(r, zo[col][qb]);
                        const cplx<T> aP = cmul<T>(a, ph);
                        zs = mk<T>(zs.x + aP.x * Cz.x, zs.y + aP.y * Cz.x);
                        if (sp.has_k) {
                            const cplx<T> bD = cmul<T>(bk, ph);
                            zs = mk<T>(zs.x + bD.x * Cz.y, zs.y + bD.y * Cz.y);
                        }
                        Zb[o] = zs;
                        y[bb][col][q] = zs;
                    }
                    dftR<RL, +1, T>(y[bb][col]);
                }
            }
            __syncthreads();
#pragma unroll
            for (int bb = 0; bb < BL; ++bb) {
                const int id = threadIdx.x + bb * NT;
                const int g = id % GA, j = id / GA;
#pragma unroll
                for (int r = 0; r < RL; ++r)
                    st_pair(&tile[IL::template off<1>(j * RL, r, g)], LinePair<T>{y[bb][0][r], y[bb][1][r]});
            }
            __syncthreads();
        }
        InvStagesPairs<T, M, GA, NT, 1, K - 1, true>::run(tile, s_twi);
        // ---- last inverse stage: rows [0, n) of both columns, into D (in place)
#pragma unroll
        for (int bb = 0; bb < (M / 8) * GA / NT; ++bb) {
            const int id = threadIdx.x + bb * NT;
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
                    cplx<T>* yr = Db + static_cast<size_t>(i) * hp + v0 + g;
                    yr[0] = o[0][r];
                    yr[GA] = o[1][r];
                }
            }
        }
    }
}

// ---------------------------------------------------------------- rows inverse
template <typename T, int M>
__global__ void __launch_bounds__(TileGeom<T, M>::NT, TileGeom<T, M>::MINB)
tr_rows_inv(int b0, int count, TRBuf<T> bf, TRStep sp, int nframes, int law, T beta, T* __restrict__ out,
            double* __restrict__ fmax_bits, const cplx<T>* __restrict__ g_tw) {
    using Gm = TRGeom<T, M>;
    constexpr int n = Gm::n, h = Gm::h, L = Gm::L, LP = Gm::LP, NT = Gm::NT, hp = Gm::hp, RPB = Gm::RPB;
    constexpr size_t nn = size_t(n) * n;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_tw = tile + M * LP;
    load_twiddles<T, M, NT>(s_tw, g_tw);
    constexpr T inv = T(1.0 / (double(M) * double(M)));
    for (int item = blockIdx.x; item < count * RPB; item += gridDim.x) {
        const int b = item / RPB, p0 = (item - b * RPB) * L;
        const int bg = b0 + b;
        const cplx<T>* Yb = bf.D + static_cast<size_t>(bg) * n * hp;
        __syncthreads();
        for (int idx = threadIdx.x; idx < L * h; idx += NT) {
            const int l = idx / h, v = idx - l * h;
            const int xa = 2 * (p0 + l);
            cplx<T> y = mk<T>(T(0), T(0)), r = y;
            if (xa < n) {
                y = Yb[static_cast<size_t>(xa) * hp + v];
                r = Yb[static_cast<size_t>(xa + 1) * hp + v];
            }
            if (v == 0 || v == n) {
                tile[v * LP + l] = mk<T>(y.x, r.x);
            } else {
                tile[v * LP + l] = mk<T>(y.x - r.y, y.y + r.x);
                tile[(M - v) * LP + l] = mk<T>(y.x + r.y, r.x - y.y);
            }
        }
        __syncthreads();
        tile_fft<T, M, L, LP, NT, +1>(tile, s_tw);
        T* ring = bf.ring + static_cast<size_t>(bg) * bf.ring_stride;
        T* Pnext = sp.slot_next >= 0 ? ring + sp.slot_next * nn : nullptr;
        const int* blk = bf.blk + static_cast<size_t>(bg) * bf.blk_stride;
        const T* sch = bf.sched + (static_cast<size_t>(bg) * bf.steps + (sp.step < bf.steps ? sp.step : 0)) * bf.nblk;
        const T* L0 = bf.leak0 + static_cast<size_t>(bg) * bf.leak_stride;
        T* O = sp.frame >= 0 ? out + (static_cast<size_t>(bg) * nframes + sp.frame) * nn : nullptr;
        T mx = T(0);
        for (int idx = threadIdx.x; idx < 2 * L * n; idx += NT) {
            const int lr = idx / n, j = idx - lr * n;
            const int l = lr >> 1, half = lr & 1;
            const int x = 2 * p0 + lr;
            if (x >= n) continue;
            const cplx<T> z = tile[j * LP + l];
            T t = (half ? z.y : z.x) * inv;
            t = t > T(0) ? t : T(0);  // clamp_negatives (solver.cpp:33-46)
            const size_t o = static_cast<size_t>(x) * n + j;
            if (O) O[o] = t;
            mx = mx > t ? mx : t;
            if (Pnext) {
                const T f = law ? T(exp(beta * t)) : T(1) + beta * t;
                Pnext[o] = sch[blk[o]] + L0[o] * f;
            }
        }
        if (O && fmax_bits) {
            double m = double(mx);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
            if ((threadIdx.x & 31) == 0)
                atomicMax(reinterpret_cast<unsigned long long*>(fmax_bits) + static_cast<size_t>(bg) * nframes + sp.frame,
                          static_cast<unsigned long long>(__double_as_longlong(m)));
        }
    }
}

// ---------------------------------------------------------------- warp-per-row rows (M = 128 .. 1024)
constexpr int TRW_WARPS = 8;

template <int M>
constexpr bool tr_warp_rows() {
    return M == 128 || M == 256 || M == 512 || M == 1024;
}

template <typename T, int M>
__global__ void __launch_bounds__(TRW_WARPS * 32, sizeof(T) == 8 ? 1 : 2)
tr_rows_fwd_w(int b0, int count, TRBuf<T> bf, TRStep sp, const cplx<T>* __restrict__ g_tw,
              const cplx<T>* __restrict__ g_hs) {
    using Gm = TRGeom<T, M>;
    using WF = WarpFFT<T, M>;
    constexpr int n = Gm::n, hp = Gm::hp, P = WF::P, E = n / 32;
    constexpr size_t nn = size_t(n) * n;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* s_tw = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_tw1 = s_tw + M;
    cplx<T>* s_hs = s_tw1 + WF::TW1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    cplx<T>* scr = s_hs + n + warp * WF::SCRATCH;
    for (int t = threadIdx.x; t < M; t += TRW_WARPS * 32) s_tw[t] = g_tw[t];
    for (int t = threadIdx.x; t < n; t += TRW_WARPS * 32) s_hs[t] = g_hs[t];
    WF::build_tw1(s_tw1, g_tw, threadIdx.x, TRW_WARPS * 32);
    __syncthreads();
    for (int item = blockIdx.x * TRW_WARPS + warp; item < count * n; item += gridDim.x * TRW_WARPS) {
        const int b = item / n, x = item - b * n;
        const T* ring = bf.ring + static_cast<size_t>(b0 + b) * bf.ring_stride + static_cast<size_t>(x) * n;
        const T* Pn = ring + sp.slot_n * nn;
        T pv[E], dv[E];
#pragma unroll
        for (int t = 0; t < E; ++t) {
            const int y = lane + 32 * t;
            pv[t] = Pn[y];
            dv[t] = T(0);
            if (sp.has_k) dv[t] = ring[sp.slot_k * nn + y] - (sp.slot_k1 >= 0 ? ring[sp.slot_k1 * nn + y] : T(0));
        }
        // z[i] = mirror(P_n row)[i] + i mirror(d row)[i], i = lane + 32 k; mirror by shuffle for k >= E
        cplx<T> z[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
            if (k < E)
                z[k] = mk<T>(pv[k], dv[k]);
            else
                z[k] = mk<T>(__shfl_xor_sync(0xffffffffu, pv[P - 1 - k], 31),
                             __shfl_xor_sync(0xffffffffu, dv[P - 1 - k], 31));
        }
        WF::template run<-1>(z, scr, s_tw, s_tw1, lane);
        __syncwarp();
#pragma unroll
        for (int m1 = 0; m1 < P; ++m1) scr[WF::out_pos(lane, m1)] = z[m1];
        __syncwarp();
        cplx<T>* Dx = bf.D + (static_cast<size_t>(b0 + b) * n + x) * hp;
        for (int v = lane; v < hp; v += 32) {
            cplx<T> o = mk<T>(T(0), T(0));
            if (v < n) {
                const cplx<T> Zv = scr[v];
                const cplx<T> Zc = cconj<T>(scr[(M - v) & (M - 1)]);
                o = mk<T>(dct_part<T>(Zv, Zc, s_hs[v]), dct_part_im<T>(Zv, Zc, s_hs[v]));
            }
            Dx[v] = o;
        }
        __syncwarp();
    }
}

template <typename T, int M>
__global__ void __launch_bounds__(TRW_WARPS * 32, sizeof(T) == 8 ? 1 : 2)
tr_rows_inv_w(int b0, int count, TRBuf<T> bf, TRStep sp, int nframes, int law, T beta, T* __restrict__ out,
              double* __restrict__ fmax_bits, const cplx<T>* __restrict__ g_tw) {
    using Gm = TRGeom<T, M>;
    using WF = WarpFFT<T, M>;
    constexpr int n = Gm::n, hp = Gm::hp, P = WF::P, E = n / 32, RP = n / 2;
    constexpr size_t nn = size_t(n) * n;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* s_tw = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_tw1 = s_tw + M;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    cplx<T>* scr = s_tw1 + WF::TW1 + warp * WF::SCRATCH;
    for (int t = threadIdx.x; t < M; t += TRW_WARPS * 32) s_tw[t] = g_tw[t];
    WF::build_tw1(s_tw1, g_tw, threadIdx.x, TRW_WARPS * 32);
    __syncthreads();
    constexpr T inv = T(1.0 / (double(M) * double(M)));
    for (int item = blockIdx.x * TRW_WARPS + warp; item < count * RP; item += gridDim.x * TRW_WARPS) {
        const int b = item / RP, x0 = 2 * (item - b * RP);
        const int bg = b0 + b;
        const cplx<T>* Y0 = bf.D + (static_cast<size_t>(bg) * n + x0) * hp;
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
        T* ring = bf.ring + static_cast<size_t>(bg) * bf.ring_stride;
        T* Pnext = sp.slot_next >= 0 ? ring + sp.slot_next * nn : nullptr;
        const int* blk = bf.blk + static_cast<size_t>(bg) * bf.blk_stride;
        const T* sch = bf.sched + (static_cast<size_t>(bg) * bf.steps + (sp.step < bf.steps ? sp.step : 0)) * bf.nblk;
        const T* L0 = bf.leak0 + static_cast<size_t>(bg) * bf.leak_stride;
        T* O = sp.frame >= 0 ? out + (static_cast<size_t>(bg) * nframes + sp.frame) * nn : nullptr;
        T mx = T(0);
        // next power rows: the block ids and leakage of both rows are requested together,
        // then the schedule gathers -- two exposed round trips per row pair instead of a
        // dependent blk -> sched chain per element (the pass was 84% long-scoreboard stalls)
        int bk[2][E];
        T lv[2][E], sv[2][E];
        if (Pnext) {
#pragma unroll
            for (int half = 0; half < 2; ++half)
#pragma unroll
                for (int t = 0; t < E; ++t) {
                    const size_t o = static_cast<size_t>(x0 + half) * n + lane + 32 * t;
                    bk[half][t] = blk[o];
                    lv[half][t] = L0[o];
                }
#pragma unroll
            for (int half = 0; half < 2; ++half)
#pragma unroll
                for (int t = 0; t < E; ++t) sv[half][t] = sch[bk[half][t]];
        }
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const size_t rowo = static_cast<size_t>(x0 + half) * n;
#pragma unroll
            for (int t = 0; t < E; ++t) {
                const int j = lane + 32 * t;
                const cplx<T> zz = scr[j];
                T tv = (half ? zz.y : zz.x) * inv;
                tv = tv > T(0) ? tv : T(0);  // clamp_negatives (solver.cpp:33-46)
                if (O) O[rowo + j] = tv;
                mx = mx > tv ? mx : tv;
                if (Pnext) {
                    const T f = law ? T(exp(beta * tv)) : T(1) + beta * tv;
                    Pnext[rowo + j] = sv[half][t] + lv[half][t] * f;
                }
            }
        }
        if (O && fmax_bits) {
            double m = double(mx);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
            if (lane == 0)
                atomicMax(reinterpret_cast<unsigned long long*>(fmax_bits) + static_cast<size_t>(bg) * nframes + sp.frame,
                          static_cast<unsigned long long>(__double_as_longlong(m)));
        }
        __syncwarp();
    }
}

// P_1 = P_dyn,1 + L0 (T_0 = 0); Z = 0
template <typename T>
__global__ void tr_init(int b0, int count, TRBuf<T> bf, int nn, size_t zcount) {
    const size_t total = static_cast<size_t>(count) * nn;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
        const int b = static_cast<int>(i / nn);
        const size_t o = i - static_cast<size_t>(b) * nn;
        const int bg = b0 + b;
        const int* blk = bf.blk + static_cast<size_t>(bg) * bf.blk_stride;
        const T* sch = bf.sched + static_cast<size_t>(bg) * bf.steps * bf.nblk;
        const T* L0 = bf.leak0 + static_cast<size_t>(bg) * bf.leak_stride;
        bf.ring[static_cast<size_t>(bg) * bf.ring_stride + 1 * size_t(nn) + o] = sch[blk[o]] + L0[o];
    }
    const size_t zt = static_cast<size_t>(count) * zcount;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < zt; i += size_t(gridDim.x) * blockDim.x)
        bf.Z[static_cast<size_t>(b0) * zcount + i] = mk<T>(T(0), T(0));
}

// {(1 - r) F, r, r^{k+1} F} on the half-width pitch from the fp64 full spectra.
template <typename T>
__global__ void tr_tables(const double2* __restrict__ F, const double2* __restrict__ r,
                          const double2* __restrict__ rk, int m, int h, int hp, cplx<T>* __restrict__ tab) {
    const int u = blockIdx.y, v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= hp) return;
    const size_t o = static_cast<size_t>(u) * hp + v, plane = static_cast<size_t>(m) * hp;
    double2 a = make_double2(0.0, 0.0), rr = a, b = a;
    if (v < h) {
        const size_t f = static_cast<size_t>(u) * m + v;
        const double2 Fv = F[f], rv = r[f], kv = rk[f];
        a = make_double2((1.0 - rv.x) * Fv.x + rv.y * Fv.y, (1.0 - rv.x) * Fv.y - rv.y * Fv.x);
        rr = rv;
        b = make_double2(kv.x * Fv.x - kv.y * Fv.y, kv.x * Fv.y + kv.y * Fv.x);
    }
    tab[o] = mk<T>(T(a.x), T(a.y));
    tab[plane + o] = mk<T>(T(rr.x), T(rr.y));
    tab[2 * plane + o] = mk<T>(T(b.x), T(b.y));
}

template <typename T, int M>
struct TRLaunch {
    using Gm = TRGeom<T, M>;
    static size_t smem_rf() { return sizeof(cplx<T>) * (M * Gm::LP + M + Gm::n); }
    static size_t smem_ri() { return sizeof(cplx<T>) * (M * Gm::LP + M); }
    static size_t smem_w(bool fwd) {
        if constexpr (tr_warp_rows<M>())
            return sizeof(cplx<T>) * (M + WarpFFT<T, M>::TW1 + (fwd ? Gm::n : 0) +
                                      TRW_WARPS * WarpFFT<T, M>::SCRATCH);
        else
            return 0;
    }
    static size_t smem_c() {
        return sizeof(cplx<T>) * (Gm::TILEC + StageTw<M, false>::SIZE + StageTw<M, true>::SIZE + M);
    }
    static int run(const gtd_greens* g, const void* tabv, const gtd_trace_in* ti, int batch, const gtd_trace_opts* o,
                   void* t_out, double* max_out, void* scratch, int chunk, cudaStream_t st, long long* launches) {
        constexpr int n = Gm::n, hp = Gm::hp;
        static int res[3] = {0, 0, 0}, sms = 0;
        static DeviceOnce once_;
        once_([&] {
            cudaFuncSetAttribute(tr_rows_fwd<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_rf()));
            cudaFuncSetAttribute(tr_rows_inv<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_ri()));
            cudaFuncSetAttribute(tr_cols<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_c()));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[0], tr_rows_fwd<T, M>, Gm::NT, smem_rf());
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[1], tr_cols<T, M>, Gm::NTC, smem_c());
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[2], tr_rows_inv<T, M>, Gm::NT, smem_ri());
            if constexpr (tr_warp_rows<M>()) {
                cudaFuncSetAttribute(tr_rows_fwd_w<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_w(true)));
                cudaFuncSetAttribute(tr_rows_inv_w<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smem_w(false)));
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[0], tr_rows_fwd_w<T, M>, TRW_WARPS * 32,
                                                              smem_w(true));
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[2], tr_rows_inv_w<T, M>, TRW_WARPS * 32,
                                                              smem_w(false));
            }
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            for (int& r : res) r = r < 1 ? 1 : r;
        });
        const int k = o->window, steps = ti->steps, os = o->out_stride;
        const int nframes = steps / os;
        const size_t nn = size_t(n) * n;
        TRBuf<T> bf;
        bf.ring_stride = static_cast<size_t>(k + 2) * nn;
        bf.ring = static_cast<T*>(scratch);
        cplx<T>* rest = reinterpret_cast<cplx<T>*>(bf.ring + bf.ring_stride * chunk);
        bf.D = rest;
        bf.Z = rest + static_cast<size_t>(chunk) * n * hp;
        bf.blk = ti->blk;
        bf.blk_stride = ti->blk_stride;
        bf.sched = static_cast<const T*>(ti->sched);
        bf.nblk = ti->nblk;
        bf.steps = steps;
        bf.leak0 = static_cast<const T*>(ti->leak0);
        bf.leak_stride = ti->leak_stride;
        // per-chunk views: the buffers are indexed by (trace - b0) -> shift the bases
        const cplx<T>* tw = static_cast<const cplx<T>*>(g->tw);
        const cplx<T>* hs = static_cast<const cplx<T>*>(g->hs);
        const cplx<T>* tab = static_cast<const cplx<T>*>(tabv);
        auto grid = [&](int items, int r) { return items < sms * r ? items : sms * r; };
        long long kc = 0;
        if (max_out) cudaMemsetAsync(max_out, 0, sizeof(double) * size_t(batch) * nframes, st);
        for (int b0 = 0; b0 < batch; b0 += chunk) {
            const int cnt = batch - b0 < chunk ? batch - b0 : chunk;
            TRBuf<T> cb = bf;  // chunk-local scratch, global inputs / outputs
            cb.ring = bf.ring - static_cast<size_t>(b0) * bf.ring_stride;
            cb.D = bf.D - static_cast<size_t>(b0) * n * hp;
            cb.Z = bf.Z - static_cast<size_t>(b0) * M * hp;
            tr_init<T><<<sms * 4, 256, 0, st>>>(b0, cnt, cb, int(nn), size_t(M) * hp);
            kc += 1;
            for (int s = 1; s <= steps; ++s) {
                TRStep sp;
                sp.step = s;
                sp.slot_n = s % (k + 2);
                sp.has_k = s > k;
                sp.slot_k = sp.has_k ? (s - k) % (k + 2) : 0;
                sp.slot_k1 = (sp.has_k && s - k - 1 >= 1) ? (s - k - 1) % (k + 2) : -1;
                sp.slot_next = s < steps ? (s + 1) % (k + 2) : -1;
                sp.frame = (s % os == 0) ? s / os - 1 : -1;
                if constexpr (tr_warp_rows<M>())
                    tr_rows_fwd_w<T, M><<<grid((cnt * n + TRW_WARPS - 1) / TRW_WARPS, res[0]), TRW_WARPS * 32,
                                          smem_w(true), st>>>(b0, cnt, cb, sp, tw, hs);
                else
                    tr_rows_fwd<T, M><<<grid(cnt * Gm::RB, res[0]), Gm::NT, smem_rf(), st>>>(b0, cnt, cb, sp, tw, hs);
                tr_cols<T, M><<<grid(cnt * Gm::CT, res[1]), Gm::NTC, smem_c(), st>>>(b0, cnt, cb, sp, tw, hs, tab);
                if constexpr (tr_warp_rows<M>())
                    tr_rows_inv_w<T, M><<<grid((cnt * n / 2 + TRW_WARPS - 1) / TRW_WARPS, res[2]), TRW_WARPS * 32,
                                          smem_w(false), st>>>(b0, cnt, cb, sp, nframes, o->law, T(o->beta),
                                                               static_cast<T*>(t_out), max_out, tw);
                else
                    tr_rows_inv<T, M><<<grid(cnt * Gm::RPB, res[2]), Gm::NT, smem_ri(), st>>>(
                        b0, cnt, cb, sp, nframes, o->law, T(o->beta), static_cast<T*>(t_out), max_out, tw);
                kc += 3;
            }
        }
        // max_out holds the bit patterns of non-negative doubles: already the values
        if (launches) *launches = kc;
        return static_cast<int>(cudaGetLastError());
    }
};

template <typename T>
int tr_hp(int m) {
    switch (m) {
        case 64: return TRGeom<T, 64>::hp;
        case 128: return TRGeom<T, 128>::hp;
        case 256: return TRGeom<T, 256>::hp;
        case 512: return TRGeom<T, 512>::hp;
        case 1024: return TRGeom<T, 1024>::hp;
        case 2048: return TRGeom<T, 2048>::hp;
        default: return -1;
    }
}

template <typename T>
int dispatch_tr(const gtd_greens* g, const void* tab, const gtd_trace_in* ti, int batch, const gtd_trace_opts* o,
                void* t_out, double* max_out, void* scratch, int chunk, cudaStream_t st, long long* launches) {
    switch (g->m) {
#define GT_TR_CASE(MM) \
    case MM: return TRLaunch<T, MM>::run(g, tab, ti, batch, o, t_out, max_out, scratch, chunk, st, launches);
        GT_TR_CASE(64)
        GT_TR_CASE(128)
        GT_TR_CASE(256)
        GT_TR_CASE(512)
        GT_TR_CASE(1024)
        GT_TR_CASE(2048)
#undef GT_TR_CASE
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}

}  // namespace
}  // namespace gtb

using namespace gtb;

extern "C" {

int gtd_trace_pitch(int n, int fp64) { return fp64 ? tr_hp<double>(2 * n) : tr_hp<float>(2 * n); }

size_t gtd_trace_bytes_per_trace(int n, int fp64, int window) {
    const int hp = gtd_trace_pitch(n, fp64);
    if (hp < 0) return 0;
    const size_t rb = fp64 ? 8 : 4, cb = 2 * rb, nn = size_t(n) * n;
    return size_t(window + 2) * nn * rb + size_t(n) * hp * cb + size_t(2 * n) * hp * cb;
}

size_t gtd_trace_table_bytes(int n, int fp64) {
    const int hp = gtd_trace_pitch(n, fp64);
    return hp < 0 ? 0 : size_t(3) * 2 * n * hp * (fp64 ? 16 : 8);
}

int gtd_trace_tables(const gtd_greens* g, const void* Fd, const void* r, const void* rk, void* tab, cudaStream_t st) {
    const int hp = gtd_trace_pitch(g->n, g->fp64);
    if (hp < 0) return static_cast<int>(cudaErrorInvalidValue);
    const dim3 grid((hp + 127) / 128, g->m);
    if (g->fp64)
        tr_tables<double><<<grid, 128, 0, st>>>(static_cast<const double2*>(Fd), static_cast<const double2*>(r),
                                                static_cast<const double2*>(rk), g->m, g->n + 1, hp,
                                                static_cast<double2*>(tab));
    else
        tr_tables<float><<<grid, 128, 0, st>>>(static_cast<const double2*>(Fd), static_cast<const double2*>(r),
                                               static_cast<const double2*>(rk), g->m, g->n + 1, hp,
                                               static_cast<float2*>(tab));
    return static_cast<int>(cudaGetLastError());
}

int gtd_trace_batch(const gtd_greens* g, const void* tab, const gtd_trace_in* in, int batch, const gtd_trace_opts* o,
                    void* t_out, double* max_out, void* scratch, int chunk, cudaStream_t st, long long* launches) {
    if (!g || !tab || !in || !o || batch < 1 || chunk < 1 || o->window < 1 || o->out_stride < 1 || in->steps < 1)
        return static_cast<int>(cudaErrorInvalidValue);
    return g->fp64 ? dispatch_tr<double>(g, tab, in, batch, o, t_out, max_out, scratch, chunk, st, launches)
                   : dispatch_tr<float>(g, tab, in, batch, o, t_out, max_out, scratch, chunk, st, launches);
}

}  // extern "C"
