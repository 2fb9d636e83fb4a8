// fixed_point.cu — north-star mode B: the leakage-temperature fixed point
// with the Kirchhoff transform, batched over samples, two fused passes per
// iteration.
//
// Per sample (oracle: oracle/restate.cpp ref_fixed_point_batch; loop
// structure and stop rule of the reference FDM outer loop, fdm.cpp:167-205):
//   theta_{k+1} - T0 = crop(IFFT(fk . FFT(mirror(P + L0 f(T_k)))))
//   L0 = nom_scale * N * V,  f(dT) = exp(beta dT) (law 1) or 1 + beta dT (law 0)
//   T_{k+1} = Kirchhoff inverse of theta for k = k_ref (T/T0)^-eta (kirchhoff=1)
//   stop when max|T_{k+1} - T_k| < tol after iteration 1; max_iters -> error.
//
// Kernels per iteration:
//   fp_cols : per half-spectrum column tile: mirror-expand the row spectra,
//             forward column FFT, multiply by fk, inverse column FFT, keep rows
//             [0, n) -- in place.
//   fp_rows : per block of die-row PAIRS (two real rows share one complex
//             line): inverse row FFT -> theta rows -> Kirchhoff inverse ->
//             residual vs T_k -> T_{k+1} written in place -> next leakage ->
//             forward row FFT of the mirrored applied rows -> row spectra.
//   fp_update: per-sample iteration count / convergence / failure state.
#include <cuda_runtime.h>

#include "fft_tile.cuh"
#include "gt_device.h"

namespace gtb {
namespace {

template <typename T, int M>
struct FPGeom {
    using G = TileGeom<T, M>;
    static constexpr int n = M / 2;
    static constexpr int h = n + 1;
    static constexpr int L = G::L;
    static constexpr int NT = G::NT;
    static constexpr int hp = ((h + L - 1) / L) * L;  // column tiles of L columns
    static constexpr int LP = L + 2;
    static constexpr int RP = n / 2;                   // die-row pairs
    static constexpr int RB = (RP + L - 1) / L;        // row-pair blocks per sample
    static constexpr int CT = hp / L;                  // column tiles per sample
};

struct FPState {
    unsigned long long res_bits;  // max |T_{k+1} - T_k| of the current iteration (double bits)
    int iters;
    int active;
};

template <typename T>
struct FPIn {
    const T* P;
    const T* N;
    const T* V;
    long long sP, sN, sV;
    T nom_scale;
};

__device__ __forceinline__ void or_flags_fp(int* dst, int flags) {
    const int w = __reduce_or_sync(0xffffffffu, flags);
    if ((threadIdx.x & 31) == 0 && w) atomicOr(dst, w);
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <typename T>
__device__ __forceinline__ bool finite_val(T v) {
    return isfinite(v);
}

// ----------------------------------------------------------------- rows
template <typename T, int M, bool FIRST>
__global__ void __launch_bounds__(TileGeom<T, M>::NT, TileGeom<T, M>::MINB)
fp_rows(FPIn<T> in, int sample0, int count, cplx<T>* __restrict__ A, T* __restrict__ Tst,
        FPState* __restrict__ state, int* __restrict__ status, const cplx<T>* __restrict__ g_tw, T beta,
        int law, int kirchhoff, T ka, T kb, T kexp, T t_ambient) {
    using Gm = FPGeom<T, M>;
    constexpr int n = Gm::n, h = Gm::h, L = Gm::L, LP = Gm::LP, NT = Gm::NT, hp = Gm::hp;
    constexpr int RB = Gm::RB;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    T* tileT = reinterpret_cast<T*>(tile);
    cplx<T>* s_tw = tile + M * LP;
    double* red = reinterpret_cast<double*>(s_tw + M);
    load_twiddles<T, M, NT>(s_tw, g_tw);
    __syncthreads();

    for (int item = blockIdx.x; item < count * RB; item += gridDim.x) {
        const int s = item / RB;
        const int p0 = (item - s * RB) * L;  // first row pair of the block
        const size_t sg = static_cast<size_t>(sample0) + s;
        if (!FIRST && !state[sg].active) continue;
        const T* P = in.P + sg * in.sP;
        const T* Nm = in.N + sg * in.sN;
        const T* V = in.V + sg * in.sV;
        T* Ts = Tst + sg * n * n;
        cplx<T>* As = A + static_cast<size_t>(s) * n * hp;
        constexpr T inv = T(1.0 / (double(M) * double(M)));
        double dmax = 0.0;
        int bad = 0;

        if (!FIRST) {
            // pack rows (2p, 2p+1) of the column-pass output into one Hermitian line pair
            for (int idx = threadIdx.x; idx < L * h; idx += NT) {
                const int l = idx / h, v = idx - l * h;
                const int xa = 2 * (p0 + l);
                cplx<T> y = mk<T>(T(0), T(0)), r = y;
                if (xa < n) {
                    y = As[static_cast<size_t>(xa) * hp + v];
                    r = As[static_cast<size_t>(xa + 1) * hp + v];
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
            // theta -> T_{k+1}; residual; write state; build next applied rows in place
            for (int idx = threadIdx.x; idx < 2 * L * n; idx += NT) {
                const int lr = idx / n, j = idx - lr * n;  // local row 0..2L-1
                const int l = lr >> 1, half = lr & 1;
                const int x = 2 * p0 + lr;
                if (x >= n) continue;
                const cplx<T> z = tile[j * LP + l];
                T th = (half ? z.y : z.x) * inv;  // theta - T0
                T t = th;
                if (kirchhoff) {
                    const T br = ka + kb * th;
                    if (!(br > T(0))) bad |= GTD_ST_KIRCHHOFF;
                    t = pow(br, kexp) - t_ambient;
                }
                if (!finite_val(t)) bad |= GTD_ST_NONFINITE;
                const T old = Ts[x * n + j];
                dmax = fmax(dmax, double(fabs(t - old)));
                Ts[x * n + j] = t;
            }
            __syncthreads();
        }
        // forward: z = mirror(applied row 2p) + i mirror(applied row 2p+1)
        for (int idx = threadIdx.x; idx < 2 * L * n; idx += NT) {
            const int lr = idx / n, y = idx - lr * n;
            const int l = lr >> 1, half = lr & 1;
            const int x = 2 * p0 + lr;
            T a = T(0);
            if (x < n) {
                const T dT = FIRST ? T(0) : Ts[x * n + y];
                const T p = P[x * n + y];
                const T lk = in.nom_scale * Nm[x * n + y] * V[x * n + y];
                const T f = law ? T(exp(beta * dT)) : T(1) + beta * dT;
                a = p + lk * f;
            }
            tileT[2 * (y * LP + l) + half] = a;
            tileT[2 * ((M - 1 - y) * LP + l) + half] = a;
        }
        __syncthreads();
        tile_fft<T, M, L, LP, NT, -1>(tile, s_tw);
        for (int idx = threadIdx.x; idx < 2 * L * hp; idx += NT) {
            const int lr = idx / hp, v = idx - lr * hp;
            const int l = lr >> 1, half = lr & 1;
            const int x = 2 * p0 + lr;
            if (x >= n) continue;
            cplx<T> o = mk<T>(T(0), T(0));
            if (v < h) {
                const cplx<T> Z = tile[v * LP + l];
                const cplx<T> Zc = cconj<T>(tile[((M - v) & (M - 1)) * LP + l]);
                if (!half)
                    o = mk<T>(T(0.5) * (Z.x + Zc.x), T(0.5) * (Z.y + Zc.y));
                else
                    o = mk<T>(T(0.5) * (Z.y - Zc.y), T(-0.5) * (Z.x - Zc.x));
            }
            As[static_cast<size_t>(x) * hp + v] = o;
        }
        if (!FIRST) {
            or_flags_fp(&status[sg], bad);
            dmax = warp_max_d(dmax);
            if ((threadIdx.x & 31) == 0) {
                // non-negative doubles order like their bit patterns
                atomicMax(&state[sg].res_bits, static_cast<unsigned long long>(__double_as_longlong(dmax)));
            }
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------------- columns
template <typename T, int M>
__global__ void __launch_bounds__(TileGeom<T, M>::NT, TileGeom<T, M>::MINB)
fp_cols(int sample0, int count, cplx<T>* __restrict__ A, const FPState* __restrict__ state,
        const cplx<T>* __restrict__ g_tw, const cplx<T>* __restrict__ fk, int fk_pitch) {
    using Gm = FPGeom<T, M>;
    constexpr int n = Gm::n, h = Gm::h, L = Gm::L, NT = Gm::NT, hp = Gm::hp, CT = Gm::CT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_tw = tile + M * L;
    load_twiddles<T, M, NT>(s_tw, g_tw);
    __syncthreads();
    for (int item = blockIdx.x; item < count * CT; item += gridDim.x) {
        const int s = item / CT;
        const int v0 = (item - s * CT) * L;
        const size_t sg = static_cast<size_t>(sample0) + s;
        if (!state[sg].active) continue;
        cplx<T>* As = A + static_cast<size_t>(s) * n * hp;
        for (int idx = threadIdx.x; idx < n * L; idx += NT) {
            const int w = idx % L, x = idx / L;
            const cplx<T> a = As[static_cast<size_t>(x) * hp + v0 + w];
            tile[x * L + w] = a;
            tile[(M - 1 - x) * L + w] = a;
        }
        __syncthreads();
        tile_fft<T, M, L, L, NT, -1>(tile, s_tw);
        for (int idx = threadIdx.x; idx < M * L; idx += NT) {
            const int w = idx % L, u = idx / L;
            const int v = v0 + w;
            if (v >= h) continue;
            tile[u * L + w] = cmul<T>(tile[u * L + w], fk[static_cast<size_t>(u) * fk_pitch + v]);
        }
        __syncthreads();
        tile_fft<T, M, L, L, NT, +1>(tile, s_tw);
        for (int idx = threadIdx.x; idx < n * L; idx += NT) {
            const int w = idx % L, x = idx / L;
            As[static_cast<size_t>(x) * hp + v0 + w] = tile[x * L + w];
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------------- state
__global__ void fp_init(FPState* st, int* status, int* iters, int sample0, int count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    st[sample0 + i] = FPState{0ull, 0, 1};
    status[sample0 + i] = 0;
    iters[sample0 + i] = 0;
}

// Reference stop rule (fdm.cpp:190-200): converge check first, then max_iters.
__global__ void fp_update(FPState* st, int* status, int* iters, int sample0, int count, double tol, int max_iters,
                          int* active_count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    FPState& s = st[sample0 + i];
    if (!s.active) return;
    s.iters += 1;
    iters[sample0 + i] = s.iters;
    const double res = __longlong_as_double(static_cast<long long>(s.res_bits));
    s.res_bits = 0ull;
    if (status[sample0 + i]) {
        s.active = 0;
    } else if (s.iters > 1 && res < tol) {
        s.active = 0;
    } else if (s.iters >= max_iters) {
        status[sample0 + i] |= GTD_ST_NOCONVERGE;
        s.active = 0;
    }
    if (s.active) atomicAdd(active_count, 1);
}

// per-sample max / mean of the converged maps
template <typename T>
__global__ void fp_stats(const T* __restrict__ Tst, int n, int sample0, double* __restrict__ mx,
                         double* __restrict__ mean) {
    const size_t sg = static_cast<size_t>(sample0) + blockIdx.x;
    const T* t = Tst + sg * n * n;
    double m = -1.0 / 0.0, s = 0.0;
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
        m = fmax(m, double(t[i]));
        s += double(t[i]);
    }
    __shared__ double rm[32], rs[32];
    for (int o = 16; o > 0; o >>= 1) {
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    if ((threadIdx.x & 31) == 0) {
        rm[threadIdx.x >> 5] = m;
        rs[threadIdx.x >> 5] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w) {
            m = fmax(m, rm[w]);
            s += rs[w];
        }
        if (mx) mx[sg] = m;
        if (mean) mean[sg] = s / (double(n) * double(n));
    }
}

template <typename T, int M>
struct FPLaunch {
    using Gm = FPGeom<T, M>;
    static size_t smem_rows() { return sizeof(cplx<T>) * (M * Gm::LP + M) + 64 * sizeof(double); }
    static size_t smem_cols() { return sizeof(cplx<T>) * (M * Gm::L + M); }

    static int run(const gtd_greens* g, const FPIn<T>& in, int batch, const gtd_fp_opts* o, T* Tst, int* iters,
                   int* status, double* mx, double* mean, void* scratch, FPState* state, int* counter_d,
                   int* counter_h, int chunk, cudaStream_t st, long long* launches) {
        constexpr int n = Gm::n, hp = Gm::hp, NT = Gm::NT;
        static int res[3] = {0, 0, 0}, sms = 0;
        if (!sms) {
            cudaFuncSetAttribute(fp_rows<T, M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_rows()));
            cudaFuncSetAttribute(fp_rows<T, M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_rows()));
            cudaFuncSetAttribute(fp_cols<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_cols()));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[0], fp_rows<T, M, false>, NT, smem_rows());
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[1], fp_cols<T, M>, NT, smem_cols());
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            for (int& r : res) r = r < 1 ? 1 : r;
        }
        cplx<T>* A = static_cast<cplx<T>*>(scratch);
        const cplx<T>* tw = static_cast<const cplx<T>*>(g->tw);
        const cplx<T>* fk = static_cast<const cplx<T>*>(g->fk);
        const T kexp = T(1.0 / (1.0 - o->eta));
        const T ka = T(pow(o->t_ambient, 1.0 - o->eta)), kb = T((1.0 - o->eta) * pow(o->t_ambient, -o->eta));
        auto grid = [&](int items, int r) { return items < sms * r ? items : sms * r; };
        const int poll = o->poll > 0 ? o->poll : 4;
        long long k = 0;
        for (int s0 = 0; s0 < batch; s0 += chunk) {
            const int cnt = batch - s0 < chunk ? batch - s0 : chunk;
            const int gr = grid(cnt * Gm::RB, res[0]), gc = grid(cnt * Gm::CT, res[1]);
            fp_init<<<(cnt + 127) / 128, 128, 0, st>>>(state, status, iters, s0, cnt);
            fp_rows<T, M, true><<<gr, NT, smem_rows(), st>>>(in, s0, cnt, A, Tst, state, status, tw, T(o->beta),
                                                             o->law, o->kirchhoff, ka, kb, kexp, T(o->t_ambient));
            k += 2;
            for (int it = 1; it <= o->max_iters; ++it) {
                fp_cols<T, M><<<gc, NT, smem_cols(), st>>>(s0, cnt, A, state, tw, fk, g->hp);
                fp_rows<T, M, false><<<gr, NT, smem_rows(), st>>>(in, s0, cnt, A, Tst, state, status, tw,
                                                                  T(o->beta), o->law, o->kirchhoff, ka, kb, kexp,
                                                                  T(o->t_ambient));
                cudaMemsetAsync(counter_d, 0, sizeof(int), st);
                fp_update<<<(cnt + 127) / 128, 128, 0, st>>>(state, status, iters, s0, cnt, o->tol, o->max_iters,
                                                            counter_d);
                k += 3;
                if (it % poll == 0 || it == o->max_iters) {
                    cudaMemcpyAsync(counter_h, counter_d, sizeof(int), cudaMemcpyDeviceToHost, st);
                    cudaStreamSynchronize(st);
                    if (*counter_h == 0) break;
                }
            }
            fp_stats<T><<<cnt, 256, 0, st>>>(Tst, n, s0, mx, mean);
            k += 1;
        }
        if (launches) *launches = k;
        return static_cast<int>(cudaGetLastError());
    }
};

template <typename T>
int dispatch_fp(const gtd_greens* g, const gtd_mc_in* i, int batch, const gtd_fp_opts* o, void* Tst, int* iters,
                int* status, double* mx, double* mean, void* scratch, void* state, int* counter_d, int* counter_h,
                int chunk, cudaStream_t st, long long* launches) {
    FPIn<T> in{static_cast<const T*>(i->P), static_cast<const T*>(i->N), static_cast<const T*>(i->V),
               i->sP, i->sN, i->sV, T(i->nom_scale)};
    T* t = static_cast<T*>(Tst);
    FPState* s = static_cast<FPState*>(state);
    switch (g->m) {
#define GT_FP_CASE(MM) \
    case MM: return FPLaunch<T, MM>::run(g, in, batch, o, t, iters, status, mx, mean, scratch, s, counter_d, counter_h, chunk, st, launches);
        GT_FP_CASE(32)
        GT_FP_CASE(64)
        GT_FP_CASE(128)
        GT_FP_CASE(256)
        GT_FP_CASE(512)
        GT_FP_CASE(1024)
        GT_FP_CASE(2048)
#undef GT_FP_CASE
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}

template <typename T>
int fp_hp(int m) {
    switch (m) {
        case 32: return FPGeom<T, 32>::hp;
        case 64: return FPGeom<T, 64>::hp;
        case 128: return FPGeom<T, 128>::hp;
        case 256: return FPGeom<T, 256>::hp;
        case 512: return FPGeom<T, 512>::hp;
        case 1024: return FPGeom<T, 1024>::hp;
        case 2048: return FPGeom<T, 2048>::hp;
        default: return -1;
    }
}

}  // namespace
}  // namespace gtb

using namespace gtb;

extern "C" {

size_t gtd_fp_scratch_bytes_per_sample(int n, int fp64) {
    const int hp = fp64 ? fp_hp<double>(2 * n) : fp_hp<float>(2 * n);
    if (hp < 0) return 0;
    return static_cast<size_t>(n) * hp * (fp64 ? 16 : 8);
}

size_t gtd_fp_state_bytes(void) { return sizeof(FPState); }

int gtd_fp_batch(const gtd_greens* g, const gtd_mc_in* in, int batch, const gtd_fp_opts* opts, void* t_state,
                 int* iters, int* status, double* max_out, double* mean_out, void* scratch, void* state,
                 int* counter_d, int* counter_h, int chunk, cudaStream_t stream, long long* launches) {
    if (!g || !in || !opts || batch < 1 || chunk < 1 || !t_state) return static_cast<int>(cudaErrorInvalidValue);
    return g->fp64 ? dispatch_fp<double>(g, in, batch, opts, t_state, iters, status, max_out, mean_out, scratch, state,
                                         counter_d, counter_h, chunk, stream, launches)
                   : dispatch_fp<float>(g, in, batch, opts, t_state, iters, status, max_out, mean_out, scratch, state,
                                        counter_d, counter_h, chunk, stream, launches);
}

}  // extern "C"
