// vargen.cu — seeded variation maps on the device: the
// config-1 variation model var = 1 + (sigma/mu) z, z a unit-variance Gaussian
// random field with the reference's spherical correlogram (variation.cpp:75-79)
// by circulant embedding on the m = 2n torus (the construction of
// gen_systematic_map, variation.cpp:87-132).
//
// The reference draws white noise in space and transforms it forward; the
// spectrum of real white noise is itself white Hermitian complex noise, so the
// generator draws it directly in the frequency domain (counter-based Philox,
// one draw per (sample, u, v), independent of batch layout) and runs only the
// inverse transform: a column pass over the n+1 half-spectrum columns (rows
// [0, n) kept) and a warp-per-row-pair C2R pass (columns [0, n) kept).
// Same distribution as the reference generator, not the same samples: the
// reference's libstdc++ normal_distribution stream is reproduced bit-exactly
// only on the host path (gt_monte_carlo).
#include <cuda_runtime.h>

#include <cstdint>

#include "launch_once.cuh"
#include "fft_tile.cuh"
#include "fft_warp.cuh"
#include "gt_device.h"

namespace gtb {
namespace {

// Philox4x32-10 (Salmon et al. 2011): counter (c0..c3), key (k0, k1).
__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const unsigned lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const unsigned lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

// Two standard normals from two uniforms (Box-Muller), double-precision math.
__device__ __forceinline__ double2 normals(unsigned a, unsigned b) {
    const double u1 = (double(a) + 0.5) * (1.0 / 4294967296.0), u2 = (double(b) + 0.5) * (1.0 / 4294967296.0);
    const double r = sqrt(-2.0 * log(u1));
    double s, c;
    sincospi(2.0 * u2, &s, &c);
    return make_double2(r * c, r * s);
}

// White Hermitian spectrum of real white noise on the m-torus, scaled so that
// E|W(u,v)|^2 = m^2 (the forward DFT of unit-variance noise), at half-spectrum
// column v <= m/2. Columns 0 and m/2 are Hermitian in u; (0,0), (m/2,0),
// (0,m/2), (m/2,m/2) are real.
template <typename T>
__device__ __forceinline__ cplx<T> white(unsigned long long seed, int m, int u, int v) {
    const int n = m / 2;
    const bool herm = (v == 0 || v == n);
    const int ur = herm && u > n ? m - u : u;
    const uint4 r = philox(make_uint4(unsigned(ur), unsigned(v), 0x5641u, 0u),
                           make_uint2(unsigned(seed), unsigned(seed >> 32)));
    const double2 z = normals(r.x, r.y);
    const double sc = double(m) * 0.70710678118654752440;
    if (herm && (ur == 0 || ur == n)) return mk<T>(T(z.x * double(m)), T(0));
    const double im = herm && u > n ? -z.y : z.y;
    return mk<T>(T(z.x * sc), T(im * sc));
}

// ---- column pass: per (sample, tile of L half-spectrum columns), inverse FFT over u
template <typename T, int M>
__global__ void __launch_bounds__(TileGeom<T, M>::NT, TileGeom<T, M>::MINB)
vg_cols(const unsigned long long* __restrict__ seeds, int s0, int count, const T* __restrict__ sqlam,
        cplx<T>* __restrict__ G, int hp, const cplx<T>* __restrict__ g_tw) {
    using TG = TileGeom<T, M>;
    constexpr int n = M / 2, h = n + 1, L = TG::L, NT = TG::NT;
    constexpr int CT = (h + L - 1) / L;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_tw = tile + M * L;
    load_twiddles<T, M, NT>(s_tw, g_tw);
    for (int item = blockIdx.x; item < count * CT; item += gridDim.x) {
        const int s = item / CT, v0 = (item - s * CT) * L;
        const unsigned long long seed = seeds[s0 + s];
        __syncthreads();
        for (int idx = threadIdx.x; idx < M * L; idx += NT) {
            const int l = idx % L, u = idx / L, v = v0 + l;
            cplx<T> w = mk<T>(T(0), T(0));
            if (v < h) w = cscale<T>(white<T>(seed, M, u, v), sqlam[static_cast<size_t>(u) * hp + v]);
            tile[u * L + l] = w;
        }
        __syncthreads();
        tile_fft<T, M, L, L, NT, +1>(tile, s_tw);
        cplx<T>* Gs = G + static_cast<size_t>(s) * n * hp;
        for (int idx = threadIdx.x; idx < n * L; idx += NT) {
            const int l = idx % L, x = idx / L, v = v0 + l;
            if (v < hp) Gs[static_cast<size_t>(x) * hp + v] = tile[x * L + l];
        }
    }
}

// ---- row pass: warp per die-row pair, C2R of the half spectra, var = 1 + sigma z
constexpr int VGW_WARPS = 8;

template <typename T, int M>
__global__ void __launch_bounds__(VGW_WARPS * 32, sizeof(T) == 8 ? 1 : 2)
vg_rows(int count, const cplx<T>* __restrict__ G, int hp, T sigma, T* __restrict__ var, long long vstride,
        const cplx<T>* __restrict__ g_tw) {
    using WF = WarpFFT<T, M>;
    constexpr int n = M / 2, P = WF::P, E = n / 32, RP = n / 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* s_tw = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_tw1 = s_tw + M;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    cplx<T>* scr = s_tw1 + WF::TW1 + warp * WF::SCRATCH;
    for (int t = threadIdx.x; t < M; t += VGW_WARPS * 32) s_tw[t] = g_tw[t];
    WF::build_tw1(s_tw1, g_tw, threadIdx.x, VGW_WARPS * 32);
    __syncthreads();
    const T scale = sigma * T(1.0 / (double(M) * double(M)));
    for (int item = blockIdx.x * VGW_WARPS + warp; item < count * RP; item += gridDim.x * VGW_WARPS) {
        const int s = item / RP, x0 = 2 * (item - s * RP);
        const cplx<T>* Y0 = G + (static_cast<size_t>(s) * n + x0) * hp;
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
        T* V0 = var + static_cast<size_t>(s) * vstride + static_cast<size_t>(x0) * n;
#pragma unroll
        for (int t = 0; t < E; ++t) {
            const int j = lane + 32 * t;
            const cplx<T> q = scr[j];
            V0[j] = T(1) + scale * q.x;
            V0[n + j] = T(1) + scale * q.y;
        }
        __syncwarp();
    }
}

// ---- sqrt(lambda): spherical correlogram on the m-torus -> FFT -> clamp -> normalise
__global__ void k_cov(int m, double pitch, double range, double2* __restrict__ out) {
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const double di = double(i < m - i ? i : m - i) * pitch, dj = double(j < m - j ? j : m - j) * pitch;
    const double d = sqrt(di * di + dj * dj), x = d / range;
    out[static_cast<size_t>(i) * m + j] = make_double2(d < range ? 1.0 - 1.5 * x + 0.5 * x * x * x : 0.0, 0.0);
}

__global__ void k_lambda(const double2* __restrict__ F, size_t count, double* __restrict__ lam) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x)
        lam[i] = F[i].x > 0.0 ? F[i].x : 0.0;
}

template <typename T>
__global__ void k_sqlam(const double* __restrict__ lam, int m, int h, int hp, const double* __restrict__ sum3,
                        T* __restrict__ out) {
    const int u = blockIdx.y, v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= hp) return;
    const double norm = double(m) * double(m) / sum3[0];
    out[static_cast<size_t>(u) * hp + v] = v < h ? T(sqrt(lam[static_cast<size_t>(u) * m + v] * norm)) : T(0);
}

template <typename T, int M>
struct VGLaunch {
    static size_t smem_c() { return sizeof(cplx<T>) * (M * TileGeom<T, M>::L + M); }
    static size_t smem_r() { return sizeof(cplx<T>) * (M + WarpFFT<T, M>::TW1 + VGW_WARPS * WarpFFT<T, M>::SCRATCH); }
    static int run(const gtd_greens* g, const void* sqlam, int hp, const unsigned long long* seeds, int batch,
                   double sigma, void* var, long long vstride, void* scratch, int chunk, cudaStream_t st) {
        static int res[2] = {0, 0}, sms = 0;
        static DeviceOnce once_;
        once_([&] {
            cudaFuncSetAttribute(vg_cols<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_c()));
            cudaFuncSetAttribute(vg_rows<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_r()));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[0], vg_cols<T, M>, TileGeom<T, M>::NT, smem_c());
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res[1], vg_rows<T, M>, VGW_WARPS * 32, smem_r());
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            for (int& r : res) r = r < 1 ? 1 : r;
        });
        constexpr int n = M / 2, L = TileGeom<T, M>::L, CT = (n + 1 + L - 1) / L;
        auto grid = [&](int items, int r) { return items < sms * r ? items : sms * r; };
        const cplx<T>* tw = static_cast<const cplx<T>*>(g->tw);
        cplx<T>* G = static_cast<cplx<T>*>(scratch);
        for (int s0 = 0; s0 < batch; s0 += chunk) {
            const int cnt = batch - s0 < chunk ? batch - s0 : chunk;
            vg_cols<T, M><<<grid(cnt * CT, res[0]), TileGeom<T, M>::NT, smem_c(), st>>>(
                seeds, s0, cnt, static_cast<const T*>(sqlam), G, hp, tw);
            vg_rows<T, M><<<grid((cnt * n / 2 + VGW_WARPS - 1) / VGW_WARPS, res[1]), VGW_WARPS * 32, smem_r(), st>>>(
                cnt, G, hp, T(sigma), static_cast<T*>(var) + static_cast<size_t>(s0) * vstride, vstride, tw);
        }
        return static_cast<int>(cudaGetLastError());
    }
};

}  // namespace
}  // namespace gtb

using namespace gtb;

extern "C" {

int gtd_var_pitch(int n) { return ((n + 1 + 31) / 32) * 32; }

size_t gtd_var_scratch_bytes_per_sample(int n, int fp64) {
    return static_cast<size_t>(n) * gtd_var_pitch(n) * (fp64 ? 16 : 8);
}

int gtd_var_model(const gtd_greens* g, const void* tw64, double pitch, double range, void* work_d, double* lam_d,
                  double* red_d, void* sqlam_out, cudaStream_t st) {
    const int m = g->m, hp = gtd_var_pitch(g->n);
    k_cov<<<dim3((m + 127) / 128, m), 128, 0, st>>>(m, pitch, range, static_cast<double2*>(work_d));
    int e = gtd_fft2d(work_d, m, 1, -1, 1, tw64, st);
    if (e) return e;
    k_lambda<<<592, 256, 0, st>>>(static_cast<const double2*>(work_d), static_cast<size_t>(m) * m, lam_d);
    e = gtd_reduce(lam_d, static_cast<size_t>(m) * m, red_d, st);
    if (e) return e;
    if (g->fp64)
        k_sqlam<double><<<dim3((hp + 127) / 128, m), 128, 0, st>>>(lam_d, m, g->n + 1, hp, red_d,
                                                                   static_cast<double*>(sqlam_out));
    else
        k_sqlam<float><<<dim3((hp + 127) / 128, m), 128, 0, st>>>(lam_d, m, g->n + 1, hp, red_d,
                                                                  static_cast<float*>(sqlam_out));
    return static_cast<int>(cudaGetLastError());
}

int gtd_var_generate(const gtd_greens* g, const void* sqlam, const unsigned long long* seeds, int batch,
                     double sigma, void* var, void* scratch, int chunk, cudaStream_t st) {
    const int hp = gtd_var_pitch(g->n);
    const long long vs = static_cast<long long>(g->n) * g->n;
#define GT_VG(TT, MM) \
    case MM: return VGLaunch<TT, MM>::run(g, sqlam, hp, seeds, batch, sigma, var, vs, scratch, chunk, st);
    if (g->fp64) {
        switch (g->m) {
            GT_VG(double, 128)
            GT_VG(double, 256)
            GT_VG(double, 512)
            default: return static_cast<int>(cudaErrorInvalidValue);
        }
    }
    switch (g->m) {
        GT_VG(float, 128)
        GT_VG(float, 256)
        GT_VG(float, 512)
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
#undef GT_VG
}

}  // extern "C"
