// fft2d.cu — generic batched 2-D complex FFT on m x m grids (row pass + column
// pass over the shared-memory tile engine) and the one-time GreensSet setup
// kernels: the baseline kernel spectrum fk (reference greens.cpp:194-201,
// spectral.cpp:126-148) and the alpha multiplier table g (greens.cpp:186-192,
// spectral.cpp:167-185). Setup runs in fp64 on the device; the hot path reads
// the resulting tables in its own precision.
#include <cuda_runtime.h>

#include "launch_once.cuh"
#include "fft_tile.cuh"
#include "gt_device.h"

namespace gtb {

// Row pass: X is [batch*M][M] complex, every row transformed in place.
template <typename T, int M, int SIGN>
__global__ void __launch_bounds__(TileGeom<T, M>::NT)
fft_rows(cplx<T>* __restrict__ X, const cplx<T>* __restrict__ g_tw, int rows) {
    using G = TileGeom<T, M>;
    constexpr int L = G::L, LP = L + 2, NT = G::NT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_tw = tile + M * LP;
    load_twiddles<T, M, NT>(s_tw, g_tw);
    const size_t r0 = static_cast<size_t>(blockIdx.x) * L;
    for (int idx = threadIdx.x; idx < L * M; idx += NT) {
        const int l = idx / M, j = idx - l * M;
        const size_t r = r0 + l;
        tile[j * LP + l] = r < static_cast<size_t>(rows) ? X[r * M + j] : mk<T>(T(0), T(0));
    }
    __syncthreads();
    tile_fft<T, M, L, LP, NT, SIGN>(tile, s_tw);
    for (int idx = threadIdx.x; idx < L * M; idx += NT) {
        const int l = idx / M, j = idx - l * M;
        const size_t r = r0 + l;
        if (r < static_cast<size_t>(rows)) X[r * M + j] = tile[j * LP + l];
    }
}

// Column pass: X is [batch][M][M]; tile = L adjacent columns of one grid.
template <typename T, int M, int SIGN>
__global__ void __launch_bounds__(TileGeom<T, M>::NT)
fft_cols(cplx<T>* __restrict__ X, const cplx<T>* __restrict__ g_tw) {
    using G = TileGeom<T, M>;
    constexpr int L = G::L, NT = G::NT;
    constexpr int LL = L < M ? L : M;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* tile = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* s_tw = tile + M * L;
    load_twiddles<T, M, NT>(s_tw, g_tw);
    const int c0 = blockIdx.x * LL;
    cplx<T>* G0 = X + static_cast<size_t>(blockIdx.y) * M * M;
    for (int idx = threadIdx.x; idx < L * M; idx += NT) {
        const int l = idx % L, u = idx / L;
        tile[u * L + l] = l < LL ? G0[static_cast<size_t>(u) * M + c0 + l] : mk<T>(T(0), T(0));
    }
    __syncthreads();
    tile_fft<T, M, L, L, NT, SIGN>(tile, s_tw);
    for (int idx = threadIdx.x; idx < L * M; idx += NT) {
        const int l = idx % L, u = idx / L;
        if (l < LL) G0[static_cast<size_t>(u) * M + c0 + l] = tile[u * L + l];
    }
}

template <typename T, int M>
int run_fft2d(void* data, int batch, int sign, const void* tw, cudaStream_t st) {
    using G = TileGeom<T, M>;
    constexpr int L = G::L, NT = G::NT;
    constexpr int LL = L < M ? L : M;
    const size_t sm_r = sizeof(cplx<T>) * (M * (L + 2) + M);
    const size_t sm_c = sizeof(cplx<T>) * (M * L + M);
    static DeviceOnce once_;
    once_([&] {
        cudaFuncSetAttribute(fft_rows<T, M, -1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm_r));
        cudaFuncSetAttribute(fft_rows<T, M, +1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm_r));
        cudaFuncSetAttribute(fft_cols<T, M, -1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm_c));
        cudaFuncSetAttribute(fft_cols<T, M, +1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm_c));
    });
    cplx<T>* X = static_cast<cplx<T>*>(data);
    const cplx<T>* w = static_cast<const cplx<T>*>(tw);
    const int rows = batch * M;
    dim3 gr((rows + L - 1) / L), gc(M / LL, batch);
    if (sign < 0) {
        fft_rows<T, M, -1><<<gr, NT, sm_r, st>>>(X, w, rows);
        fft_cols<T, M, -1><<<gc, NT, sm_c, st>>>(X, w);
    } else {
        fft_rows<T, M, +1><<<gr, NT, sm_r, st>>>(X, w, rows);
        fft_cols<T, M, +1><<<gc, NT, sm_c, st>>>(X, w);
    }
    return static_cast<int>(cudaGetLastError());
}

template <typename T>
int dispatch_fft2d(void* data, int m, int batch, int sign, const void* tw, cudaStream_t st) {
    switch (m) {
        case 32: return run_fft2d<T, 32>(data, batch, sign, tw, st);
        case 64: return run_fft2d<T, 64>(data, batch, sign, tw, st);
        case 128: return run_fft2d<T, 128>(data, batch, sign, tw, st);
        case 256: return run_fft2d<T, 256>(data, batch, sign, tw, st);
        case 512: return run_fft2d<T, 512>(data, batch, sign, tw, st);
        case 1024: return run_fft2d<T, 1024>(data, batch, sign, tw, st);
        case 2048: return run_fft2d<T, 2048>(data, batch, sign, tw, st);
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}

// ------------------------------------------------------------- setup kernels
// K[(x-c) mod m][(y-c) mod m] = f(x,y) - phi, zero elsewhere (center_kernel).
__global__ void k_center_kernel(const double* __restrict__ f, double phi, int n,
                                double2* __restrict__ K) {
    const int m = 2 * n, c = n / 2;
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int x = (i + c) % m, y = (j + c) % m;  // inverse of (x - c) mod m
    double v = 0.0;
    if (x < n && y < n) v = f[x * n + y] - phi;
    K[static_cast<size_t>(i) * m + j] = make_double2(v, 0.0);
}

// fk[0] += phi m^2 / 4 (greens.cpp:199-200): the spreader constant counted once
// per die source across its four mirror images.
__global__ void k_dc_add(double2* K, double dc_add) { K[0].x += dc_add; }

// fk half spectrum (v < m/2+1) in the hot-path precision.
template <typename T>
__global__ void k_fk_half(const double2* __restrict__ K, int m, int hp,
                          cplx<T>* __restrict__ fk) {
    const int u = blockIdx.y, v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= hp) return;
    const int h = m / 2 + 1;
    double2 z = make_double2(0.0, 0.0);
    if (v < h) z = K[static_cast<size_t>(u) * m + v];
    fk[static_cast<size_t>(u) * hp + v] = mk<T>(T(z.x), T(z.y));
}

// g(du,dv) = g_sp0(c,c) - 1/4 sum_{+-,+-} g_sp0(clamp(c+-du), clamp(c+-dv)); row pitch hp.
template <typename T>
__global__ void k_gtab(const double* __restrict__ g_sp0, int n, int hp, T* __restrict__ gt) {
    const int du = blockIdx.y, dv = blockIdx.x * blockDim.x + threadIdx.x;
    if (dv > n) return;
    const int c = n / 2;
    auto cl = [n](int i) { return i < 0 ? 0 : (i > n - 1 ? n - 1 : i); };
    const int ip = cl(c + du), im = cl(c - du), jp = cl(c + dv), jm = cl(c - dv);
    const double s = g_sp0[ip * n + jp] + g_sp0[ip * n + jm] + g_sp0[im * n + jp] + g_sp0[im * n + jm];
    gt[du * hp + dv] = T(g_sp0[c * n + c] - 0.25 * s);
}

// Packed per-frequency table of the fused column pass (mc_pass2): one 16-byte
// (fp32) load per (u, v) of {fk.re, fk.im, alpha g(du, v), D(u) D(v)}, derived in
// fp64 and rounded once. D(u) = sin(pi u/2) / sin(pi u/m) is the real factor of
// the centred die-box spectrum (k1 (x) k1 = conj(w^{u/2} w^{v/2}) D(u) D(v)).
// Columns v > n are zero (they evaluate to 0 in the pass).
template <typename T>
__global__ void k_fg(const double2* __restrict__ K, const double* __restrict__ g_sp0, int n, int hp, double alpha,
                     T* __restrict__ fg) {
    const int m = 2 * n, u = blockIdx.y, v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= hp) return;
    T* o = fg + (static_cast<size_t>(u) * hp + v) * 4;
    if (v > n) {
        o[0] = o[1] = o[2] = o[3] = T(0);
        return;
    }
    const double2 z = K[static_cast<size_t>(u) * m + v];
    const int c = n / 2, du = u <= m - u ? u : m - u;
    auto cl = [n](int i) { return i < 0 ? 0 : (i > n - 1 ? n - 1 : i); };
    const int ip = cl(c + du), im = cl(c - du), jp = cl(c + v), jm = cl(c - v);
    const double s = g_sp0[ip * n + jp] + g_sp0[ip * n + jm] + g_sp0[im * n + jp] + g_sp0[im * n + jm];
    auto D = [n, m](int t) { return t == 0 ? double(n) : sinpi(0.5 * t) / sinpi(double(t) / m); };
    o[0] = T(z.x);
    o[1] = T(z.y);
    o[2] = T(alpha * (g_sp0[c * n + c] - 0.25 * s));
    o[3] = T(D(u) * D(v));
}

// Per-frequency table of the column pass at a FIXED mu (the reference's
// monte_carlo: deterministic_spectrum and random_greens both at gs.mu,
// solver.cpp:350-351,361): F_det = fk / den1 is then sample-invariant, so it
// is divided once here (fp64) instead of per pair. One 16-byte load per (u, v):
// {F_det.re, F_det.im, fk.re, fk.im}; den1 = 1 - alpha g - mu beta fk is rebuilt
// in the pass from the (L1-resident) alpha-multiplier table g(du, v). Padded
// columns (v > n) are zero. *flag gets 1 if |den1|^2 < 1e-12 anywhere
// (check_denominator, greens.cpp:32-39).
template <typename T>
__global__ void k_fgm(const double2* __restrict__ K, const double* __restrict__ g_sp0, int n, int hp, double alpha,
                      double mub, T* __restrict__ fg, int* __restrict__ flag) {
    const int m = 2 * n, u = blockIdx.y, v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= hp) return;
    T* o = fg + (static_cast<size_t>(u) * hp + v) * 4;
    if (v > n) {
        for (int k = 0; k < 4; ++k) o[k] = T(0);
        return;
    }
    const double2 z = K[static_cast<size_t>(u) * m + v];
    const int c = n / 2, du = u <= m - u ? u : m - u;
    auto cl = [n](int i) { return i < 0 ? 0 : (i > n - 1 ? n - 1 : i); };
    const int ip = cl(c + du), im = cl(c - du), jp = cl(c + v), jm = cl(c - v);
    const double s = g_sp0[ip * n + jp] + g_sp0[ip * n + jm] + g_sp0[im * n + jp] + g_sp0[im * n + jm];
    const double ag = alpha * (g_sp0[c * n + c] - 0.25 * s);
    const double d1x = 1.0 - ag - mub * z.x, d1y = -mub * z.y;
    const double dd = d1x * d1x + d1y * d1y;
    if (dd < 1e-12) atomicOr(flag, 1);
    o[0] = T((z.x * d1x + z.y * d1y) / dd);  // fk / den1
    o[1] = T((z.y * d1x - z.x * d1y) / dd);
    o[2] = T(z.x);
    o[3] = T(z.y);
}

}  // namespace gtb

using namespace gtb;

extern "C" {

int gtd_fft2d(void* data, int m, int batch, int sign, int fp64, const void* tw, cudaStream_t st) {
    return fp64 ? dispatch_fft2d<double>(data, m, batch, sign, tw, st)
                : dispatch_fft2d<float>(data, m, batch, sign, tw, st);
}

// Builds the device tables of a prepared GreensSet. f_sp0_d, g_sp0_d: device
// n x n fp64 maps; tw64_d: fp64 twiddles for m; work_d: m*m double2 that
// receives the full fp64 baseline kernel spectrum fk (kept by the caller).
int gtd_greens_tables(const double* f_sp0_d, const double* g_sp0_d, double phi, int n, int hp,
                      int fp64, const void* tw64_d, void* work_d, void* fk_out, void* gtab_out, void* fg_out,
                      double alpha, cudaStream_t st) {
    const int m = 2 * n;
    double2* K = static_cast<double2*>(work_d);
    k_center_kernel<<<dim3((m + 127) / 128, m), 128, 0, st>>>(f_sp0_d, phi, n, K);
    int e = dispatch_fft2d<double>(K, m, 1, -1, tw64_d, st);
    if (e) return e;
    const double dc_add = 0.25 * phi * double(m) * double(m);
    k_dc_add<<<1, 1, 0, st>>>(K, dc_add);
    if (fp64) {
        k_fk_half<double><<<dim3((hp + 127) / 128, m), 128, 0, st>>>(K, m, hp,
                                                                      static_cast<double2*>(fk_out));
        cudaMemsetAsync(gtab_out, 0, sizeof(double) * (n + 1) * hp, st);
        k_gtab<double><<<dim3((n + 1 + 127) / 128, n + 1), 128, 0, st>>>(g_sp0_d, n, hp,
                                                                          static_cast<double*>(gtab_out));
        if (fg_out)
            k_fg<double><<<dim3((hp + 127) / 128, m), 128, 0, st>>>(K, g_sp0_d, n, hp, alpha, static_cast<double*>(fg_out));
    } else {
        k_fk_half<float><<<dim3((hp + 127) / 128, m), 128, 0, st>>>(K, m, hp,
                                                                     static_cast<float2*>(fk_out));
        cudaMemsetAsync(gtab_out, 0, sizeof(float) * (n + 1) * hp, st);  // padded columns v > n read as 0
        k_gtab<float><<<dim3((n + 1 + 127) / 128, n + 1), 128, 0, st>>>(g_sp0_d, n, hp,
                                                                         static_cast<float*>(gtab_out));
        if (fg_out)
            k_fg<float><<<dim3((hp + 127) / 128, m), 128, 0, st>>>(K, g_sp0_d, n, hp, alpha, static_cast<float*>(fg_out));
    }
    return static_cast<int>(cudaGetLastError());
}

int gtd_greens_fgm(const void* work_d, const double* g_sp0_d, int n, int hp, int fp64, double alpha, double mub,
                   void* fgm_out, int* flag_d, cudaStream_t st) {
    const int m = 2 * n;
    const double2* K = static_cast<const double2*>(work_d);
    cudaMemsetAsync(flag_d, 0, sizeof(int), st);
    if (fp64)
        k_fgm<double><<<dim3((hp + 127) / 128, m), 128, 0, st>>>(K, g_sp0_d, n, hp, alpha, mub,
                                                                  static_cast<double*>(fgm_out), flag_d);
    else
        k_fgm<float><<<dim3((hp + 127) / 128, m), 128, 0, st>>>(K, g_sp0_d, n, hp, alpha, mub,
                                                                 static_cast<float*>(fgm_out), flag_d);
    return static_cast<int>(cudaGetLastError());
}

}  // extern "C"
