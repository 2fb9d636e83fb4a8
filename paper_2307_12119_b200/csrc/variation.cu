// variation.cu — fp64 device kernels for the variation / leakage inputs
// (reference variation.cpp:87-222) and the closed-form maps of calibration
// (greens.cpp:186-251): circulant-embedding eigenvalues of the spherical
// correlogram, spectral shaping of host-drawn noise, the leakage exponent and
// its cap, centre_kernel / kernel_to_die layouts, the symmetric multiplier and
// the random_greens spectral algebra over full m x m spectra.
#include <cuda_runtime.h>

#include "gt_device.h"

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
    const double d = b.x * b.x + b.y * b.y;
    return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
__device__ __forceinline__ int mdist(int i, int m) { return i <= m - i ? i : m - i; }
__device__ __forceinline__ int clampi(int i, int n) { return i < 0 ? 0 : (i > n - 1 ? n - 1 : i); }

dim3 g2(int cols, int rows) { return dim3((cols + 127) / 128, rows); }

// cov on the m-torus: spherical correlogram of the torus distance (variation.cpp:75-79, 97-105)
__global__ void k_cov(int n, double pitch, double range, double2* __restrict__ K) {
    const int m = 2 * n, i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const double d = hypot(mdist(i, m) * pitch, mdist(j, m) * pitch);
    double r = 0.0;
    if (d < range) {
        const double x = d / range;
        r = 1.0 - 1.5 * x + 0.5 * x * x * x;
    }
    K[static_cast<size_t>(i) * m + j] = make_double2(r, 0.0);
}

__global__ void k_clamp_re(const double2* __restrict__ K, size_t count, double* __restrict__ lam) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x)
        lam[i] = K[i].x > 0.0 ? K[i].x : 0.0;
}

__global__ void k_sqrt_fix(double* __restrict__ lam, size_t count, const double* __restrict__ sum3, double want) {
    const double fix = want / sum3[0];
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x)
        lam[i] = sqrt(lam[i] * fix);
}

__global__ void k_real_to_c(const double* __restrict__ x, size_t count, double2* __restrict__ X) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x)
        X[i] = make_double2(x[i], 0.0);
}

__global__ void k_scale_c(double2* __restrict__ X, const double* __restrict__ s, size_t count) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x) {
        X[i].x *= s[i];
        X[i].y *= s[i];
    }
}

__global__ void k_crop_re(const double2* __restrict__ X, int n, double scale, double* __restrict__ out) {
    const int m = 2 * n, i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    out[i * n + j] = scale * X[static_cast<size_t>(i) * m + j].x;
}

__global__ void k_leak_exp(const double* __restrict__ nom, const double* __restrict__ dl, const double* __restrict__ dt,
                           double bl, double bt, double cap, size_t count, double* __restrict__ out, int* flag) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x) {
        const double e = bl * dl[i] + bt * dt[i];
        if (fabs(e) > cap) atomicOr(flag, 1);
        out[i] = (nom ? nom[i] : 1.0) * exp(e);
    }
}

__global__ void k_add(const double* __restrict__ a, const double* __restrict__ b, size_t count, double* __restrict__ o) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x)
        o[i] = a[i] + b[i];
}

__global__ void k_subs(const double* __restrict__ a, double s, size_t count, double* __restrict__ o) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x)
        o[i] = a[i] - s;
}

__global__ void k_center(const double* __restrict__ f, double phi, int n, double2* __restrict__ K) {
    const int m = 2 * n, c = n / 2;
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int x = (i + c) % m, y = (j + c) % m;
    double v = 0.0;
    if (x < n && y < n) v = f[x * n + y] - phi;
    K[static_cast<size_t>(i) * m + j] = make_double2(v, 0.0);
}

__global__ void k_k2die(const double2* __restrict__ K, int n, double scale, double* __restrict__ out) {
    const int m = 2 * n, c = n / 2;
    const int x = blockIdx.y, y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= n) return;
    const int i = (x - c + m) % m, j = (y - c + m) % m;
    out[x * n + y] = scale * K[static_cast<size_t>(i) * m + j].x;
}

__global__ void k_sym(const double* __restrict__ f, int n, double shift, double* __restrict__ tab) {
    const int du = blockIdx.y, dv = blockIdx.x * blockDim.x + threadIdx.x;
    if (dv > n) return;
    const int c = n / 2;
    const int ip = clampi(c + du, n), im = clampi(c - du, n), jp = clampi(c + dv, n), jm = clampi(c - dv, n);
    // sum of the four shifted samples (symmetric_multiplier applied to f + shift)
    const double s = (f[ip * n + jp] + shift) + (f[ip * n + jm] + shift) + (f[im * n + jp] + shift) +
                     (f[im * n + jm] + shift);
    tab[du * (n + 1) + dv] = 0.25 * s;
}

__global__ void k_rand_spec(const double2* __restrict__ Fd, const double2* __restrict__ fk,
                            const double* __restrict__ gtab, int hp, const double* __restrict__ qtab, int n,
                            double alpha, double beta, double mu, double2* __restrict__ Fp, int* flag) {
    const int m = 2 * n;
    const int u = blockIdx.y, v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= m) return;
    const size_t o = static_cast<size_t>(u) * m + v;
    const int du = mdist(u, m), dv = mdist(v, m);
    const double g = gtab[du * hp + dv], q = qtab[du * (n + 1) + dv];
    const double2 f = fk[o], p = Fp[o], F = Fd[o];
    const double fmu = (u == 0 && v == 0) ? mu : 0.0;
    const double2 num0 = make_double2(beta * f.x * q + alpha * p.x * g, beta * f.y * q + alpha * p.y * g);
    const double2 num = cmul(F, num0);
    const double2 den = make_double2(1.0 - alpha * (1.0 + fmu + p.x) * g - mu * beta * f.x - beta * f.x * q,
                                     -alpha * p.y * g - mu * beta * f.y - beta * f.y * q);
    if (sqrt(den.x * den.x + den.y * den.y) < 1e-6) atomicOr(flag, GTD_ST_RUNAWAY_RAND);
    Fp[o] = cdiv(num, den);
}

int last() { return static_cast<int>(cudaGetLastError()); }

}  // namespace

extern "C" {

int gtd_var_eigs(int n, double pitch, double range, int, const void* tw64, void* work, double* sqrt_lam, double* red3,
                 cudaStream_t st) {
    const int m = 2 * n;
    const size_t mm = static_cast<size_t>(m) * m;
    double2* K = static_cast<double2*>(work);
    k_cov<<<g2(m, m), 128, 0, st>>>(n, pitch, range, K);
    int e = gtd_fft2d(K, m, 1, -1, 1, tw64, st);
    if (e) return e;
    k_clamp_re<<<592, 256, 0, st>>>(K, mm, sqrt_lam);
    e = gtd_reduce(sqrt_lam, mm, red3, st);
    if (e) return e;
    k_sqrt_fix<<<592, 256, 0, st>>>(sqrt_lam, mm, red3, double(m) * double(m));
    return last();
}

int gtd_var_shape(const double* noise, const double* sqrt_lam, int n, double sigma, const void* tw64, void* work,
                  double* out, cudaStream_t st) {
    const int m = 2 * n;
    const size_t mm = static_cast<size_t>(m) * m;
    double2* X = static_cast<double2*>(work);
    k_real_to_c<<<592, 256, 0, st>>>(noise, mm, X);
    int e = gtd_fft2d(X, m, 1, -1, 1, tw64, st);
    if (e) return e;
    k_scale_c<<<592, 256, 0, st>>>(X, sqrt_lam, mm);
    e = gtd_fft2d(X, m, 1, +1, 1, tw64, st);
    if (e) return e;
    k_crop_re<<<g2(n, n), 128, 0, st>>>(X, n, sigma / (double(m) * double(m)), out);
    return last();
}

int gtd_leak_exp(const double* nominal, const double* dl, const double* dt, double bl, double bt, double cap, int n,
                 double* out, int* flag, cudaStream_t st) {
    k_leak_exp<<<592, 256, 0, st>>>(nominal, dl, dt, bl, bt, cap, static_cast<size_t>(n) * n, out, flag);
    return last();
}

int gtd_add_maps(const double* a, const double* b, size_t count, double* out, cudaStream_t st) {
    k_add<<<592, 256, 0, st>>>(a, b, count, out);
    return last();
}

int gtd_sub_scalar(const double* a, double s, size_t count, double* out, cudaStream_t st) {
    k_subs<<<592, 256, 0, st>>>(a, s, count, out);
    return last();
}

int gtd_center_kernel(const double* f, double phi, int n, void* K, cudaStream_t st) {
    k_center<<<g2(2 * n, 2 * n), 128, 0, st>>>(f, phi, n, static_cast<double2*>(K));
    return last();
}

int gtd_kernel_to_die(const void* K, int n, double scale, double* out, cudaStream_t st) {
    k_k2die<<<g2(n, n), 128, 0, st>>>(static_cast<const double2*>(K), n, scale, out);
    return last();
}

int gtd_sym_table(const double* f, int n, double shift, double* tab, cudaStream_t st) {
    k_sym<<<g2(n + 1, n + 1), 128, 0, st>>>(f, n, shift, tab);
    return last();
}

int gtd_rand_spectrum(const void* Fd, const void* fk, const double* gtab, int hp, const double* qtab, int n,
                      double alpha, double beta, double mu, void* Fp, int* flag, cudaStream_t st) {
    k_rand_spec<<<g2(2 * n, 2 * n), 128, 0, st>>>(static_cast<const double2*>(Fd), static_cast<const double2*>(fk),
                                                 gtab, hp, qtab, n, alpha, beta, mu, static_cast<double2*>(Fp), flag);
    return last();
}

}  // extern "C"
