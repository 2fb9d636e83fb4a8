// ops.cu — fp64 full-spectrum kernels behind the reference-API solves
// (gt_solve_steady / gt_solve_step / gt_solve_trace): mirror padding, the
// closed-form deterministic spectrum, transient per-mode factors, the D10
// per-mode recursion of the windowed superposition, crops and reductions.
// These paths keep the reference's full m x m complex layout (spectral.cpp,
// solver.cpp:123-287) so every intermediate has a reference counterpart; the
// batched Monte-Carlo hot path lives in mc_modeA.cu.
#include <cuda_runtime.h>

#include <cstdint>

#include "gt_device.h"

namespace {

constexpr int RED_T = 1024;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
    const double d = b.x * b.x + b.y * b.y;
    return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
// exp(-t / tau) for complex tau
__device__ __forceinline__ double2 cexp_neg_over(double t, double2 tau) {
    const double d = tau.x * tau.x + tau.y * tau.y;
    const double zr = -t * tau.x / d, zi = t * tau.y / d;  // -t/tau = -t conj(tau)/|tau|^2
    const double e = exp(zr);
    double s, c;
    sincos(zi, &s, &c);
    return make_double2(e * c, e * s);
}

__device__ __forceinline__ int gidx_du(int u, int m) { return u <= m - u ? u : m - u; }

// mirror_pad (spectral.cpp:105-114) of a - b, as complex with zero imaginary part.
__global__ void k_mirror_pad(const double* __restrict__ a, const double* __restrict__ b, int n,
                             double2* __restrict__ X) {
    const int m = 2 * n;
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int x = i < n ? i : m - 1 - i, y = j < n ? j : m - 1 - j;
    double v = a[x * n + y];
    if (b) v -= b[x * n + y];
    X[static_cast<size_t>(i) * m + j] = make_double2(v, 0.0);
}

// F_det = fk / (1 - alpha g (1 + F(mu)) - mu beta fk)  (greens.cpp:203-216)
__global__ void k_fdet(const double2* __restrict__ fk, const double* __restrict__ gtab, int n, int hp,
                       double alpha, double beta, double mu, double2* __restrict__ Fd, int* flag) {
    const int m = 2 * n;
    const int u = blockIdx.y, v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= m) return;
    const size_t o = static_cast<size_t>(u) * m + v;
    const double g = gtab[gidx_du(u, m) * hp + gidx_du(v, m)];
    const double2 f = fk[o];
    const double fmu = (u == 0 && v == 0) ? mu : 0.0;
    const double2 den = make_double2(1.0 - alpha * g * (1.0 + fmu) - mu * beta * f.x, -mu * beta * f.y);
    if (sqrt(den.x * den.x + den.y * den.y) < 1e-6) atomicOr(flag, GTD_ST_RUNAWAY_DET);
    Fd[o] = cdiv(f, den);
}

// tau = C fk + alpha C g F_det (solver.cpp:129-149). Writes, per mode,
// out0 = F_det (1 - exp(-t/tau)) (t > 0; F_det for spectrally empty modes),
// r = exp(-dt/tau) and rk = exp(-(k+1) dt/tau) (0 for empty modes) when
// requested. flag |= 1 when Re tau <= 0 at an energetic mode.
__global__ void k_transient(const double2* __restrict__ fk, const double* __restrict__ gtab,
                            const double2* __restrict__ Fd, int n, int hp, double alpha, double cap,
                            double fk_floor, double t, double2* __restrict__ out, double dt, int kwin,
                            double2* __restrict__ r, double2* __restrict__ rk, int* flag) {
    const int m = 2 * n;
    const int u = blockIdx.y, v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= m) return;
    const size_t o = static_cast<size_t>(u) * m + v;
    const double2 f = fk[o], F = Fd[o];
    const bool empty = sqrt(f.x * f.x + f.y * f.y) <= fk_floor;
    double2 tau = make_double2(0.0, 0.0);
    if (!empty) {
        const double g = gtab[gidx_du(u, m) * hp + gidx_du(v, m)];
        const double2 agF = make_double2(alpha * cap * g * F.x, alpha * cap * g * F.y);
        tau = make_double2(cap * f.x + agF.x, cap * f.y + agF.y);
        if (tau.x <= 0.0) atomicOr(flag, 1);
    }
    if (out) {
        if (t == 0.0) {
            out[o] = make_double2(0.0, 0.0);
        } else if (empty || tau.x <= 0.0) {
            out[o] = F;
        } else {
            const double2 e = cexp_neg_over(t, tau);
            out[o] = cmul(F, make_double2(1.0 - e.x, -e.y));
        }
    }
    if (r) {
        const bool ok = !empty && tau.x > 0.0;
        r[o] = ok ? cexp_neg_over(dt, tau) : make_double2(0.0, 0.0);
        rk[o] = ok ? cexp_neg_over(dt * double(kwin + 1), tau) : make_double2(0.0, 0.0);
    }
}

__global__ void k_spec_mul(double2* __restrict__ X, const double2* __restrict__ S, size_t count) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x)
        X[i] = cmul(X[i], S[i]);
}

// crop_real (solver.cpp:54-61) with the inverse transform's 1/m^2.
__global__ void k_crop(const double2* __restrict__ X, int n, double scale, double* __restrict__ out) {
    const int m = 2 * n;
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    out[i * n + j] = X[static_cast<size_t>(i) * m + j].x * scale;
}

// D10 recursion step: E = r (dlt + E) - rk dk; P += dlt; X = F (P - E).
__global__ void k_trace_step(const double2* __restrict__ dlt, const double2* __restrict__ dk,
                             const double2* __restrict__ r, const double2* __restrict__ rk,
                             const double2* __restrict__ F, double2* __restrict__ E, double2* __restrict__ Pacc,
                             double2* __restrict__ X, size_t count) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x) {
        const double2 d = dlt[i];
        double2 e = cmul(r[i], make_double2(d.x + E[i].x, d.y + E[i].y));
        if (dk) {
            const double2 q = cmul(rk[i], dk[i]);
            e.x -= q.x;
            e.y -= q.y;
        }
        E[i] = e;
        const double2 p = make_double2(Pacc[i].x + d.x, Pacc[i].y + d.y);
        Pacc[i] = p;
        X[i] = cmul(F[i], make_double2(p.x - e.x, p.y - e.y));
    }
}

// Re sum_modes F (1 - r^i) for i = 1..k, partial per block: part[block][i-1].
__global__ void k_sat_partial(const double2* __restrict__ F, const double2* __restrict__ r, size_t count, int k,
                              double* __restrict__ part) {
    extern __shared__ double acc[];  // k doubles
    for (int i = threadIdx.x; i < k; i += blockDim.x) acc[i] = 0.0;
    __syncthreads();
    for (size_t q = blockIdx.x * size_t(blockDim.x) + threadIdx.x; q < count; q += size_t(gridDim.x) * blockDim.x) {
        const double2 f = F[q], rr = r[q];
        double2 p = rr;  // r^i
        for (int i = 0; i < k; ++i) {
            const double2 fp = cmul(f, p);
            atomicAdd(&acc[i], f.x - fp.x);
            p = cmul(p, rr);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += blockDim.x) part[static_cast<size_t>(blockIdx.x) * k + i] = acc[i];
}

__global__ void k_sat_final(const double* __restrict__ part, int blocks, int k, double den, double* __restrict__ sat) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    double s = 0.0;
    for (int b = 0; b < blocks; ++b) s += part[static_cast<size_t>(b) * k + i];
    sat[i] = s / den;
}

// scale_n = sum_{i<=min(k,n)} sat_i (T_{n-i+1} - T_{n-i}) + [n>k] T_{n-k}  (solver.cpp:250-276)
__global__ void k_trace_scale(const double* __restrict__ totals, const double* __restrict__ sat, int steps, int k,
                              double* __restrict__ scale) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x + 1;  // 1-based step
    if (n > steps) return;
    const int kk = n < k ? n : k;
    double s = 0.0;
    for (int i = 1; i <= kk; ++i) {
        const int cur = n - i + 1, prev = n - i;  // 1-based frames; T_0 = 0
        s += sat[i - 1] * (totals[cur - 1] - (prev >= 1 ? totals[prev - 1] : 0.0));
    }
    if (n > k) s += totals[n - k - 1];
    scale[n - 1] = s;
}

// T[s][.] += a o b * scale[s]   (a o b = f_rand o p_var; scale per map)
__global__ void k_add_rand(double* __restrict__ T, const double* __restrict__ a, const double* __restrict__ b,
                           const double* __restrict__ scale, double scale_mul, size_t nn, int maps) {
    const size_t total = nn * maps;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
        const size_t s = i / nn, k = i - s * nn;
        T[i] += a[k] * b[k] * (scale[s] * scale_mul);
    }
}

// Block-wide reductions into out[]: sum (fp64), min, max, count(<0).
__global__ void k_reduce(const double* __restrict__ x, size_t count, double* __restrict__ out) {
    __shared__ double s_sum[32], s_min[32], s_max[32];
    double sum = 0.0, mn = 1.0 / 0.0, mx = -1.0 / 0.0;
    for (size_t i = threadIdx.x; i < count; i += blockDim.x) {
        const double v = x[i];
        sum += v;
        mn = fmin(mn, v);
        mx = fmax(mx, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_sum[w] = sum;
        s_min[w] = mn;
        s_max[w] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < int(blockDim.x >> 5); ++k) {
            sum += s_sum[k];
            mn = fmin(mn, s_min[k]);
            mx = fmax(mx, s_max[k]);
        }
        out[0] = sum;
        out[1] = mn;
        out[2] = mx;
    }
}

// Complex sum (Re, Im) and max modulus.
__global__ void k_creduce(const double2* __restrict__ x, size_t count, double* __restrict__ out) {
    __shared__ double s_re[32], s_im[32], s_mx[32];
    double re = 0.0, im = 0.0, mx = 0.0;
    for (size_t i = threadIdx.x; i < count; i += blockDim.x) {
        const double2 v = x[i];
        re += v.x;
        im += v.y;
        mx = fmax(mx, sqrt(v.x * v.x + v.y * v.y));
    }
    for (int o = 16; o > 0; o >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, o);
        im += __shfl_xor_sync(0xffffffffu, im, o);
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_re[w] = re;
        s_im[w] = im;
        s_mx[w] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < int(blockDim.x >> 5); ++k) {
            re += s_re[k];
            im += s_im[k];
            mx = fmax(mx, s_mx[k]);
        }
        out[0] = re;
        out[1] = im;
        out[2] = mx;
    }
}

// clamp_negatives (solver.cpp:33-46): x < 0 -> 0, count, and most negative value.
__global__ void k_clamp(double* __restrict__ x, size_t count, unsigned long long* __restrict__ neg) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x)
        if (x[i] < 0.0) {
            x[i] = 0.0;
            atomicAdd(neg, 1ull);
        }
}

dim3 grid2(int cols, int rows) { return dim3((cols + 127) / 128, rows); }

int last() { return static_cast<int>(cudaGetLastError()); }

}  // namespace

extern "C" {

int gtd_mirror_pad(const double* a, const double* b, int n, void* X, cudaStream_t st) {
    k_mirror_pad<<<grid2(2 * n, 2 * n), 128, 0, st>>>(a, b, n, static_cast<double2*>(X));
    return last();
}

int gtd_fdet_full(const void* fk, const double* gtab, int n, int hp, double alpha, double beta, double mu,
                  void* Fd, int* flag, cudaStream_t st) {
    k_fdet<<<grid2(2 * n, 2 * n), 128, 0, st>>>(static_cast<const double2*>(fk), gtab, n, hp, alpha, beta, mu,
                                                static_cast<double2*>(Fd), flag);
    return last();
}

int gtd_transient(const void* fk, const double* gtab, const void* Fd, int n, int hp, double alpha, double cap,
                  double fk_floor, double t, void* out, double dt, int kwin, void* r, void* rk, int* flag,
                  cudaStream_t st) {
    k_transient<<<grid2(2 * n, 2 * n), 128, 0, st>>>(
        static_cast<const double2*>(fk), gtab, static_cast<const double2*>(Fd), n, hp, alpha, cap, fk_floor, t,
        static_cast<double2*>(out), dt, kwin, static_cast<double2*>(r), static_cast<double2*>(rk), flag);
    return last();
}

int gtd_spec_mul(void* X, const void* S, size_t count, cudaStream_t st) {
    k_spec_mul<<<592, 256, 0, st>>>(static_cast<double2*>(X), static_cast<const double2*>(S), count);
    return last();
}

int gtd_crop(const void* X, int n, double scale, double* out, cudaStream_t st) {
    k_crop<<<grid2(n, n), 128, 0, st>>>(static_cast<const double2*>(X), n, scale, out);
    return last();
}

int gtd_trace_step(const void* dlt, const void* dk, const void* r, const void* rk, const void* F, void* E,
                   void* Pacc, void* X, size_t count, cudaStream_t st) {
    k_trace_step<<<592, 256, 0, st>>>(static_cast<const double2*>(dlt), static_cast<const double2*>(dk),
                                      static_cast<const double2*>(r), static_cast<const double2*>(rk),
                                      static_cast<const double2*>(F), static_cast<double2*>(E),
                                      static_cast<double2*>(Pacc), static_cast<double2*>(X), count);
    return last();
}

int gtd_saturation(const void* F, const void* r, size_t count, int k, double re_sum_F, double* part, int blocks,
                   double* sat, cudaStream_t st) {
    k_sat_partial<<<blocks, 256, sizeof(double) * k, st>>>(static_cast<const double2*>(F),
                                                          static_cast<const double2*>(r), count, k, part);
    k_sat_final<<<(k + 127) / 128, 128, 0, st>>>(part, blocks, k, re_sum_F, sat);
    return last();
}

int gtd_trace_scale(const double* totals, const double* sat, int steps, int k, double* scale, cudaStream_t st) {
    k_trace_scale<<<(steps + 127) / 128, 128, 0, st>>>(totals, sat, steps, k, scale);
    return last();
}

int gtd_add_rand(double* T, const double* a, const double* b, const double* scale, double scale_mul, size_t nn,
                 int maps, cudaStream_t st) {
    k_add_rand<<<592, 256, 0, st>>>(T, a, b, scale, scale_mul, nn, maps);
    return last();
}

int gtd_reduce(const double* x, size_t count, double* out3, cudaStream_t st) {
    k_reduce<<<1, RED_T, 0, st>>>(x, count, out3);
    return last();
}

int gtd_creduce(const void* x, size_t count, double* out3, cudaStream_t st) {
    k_creduce<<<1, RED_T, 0, st>>>(static_cast<const double2*>(x), count, out3);
    return last();
}

int gtd_clamp(double* x, size_t count, unsigned long long* neg, cudaStream_t st) {
    k_clamp<<<592, 256, 0, st>>>(x, count, neg);
    return last();
}

}  // extern "C"
