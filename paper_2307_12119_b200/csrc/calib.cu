// calib.cu — device GreensSet producer (north-star subsystem 1) and the
// fp64 full-spectrum pieces of calibration.
//
// Kernel producer. The reference measures f_sp0 as the FDM impulse response
// (greens.cpp:108-124 -> fdm.cpp:288-296): a 3-layer 7-point resistor network
// (fdm.cpp:45-110) with Neumann lateral edges, uniform vertical / sink terms.
// For a uniform die conductivity that operator is diagonalised by the 2-D
// DCT-II: each mode (p, q) with lateral eigenvalue
//   lam = (2 - 2 cos(pi p / n)) + (2 - 2 cos(pi q / n))
// decouples into one 3x3 layer system (die, TIM, spreader). The die response
// of mode (p, q) to a unit modal source is H = [M(lam)^-1]_00, and
//   f_sp0(x, y) = sum_pq H_pq a_p(x) a_q(y),  a_p(x) = w_p cos(pi p (c+1/2)/n) cos(pi p (x+1/2)/n)
// (w_0 = 1/n, w_p = 2/n): two n x n fp64 matrix products on the device. This is
// the exact discrete solution of the reference network (the continuum Hankel
// form matches it only to discretisation error); tests pin it against the
// reference FDM impulse response.
//
// The same modal systems give the backward-Euler transient impulse of
// fit_capacitance (fdm.cpp:257-286) exactly: per mode a 3-state recursion
// (M + C/dt) x_{k+1} = e0 + (C/dt) x_k.
#include <cuda_runtime.h>

#include "gt_device.h"

namespace {

struct Net {  // per-cell conductances of fdm.cpp:45-110 for a uniform die k
    double Gd, Gt, Gs;       // lateral
    double gdt, gts, gsink;  // vertical / sink
    double Cd, Ct, Cs;       // node capacitances (fdm.cpp:23-43)
};

__device__ __forceinline__ double cos_half(int p, int x, int n) {
    // cos(pi p (x + 1/2) / n) = cos(pi (p (2x+1) mod 4n) / (2n)), reduced exactly in integers
    const long long a = (static_cast<long long>(p) * (2 * x + 1)) % (4LL * n);
    return cospi(static_cast<double>(a) / (2.0 * n));
}

__device__ __forceinline__ double lam(int p, int n) { return 2.0 - 2.0 * cospi(static_cast<double>(p) / n); }

// H[p][q] = [M^-1]_00 for the 3x3 modal layer system.
__global__ void k_modal_H(Net net, int n, double* __restrict__ H) {
    const int p = blockIdx.y, q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const double l = lam(p, n) + lam(q, n);
    const double m00 = net.Gd * l + net.gdt, m01 = -net.gdt;
    const double m11 = net.Gt * l + net.gdt + net.gts, m12 = -net.gts;
    const double m22 = net.Gs * l + net.gts + net.gsink;
    const double cof = m11 * m22 - m12 * m12;
    const double det = m00 * cof - m01 * m01 * m22;
    H[p * n + q] = cof / det;
}

// A[p][x] = w_p cos(pi p (c+1/2)/n) cos(pi p (x+1/2)/n)
__global__ void k_modal_A(int n, double* __restrict__ A) {
    const int p = blockIdx.y, x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= n) return;
    const int c = n / 2;
    const double w = p == 0 ? 1.0 / n : 2.0 / n;
    A[p * n + x] = w * cos_half(p, c, n) * cos_half(p, x, n);
}

// C = op(A) * B for n x n fp64 matrices; op = transpose when TA.
template <bool TA>
__global__ void k_gemm(const double* __restrict__ A, const double* __restrict__ B, int n, double* __restrict__ C) {
    __shared__ double sa[16][17], sb[16][17];
    const int r = blockIdx.y * 16 + threadIdx.y, col = blockIdx.x * 16 + threadIdx.x;
    double acc = 0.0;
    for (int k0 = 0; k0 < n; k0 += 16) {
        const int ka = k0 + threadIdx.x, kb = k0 + threadIdx.y;
        sa[threadIdx.y][threadIdx.x] = (r < n && ka < n) ? (TA ? A[ka * n + r] : A[r * n + ka]) : 0.0;
        sb[threadIdx.y][threadIdx.x] = (kb < n && col < n) ? B[kb * n + col] : 0.0;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += sa[threadIdx.y][k] * sb[k][threadIdx.x];
        __syncthreads();
    }
    if (r < n && col < n) C[r * n + col] = acc;
}

// center value sum_pq H_pq a_p(c) a_q(c) for `count` conductivity variants at once: out[v]
__global__ void k_modal_center(const Net* __restrict__ nets, int count, int n, double* __restrict__ out) {
    const int v = blockIdx.x;
    if (v >= count) return;
    const Net net = nets[v];
    const int c = n / 2;
    double s = 0.0;
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
        const int p = idx / n, q = idx - p * n;
        const double l = lam(p, n) + lam(q, n);
        const double m00 = net.Gd * l + net.gdt, m01 = -net.gdt;
        const double m11 = net.Gt * l + net.gdt + net.gts, m12 = -net.gts;
        const double m22 = net.Gs * l + net.gts + net.gsink;
        const double cof = m11 * m22 - m12 * m12;
        const double det = m00 * cof - m01 * m01 * m22;
        const double ap = (p == 0 ? 1.0 / n : 2.0 / n) * cos_half(p, c, n) * cos_half(p, c, n);
        const double aq = (q == 0 ? 1.0 / n : 2.0 / n) * cos_half(q, c, n) * cos_half(q, c, n);
        s += cof / det * ap * aq;
    }
    __shared__ double red[32];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w) s += red[w];
        out[v] = s;
    }
}

// Backward-Euler centre-cell response to a held 1 W centre source
// (transient_impulse, fdm.cpp:257-286): per mode, steps[i] backward-Euler steps
// then accumulate a_p(c) a_q(c) x_d into part[block][i].
__global__ void k_modal_transient(Net net, int n, double dt, const int* __restrict__ steps, int ntimes,
                                  double* __restrict__ part) {
    extern __shared__ double acc[];
    for (int i = threadIdx.x; i < ntimes; i += blockDim.x) acc[i] = 0.0;
    __syncthreads();
    const int c = n / 2;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * n; idx += gridDim.x * blockDim.x) {
        const int p = idx / n, q = idx - p * n;
        const double l = lam(p, n) + lam(q, n);
        const double cd = net.Cd / dt, ct = net.Ct / dt, cs = net.Cs / dt;
        // A = M + C/dt (symmetric tridiagonal 3x3), solved by Thomas elimination per step
        const double a00 = net.Gd * l + net.gdt + cd, a01 = -net.gdt;
        const double a11 = net.Gt * l + net.gdt + net.gts + ct, a12 = -net.gts;
        const double a22 = net.Gs * l + net.gts + net.gsink + cs;
        const double w = ((p == 0 ? 1.0 / n : 2.0 / n) * cos_half(p, c, n) * cos_half(p, c, n)) *
                         ((q == 0 ? 1.0 / n : 2.0 / n) * cos_half(q, c, n) * cos_half(q, c, n));
        double x0 = 0.0, x1 = 0.0, x2 = 0.0;
        int done = 0;
        // modal source of a unit centre impulse is 1 in the die layer (weights applied at readout)
        const double d1 = a11 - a01 * a01 / a00;
        const double d2 = a22 - a12 * a12 / d1;
        for (int i = 0; i < ntimes; ++i) {
            for (; done < steps[i]; ++done) {
                const double b0 = 1.0 + cd * x0, b1 = ct * x1, b2 = cs * x2;
                const double y1 = b1 - a01 / a00 * b0;
                const double y2 = b2 - a12 / d1 * y1;
                x2 = y2 / d2;
                x1 = (y1 - a12 * x2) / d1;
                x0 = (b0 - a01 * x1) / a00;
            }
            atomicAdd(&acc[i], w * x0);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ntimes; i += blockDim.x) part[static_cast<size_t>(blockIdx.x) * ntimes + i] = acc[i];
}

// fit_capacitance model (greens.cpp:274-344): for `cap`, out[i] = (1/m^2) sum_modes
// Re( f (1 - exp(-t_i / (cap f))) ) (Re f for spectrally empty modes / Re tau <= 0).
__global__ void k_cap_model(const double2* __restrict__ fk, size_t count, double floor_abs, double cap,
                            const double* __restrict__ times, int ntimes, double* __restrict__ part) {
    extern __shared__ double acc[];
    for (int i = threadIdx.x; i < ntimes; i += blockDim.x) acc[i] = 0.0;
    __syncthreads();
    double loc[16];
    for (int i = 0; i < ntimes && i < 16; ++i) loc[i] = 0.0;
    for (size_t q = blockIdx.x * size_t(blockDim.x) + threadIdx.x; q < count; q += size_t(gridDim.x) * blockDim.x) {
        const double2 f = fk[q];
        const double a = sqrt(f.x * f.x + f.y * f.y);
        const double2 tau = make_double2(cap * f.x, cap * f.y);
        const bool sat = a <= floor_abs || !(tau.x > 0.0);
        const double d = tau.x * tau.x + tau.y * tau.y;
        for (int i = 0; i < ntimes && i < 16; ++i) {
            if (sat) {
                loc[i] += f.x;
            } else {
                const double zr = -times[i] * tau.x / d, zi = times[i] * tau.y / d;
                double s, c;
                sincos(zi, &s, &c);
                const double e = exp(zr);
                // Re( f (1 - e^{z}) )
                loc[i] += f.x * (1.0 - e * c) + f.y * (e * s);
            }
        }
    }
    for (int i = 0; i < ntimes && i < 16; ++i) atomicAdd(&acc[i], loc[i]);
    __syncthreads();
    for (int i = threadIdx.x; i < ntimes; i += blockDim.x) part[static_cast<size_t>(blockIdx.x) * ntimes + i] = acc[i];
}

__global__ void k_sum_parts(const double* __restrict__ part, int blocks, int ntimes, double scale,
                            double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ntimes) return;
    double s = 0.0;
    for (int b = 0; b < blocks; ++b) s += part[static_cast<size_t>(b) * ntimes + i];
    out[i] = s * scale;
}

}  // namespace

extern "C" {

// Network of fdm.cpp:23-110 for a uniform die conductivity k_die.
static Net make_net(const gtd_stack* s, double k_die) {
    const double pitch = s->die_edge / s->n, area = pitch * pitch;
    Net net;
    net.Gd = 2.0 * s->t_die * k_die * k_die / (k_die + k_die);
    net.Gt = s->t_tim * s->k_tim;
    net.Gs = s->t_spr * s->k_spr;
    net.gdt = area / (s->t_die / (2.0 * k_die) + s->t_tim / (2.0 * s->k_tim));
    net.gts = area / (s->t_tim / (2.0 * s->k_tim) + s->t_spr / (2.0 * s->k_spr));
    const double r_spread_half = s->t_spr / (2.0 * s->k_spr * area);
    net.gsink = 1.0 / (r_spread_half + static_cast<double>(s->n) * s->n * s->sink_resistance);
    net.Cd = s->c_die * area * s->t_die;
    net.Ct = s->c_tim * area * s->t_tim;
    net.Cs = s->c_spr * area * s->t_spr;
    return net;
}

int gtd_modal_impulse(const gtd_stack* s, double k_die, double* work, double* out, cudaStream_t st) {
    const int n = s->n;
    const size_t nn = static_cast<size_t>(n) * n;
    double* H = work;
    double* A = work + nn;
    double* T = work + 2 * nn;
    const Net net = make_net(s, k_die);
    k_modal_H<<<dim3((n + 127) / 128, n), 128, 0, st>>>(net, n, H);
    k_modal_A<<<dim3((n + 127) / 128, n), 128, 0, st>>>(n, A);
    const dim3 g((n + 15) / 16, (n + 15) / 16), b(16, 16);
    k_gemm<false><<<g, b, 0, st>>>(H, A, n, T);  // T[p][y] = sum_q H[p][q] A[q][y]
    k_gemm<true><<<g, b, 0, st>>>(A, T, n, out); // out[x][y] = sum_p A[p][x] T[p][y]
    return static_cast<int>(cudaGetLastError());
}

int gtd_modal_center(const gtd_stack* s, const double* k_values, int count, double* d_nets, double* out,
                     cudaStream_t st) {
    Net hn[64];
    if (count > 64) return static_cast<int>(cudaErrorInvalidValue);
    for (int i = 0; i < count; ++i) hn[i] = make_net(s, k_values[i]);
    cudaMemcpyAsync(d_nets, hn, sizeof(Net) * count, cudaMemcpyHostToDevice, st);
    k_modal_center<<<count, 1024, 0, st>>>(reinterpret_cast<const Net*>(d_nets), count, s->n, out);
    return static_cast<int>(cudaGetLastError());
}

size_t gtd_modal_net_bytes(void) { return sizeof(Net); }

int gtd_modal_transient(const gtd_stack* s, double k_die, double dt, const int* steps_d, int ntimes,
                        double* part, int blocks, double* out, cudaStream_t st) {
    const Net net = make_net(s, k_die);
    k_modal_transient<<<blocks, 256, sizeof(double) * ntimes, st>>>(net, s->n, dt, steps_d, ntimes, part);
    k_sum_parts<<<1, 64, 0, st>>>(part, blocks, ntimes, 1.0, out);
    return static_cast<int>(cudaGetLastError());
}

int gtd_cap_model(const void* fk_full, size_t count, double floor_abs, double cap, const double* times_d,
                  int ntimes, double inv_m2, double* part, int blocks, double* out, cudaStream_t st) {
    if (ntimes > 16) return static_cast<int>(cudaErrorInvalidValue);
    k_cap_model<<<blocks, 256, sizeof(double) * ntimes, st>>>(static_cast<const double2*>(fk_full), count, floor_abs,
                                                             cap, times_d, ntimes, part);
    k_sum_parts<<<1, 64, 0, st>>>(part, blocks, ntimes, inv_m2, out);
    return static_cast<int>(cudaGetLastError());
}

}  // extern "C"
