// fdm.cu — the reference's FDM thermal network (fdm.cpp:45-110) on the device:
// matrix-free operator of the 3-layer (die, TIM, spreader) 7-point network with
// per-cell die conductivity, and the vector kernels of the Jacobi-preconditioned
// conjugate gradient the reference runs through Eigen (fdm.cpp:120-146). fp64.
// Host loops (outer fixed point, backward Euler, CG iteration control):
// fdm_host.cpp.
#include <cuda_runtime.h>

#include "gt_device.h"

namespace {

constexpr int FT = 256;

__device__ __forceinline__ double harm(double a, double b) { return 2.0 * a * b / (a + b); }

// Effective per-cell die conductivity k0 (1 - c rise) (fdm.cpp:55-64); flag on k <= 0.
__global__ void k_kcell(const double* __restrict__ k_map, const double* __restrict__ rise, double c, int nn,
                        double* __restrict__ kd, int* flag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nn) return;
    double k = k_map[i];
    if (rise) k = k * (1.0 - c * rise[i]);
    if (!(k > 0.0)) atomicOr(flag, 1);
    kd[i] = k;
}

struct Net {
    int n;
    double td, tt, ts, kt, ks, area, g_sink, cd, ct, cs, idt;
    const double* kd;
    __device__ double gdt(int c) const { return area / (td / (2.0 * kd[c]) + tt / (2.0 * kt)); }
    __device__ double gts() const { return area / (tt / (2.0 * kt) + ts / (2.0 * ks)); }
};

// diag = sum of incident conductances (+ sink, + C/dt)
__global__ void k_diag(Net net, double* __restrict__ diag) {
    const int n = net.n, nn = n * n;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= 3 * nn) return;
    const int l = idx / nn, c = idx - l * nn, i = c / n, j = c - (c / n) * n;
    double s = 0.0;
    const int nb = (j > 0) + (j + 1 < n) + (i > 0) + (i + 1 < n);
    if (l == 0) {
        const double k = net.kd[c];
        if (j > 0) s += net.td * harm(k, net.kd[c - 1]);
        if (j + 1 < n) s += net.td * harm(k, net.kd[c + 1]);
        if (i > 0) s += net.td * harm(k, net.kd[c - n]);
        if (i + 1 < n) s += net.td * harm(k, net.kd[c + n]);
        s += net.gdt(c) + net.cd * net.idt;
    } else if (l == 1) {
        s += nb * net.tt * net.kt + net.gdt(c) + net.gts() + net.ct * net.idt;
    } else {
        s += nb * net.ts * net.ks + net.gts() + net.g_sink + net.cs * net.idt;
    }
    diag[idx] = s;
}

// y = A x; optionally dot += w . y (block reduce + one atomic)
__global__ void k_spmv(Net net, const double* __restrict__ diag, const double* __restrict__ x,
                       double* __restrict__ y, const double* __restrict__ w, double* dot) {
    const int n = net.n, nn = n * n;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    double v = 0.0;
    if (idx < 3 * nn) {
        const int l = idx / nn, c = idx - l * nn, i = c / n, j = c - (c / n) * n;
        double acc = diag[idx] * x[idx];
        if (l == 0) {
            const double k = net.kd[c];
            if (j > 0) acc -= net.td * harm(k, net.kd[c - 1]) * x[idx - 1];
            if (j + 1 < n) acc -= net.td * harm(k, net.kd[c + 1]) * x[idx + 1];
            if (i > 0) acc -= net.td * harm(k, net.kd[c - n]) * x[idx - n];
            if (i + 1 < n) acc -= net.td * harm(k, net.kd[c + n]) * x[idx + n];
            acc -= net.gdt(c) * x[nn + c];
        } else {
            const double g = l == 1 ? net.tt * net.kt : net.ts * net.ks;
            double lat = 0.0;
            if (j > 0) lat += x[idx - 1];
            if (j + 1 < n) lat += x[idx + 1];
            if (i > 0) lat += x[idx - n];
            if (i + 1 < n) lat += x[idx + n];
            acc -= g * lat;
            if (l == 1) acc -= net.gdt(c) * x[c] + net.gts() * x[2 * nn + c];
            else acc -= net.gts() * x[nn + c];
        }
        y[idx] = acc;
        if (w) v = w[idx] * acc;
    }
    if (dot) {
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        __shared__ double red[FT / 32];
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int k = 0; k < FT / 32; ++k) s += red[k];
            atomicAdd(dot, s);
        }
    }
}

// Block-reduced dot products into out[0..cnt)
__device__ void block_add(double v0, double v1, double* out0, double* out1) {
    __syncthreads();  // previous call's readers of the shared partials are done
    for (int o = 16; o > 0; o >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    }
    __shared__ double r0[FT / 32], r1[FT / 32];
    if ((threadIdx.x & 31) == 0) {
        r0[threadIdx.x >> 5] = v0;
        r1[threadIdx.x >> 5] = v1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int k = 0; k < FT / 32; ++k) {
            s0 += r0[k];
            s1 += r1[k];
        }
        if (out0) atomicAdd(out0, s0);
        if (out1) atomicAdd(out1, s1);
    }
}

// r = b - Ax (Ax given); z = r / diag; p = z; sc[RZ] += r.z; sc[RR] += r.r; sc[BB] += b.b
__global__ void k_cg_init(int N, const double* __restrict__ b, const double* __restrict__ ax,
                          const double* __restrict__ diag, double* __restrict__ r, double* __restrict__ z,
                          double* __restrict__ p, double* sc) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double rz = 0.0, rr = 0.0, bb = 0.0;
    if (i < N) {
        const double ri = b[i] - ax[i], zi = ri / diag[i];
        r[i] = ri;
        z[i] = zi;
        p[i] = zi;
        rz = ri * zi;
        rr = ri * ri;
        bb = b[i] * b[i];
    }
    block_add(rz, rr, sc + 0, sc + 1);
    block_add(bb, 0.0, sc + 2, nullptr);
}

// alpha = sc[RZ] / sc[PQ]; x += alpha p; r -= alpha q; z = r / diag; sc[RR2] += r.r; sc[RZ2] += r.z
__global__ void k_cg_update(int N, const double* __restrict__ p, const double* __restrict__ q,
                            const double* __restrict__ diag, double* __restrict__ x, double* __restrict__ r,
                            double* __restrict__ z, double* sc) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const double alpha = sc[0] / sc[3];
    double rr = 0.0, rz = 0.0;
    if (i < N) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * q[i], zi = ri / diag[i];
        r[i] = ri;
        z[i] = zi;
        rr = ri * ri;
        rz = ri * zi;
    }
    block_add(rr, rz, sc + 4, sc + 5);
}

// beta = sc[RZ2] / sc[RZ]; p = z + beta p
__global__ void k_cg_p(int N, const double* __restrict__ z, double* __restrict__ p, const double* sc) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) p[i] = z[i] + (sc[5] / sc[0]) * p[i];
}

// rotate scalars for the next iteration: RZ <- RZ2, clear PQ, RR2, RZ2
__global__ void k_cg_rotate(double* sc) {
    sc[0] = sc[5];
    sc[3] = 0.0;
    sc[4] = 0.0;
    sc[5] = 0.0;
}

// rhs: die plane p_dyn + leakage (static p_leak0 or (1 + beta dT) p_leak0, leakage_at_temperature,
// variation.cpp:213-222) at the die rise x; + C/dt x for backward Euler
__global__ void k_fdm_rhs(const double* __restrict__ p_dyn, const double* __restrict__ leak, int temp_dep,
                          double beta, const double* __restrict__ x, double c_die, double c_tim, double c_spr,
                          double inv_dt, int nn, double* __restrict__ b) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * nn) return;
    const int l = i / nn, c = i - l * nn;
    double v = 0.0;
    if (l == 0) {
        v = p_dyn[c];
        if (leak) v += temp_dep ? (1.0 + beta * x[c]) * leak[c] : leak[c];
    }
    if (inv_dt > 0.0) v += (l == 0 ? c_die : l == 1 ? c_tim : c_spr) * inv_dt * x[i];
    b[i] = v;
}

__global__ void k_absdiff(const double* __restrict__ a, const double* __restrict__ b, size_t count,
                          double* __restrict__ out) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x)
        out[i] = fabs(a[i] - b[i]);
}

Net to_net(const gtd_fdm* f) {
    Net n{};
    n.n = f->n;
    n.td = f->t_die;
    n.tt = f->t_tim;
    n.ts = f->t_spr;
    n.kt = f->k_tim;
    n.ks = f->k_spr;
    n.area = f->pitch * f->pitch;
    n.g_sink = f->g_sink;
    n.cd = f->c_die;
    n.ct = f->c_tim;
    n.cs = f->c_spr;
    n.idt = f->inv_dt;
    n.kd = f->kd;
    return n;
}

int blocks(int N) { return (N + FT - 1) / FT; }

}  // namespace

extern "C" {

int gtd_fdm_kcell(const double* k_map, const double* rise, double c, int n, double* kd, int* flag, cudaStream_t st) {
    k_kcell<<<blocks(n * n), FT, 0, st>>>(k_map, rise, c, n * n, kd, flag);
    return static_cast<int>(cudaGetLastError());
}

int gtd_fdm_diag(const gtd_fdm* f, double* diag, cudaStream_t st) {
    k_diag<<<blocks(3 * f->n * f->n), FT, 0, st>>>(to_net(f), diag);
    return static_cast<int>(cudaGetLastError());
}

int gtd_fdm_spmv(const gtd_fdm* f, const double* diag, const double* x, double* y, const double* w, double* dot,
                 cudaStream_t st) {
    k_spmv<<<blocks(3 * f->n * f->n), FT, 0, st>>>(to_net(f), diag, x, y, w, dot);
    return static_cast<int>(cudaGetLastError());
}

int gtd_fdm_rhs(const double* p_dyn, const double* leak, int temp_dep, double beta, const double* x, double c_die,
                double c_tim, double c_spr, double inv_dt, int nn, double* b, cudaStream_t st) {
    k_fdm_rhs<<<blocks(3 * nn), FT, 0, st>>>(p_dyn, leak, temp_dep, beta, x, c_die, c_tim, c_spr, inv_dt, nn, b);
    return static_cast<int>(cudaGetLastError());
}

int gtd_absdiff(const double* a, const double* b, size_t count, double* out, cudaStream_t st) {
    k_absdiff<<<592, FT, 0, st>>>(a, b, count, out);
    return static_cast<int>(cudaGetLastError());
}

int gtd_cg_init(int N, const double* b, const double* ax, const double* diag, double* r, double* z, double* p,
                double* sc, cudaStream_t st) {
    cudaMemsetAsync(sc, 0, 8 * sizeof(double), st);
    k_cg_init<<<blocks(N), FT, 0, st>>>(N, b, ax, diag, r, z, p, sc);
    return static_cast<int>(cudaGetLastError());
}

int gtd_cg_step(const gtd_fdm* f, const double* diag, double* x, double* r, double* z, double* p, double* q,
                double* sc, cudaStream_t st) {
    const int N = 3 * f->n * f->n;
    k_spmv<<<blocks(N), FT, 0, st>>>(to_net(f), diag, p, q, p, sc + 3);  // q = A p, sc[PQ] = p.q
    k_cg_update<<<blocks(N), FT, 0, st>>>(N, p, q, diag, x, r, z, sc);
    return static_cast<int>(cudaGetLastError());
}

int gtd_cg_direction(int N, const double* z, double* p, double* sc, cudaStream_t st) {
    k_cg_p<<<blocks(N), FT, 0, st>>>(N, z, p, sc);
    k_cg_rotate<<<1, 1, 0, st>>>(sc);
    return static_cast<int>(cudaGetLastError());
}

}  // extern "C"
