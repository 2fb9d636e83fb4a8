// oracle/shim/fftw_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// fp64 implementation of the FFTW3 subset declared in shim/fftw3.h, so the
// unchanged reference spectral.cpp links. Power-of-two sizes use an iterative
// radix-2 decimation-in-time transform with exact (directly evaluated)
// twiddles; rows are transformed one at a time, columns are transformed with
// the butterflies vectorised across all columns of a row pair (contiguous
// inner loops). Other sizes fall back to a direct O(n^2) DFT per line.
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

namespace {

using cd = std::complex<double>;

struct Line {
    int n = 0;
    bool pow2 = false;
    int sign = -1;
    std::vector<cd> tw;        // tw[k] = exp(sign*2*pi*i*k/n), k < n (full table for direct DFT)
    std::vector<int> bitrev;   // power-of-two only

    void init(int n_, int sign_) {
        n = n_;
        sign = sign_;
        pow2 = n > 0 && (n & (n - 1)) == 0;
        tw.resize(n);
        for (int k = 0; k < n; ++k) {
            const double a = sign * 2.0 * M_PI * static_cast<double>(k) / n;
            tw[k] = cd(std::cos(a), std::sin(a));
        }
        if (pow2) {
            bitrev.resize(n);
            int lg = 0;
            while ((1 << lg) < n) ++lg;
            for (int i = 0; i < n; ++i) {
                int r = 0;
                for (int b = 0; b < lg; ++b)
                    if (i & (1 << b)) r |= 1 << (lg - 1 - b);
                bitrev[i] = r;
            }
        }
    }

    // In-place transform of one contiguous line.
    void run(cd* x, std::vector<cd>& scratch) const {
        if (n <= 1) return;
        if (!pow2) {
            scratch.assign(x, x + n);
            for (int k = 0; k < n; ++k) {
                cd s = 0.0;
                for (int j = 0; j < n; ++j)
                    s += scratch[j] * tw[(static_cast<long long>(j) * k) % n];
                x[k] = s;
            }
            return;
        }
        for (int i = 0; i < n; ++i)
            if (bitrev[i] > i) std::swap(x[i], x[bitrev[i]]);
        for (int len = 2; len <= n; len <<= 1) {
            const int half = len >> 1, step = n / len;
            for (int base = 0; base < n; base += len)
                for (int k = 0; k < half; ++k) {
                    cd b = x[base + k + half] * tw[k * step];
                    cd a = x[base + k];
                    x[base + k] = a + b;
                    x[base + k + half] = a - b;
                }
        }
    }
};

}  // namespace

struct gt_shim_fftw_plan_s {
    int n0 = 0, n1 = 0;
    Line rows, cols;  // rows: length n1 lines; cols: length n0 lines
};

extern "C" {

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex*, fftw_complex*, int sign, unsigned) {
    if (n0 < 1 || n1 < 1 || (sign != FFTW_FORWARD && sign != FFTW_BACKWARD)) return nullptr;
    auto* p = new gt_shim_fftw_plan_s;
    p->n0 = n0;
    p->n1 = n1;
    p->rows.init(n1, sign);
    p->cols.init(n0, sign);
    return p;
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    const int n0 = p->n0, n1 = p->n1;
    cd* x = reinterpret_cast<cd*>(out);
    if (in != out) std::memmove(out, in, sizeof(cd) * static_cast<size_t>(n0) * n1);
    std::vector<cd> scratch;
    // Pass 1: every row (contiguous).
    for (int r = 0; r < n0; ++r) p->rows.run(x + static_cast<size_t>(r) * n1, scratch);
    // Pass 2: columns.
    const Line& L = p->cols;
    if (n0 <= 1) return;
    if (!L.pow2) {
        std::vector<cd> col(n0);
        for (int c = 0; c < n1; ++c) {
            for (int r = 0; r < n0; ++r) col[r] = x[static_cast<size_t>(r) * n1 + c];
            L.run(col.data(), scratch);
            for (int r = 0; r < n0; ++r) x[static_cast<size_t>(r) * n1 + c] = col[r];
        }
        return;
    }
    std::vector<cd> tmp(n1);
    for (int i = 0; i < n0; ++i) {
        const int j = L.bitrev[i];
        if (j > i) {
            cd* a = x + static_cast<size_t>(i) * n1;
            cd* b = x + static_cast<size_t>(j) * n1;
            std::memcpy(tmp.data(), a, sizeof(cd) * n1);
            std::memcpy(a, b, sizeof(cd) * n1);
            std::memcpy(b, tmp.data(), sizeof(cd) * n1);
        }
    }
    for (int len = 2; len <= n0; len <<= 1) {
        const int half = len >> 1, step = n0 / len;
        for (int base = 0; base < n0; base += len)
            for (int k = 0; k < half; ++k) {
                const cd w = L.tw[k * step];
                double* a = reinterpret_cast<double*>(x + static_cast<size_t>(base + k) * n1);
                double* b = reinterpret_cast<double*>(x + static_cast<size_t>(base + k + half) * n1);
                const double wr = w.real(), wi = w.imag();
                for (int c = 0; c < n1; ++c) {
                    const double br = b[2 * c] * wr - b[2 * c + 1] * wi;
                    const double bi = b[2 * c] * wi + b[2 * c + 1] * wr;
                    const double ar = a[2 * c], ai = a[2 * c + 1];
                    a[2 * c] = ar + br;
                    a[2 * c + 1] = ai + bi;
                    b[2 * c] = ar - br;
                    b[2 * c + 1] = ai - bi;
                }
            }
    }
}

void fftw_execute(const fftw_plan) {}

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
