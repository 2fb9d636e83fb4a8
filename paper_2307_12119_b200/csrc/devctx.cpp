// devctx.cpp — device context: buffers, error mapping, GreensSet preparation.
#include "devctx.hpp"

namespace gth {

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(ST_INTERNAL, "device", std::string(what) + ": " + cudaGetErrorString(e));
}

void need_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1)
        fail(ST_INTERNAL, "device", "no CUDA device available (this library has no CPU solve path)");
}


void DBuf::ensure(size_t b) {
    if (b <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cuda_ok(cudaMalloc(&p, b), "cudaMalloc");
    bytes = b;
}


namespace {

// Host-computed fp64 constant tables (analytic; no transform work).
std::vector<double> twiddles(int m) {
    std::vector<double> t(2 * static_cast<size_t>(m));
    for (int k = 0; k < m; ++k) {
        const double a = -2.0 * M_PI * static_cast<double>(k) / m;
        t[2 * k] = std::cos(a);
        t[2 * k + 1] = std::sin(a);
    }
    return t;
}

// hs[t] = exp(-i pi t / m): half-step twiddles (w^{t/2}, w = exp(-2 pi i / m)).
std::vector<double> half_twiddles(int m) {
    std::vector<double> t(2 * static_cast<size_t>(m));
    for (int k = 0; k < m; ++k) {
        const double a = -M_PI * static_cast<double>(k) / m;
        t[2 * k] = std::cos(a);
        t[2 * k + 1] = std::sin(a);
    }
    return t;
}

// k1[u] = sum_{x<n} exp(-2 pi i u (x - c) / m): spectrum of the centred die box.
std::vector<double> box_spectrum(int n) {
    const int m = 2 * n, c = n / 2;
    std::vector<double> k(2 * static_cast<size_t>(m));
    for (int u = 0; u < m; ++u) {
        double re = 0.0, im = 0.0;
        for (int x = 0; x < n; ++x) {
            const long long e = (static_cast<long long>(u) * (x - c)) % m;
            const double a = -2.0 * M_PI * static_cast<double>((e + m) % m) / m;
            re += std::cos(a);
            im += std::sin(a);
        }
        k[2 * u] = re;
        k[2 * u + 1] = im;
    }
    return k;
}

template <typename T>
std::vector<T> narrow(const std::vector<double>& v) {
    return std::vector<T>(v.begin(), v.end());
}

}  // namespace

void upload(DBuf& b, const void* src, size_t bytes, cudaStream_t st) {
    b.ensure(bytes);
    cuda_ok(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, st), "upload");
}

// Large grids (n > 1024, config 4): fp64 only, and only what the four-step
// large-grid passes read -- twiddles and the baseline kernel half spectrum fk,
// built on the device by the same passes (large.cu). The batched mode-A/B and
// reference-API paths reject these grids (their tables are not built).
std::unique_ptr<gt_device_greens> prepare_device_large(const Greens& g, int device) {
    const int n = g.n, m = 2 * n;
    cuda_ok(cudaSetDevice(device), "cudaSetDevice");
    auto d = std::make_unique<gt_device_greens>();
    d->device = device;
    d->fp64 = 1;
    d->host = g;
    cuda_ok(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking), "stream");
    cudaStream_t st = d->stream;
    const int hp = ((n + 1 + 7) / 8) * 8;
    const std::vector<double> tw = twiddles(m), hs = half_twiddles(m);
    upload(d->tw64, tw.data(), tw.size() * 8, st);
    upload(d->tw, tw.data(), tw.size() * 8, st);
    upload(d->hs, hs.data(), hs.size() * 8, st);
    upload(d->fsp0, g.f_sp0.v.data(), g.f_sp0.v.size() * 8, st);
    d->fk.ensure(static_cast<size_t>(m) * hp * 16);
    gtd_lg lg{};
    lg.n = n;
    lg.m = m;
    if (gtd_lg_split(m, &lg.M1, &lg.M2)) fail(ST_CONFIG, "device", "large grid: m out of range");
    lg.tw = d->tw64.p;
    lg.fkp = hp;
    {
        DBuf s1, z, c1;
        s1.ensure(static_cast<size_t>(n / 2) * m * 16);
        z.ensure(static_cast<size_t>(n / 2) * m * 16);
        c1.ensure(static_cast<size_t>(m) * hp * 16);
        cuda_ok(gtd_lg_kernel_spectrum(&lg, d->fsp0.as<double>(), g.phi, s1.p, z.p, c1.p, d->fk.p, st),
                "large kernel spectrum");
        cuda_ok(cudaStreamSynchronize(st), "sync");
    }
    d->d.n = n;
    d->d.m = m;
    d->d.h = n + 1;
    d->d.hp = hp;
    d->d.fp64 = 1;
    d->d.fk = d->fk.p;
    d->d.tw = d->tw.p;
    d->d.hs = d->hs.p;
    d->d.alpha = g.alpha;
    d->d.beta = g.beta;
    d->d.rand_scale = g.rand_scale;
    d->d.mu_fixed = g.mu;
    return d;
}

std::unique_ptr<gt_device_greens> prepare_device(const Greens& g, int precision, int device) {
    need_device();
    const int n = g.n;
    if (pow2(n) && n > 1024 && n <= 16384) {
        if (precision != GT_FP64)
            fail(ST_CONFIG, "device", "grids above n = 1024 run the fp64 large-grid path only (use GT_FP64)");
        return prepare_device_large(g, device);
    }
    if (!pow2(n) || n < 16 || n > 1024)
        fail(ST_CONFIG, "device", "device path supports power-of-two grids 16..1024 (16384 in fp64), got n=" +
                                      std::to_string(n));
    if (precision != GT_FP32 && precision != GT_FP64) fail(ST_CONFIG, "device", "precision must be GT_FP32 or GT_FP64");
    cuda_ok(cudaSetDevice(device), "cudaSetDevice");
    auto d = std::make_unique<gt_device_greens>();
    d->device = device;
    d->fp64 = precision == GT_FP64;
    d->host = g;
    cuda_ok(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking), "stream");
    const int m = 2 * n, hp = gtd_padded_width(n, d->fp64);
    const size_t cb = d->fp64 ? 16 : 8, rb = d->fp64 ? 8 : 4;
    cudaStream_t st = d->stream;

    const std::vector<double> tw = twiddles(m), k1 = box_spectrum(n), hs = half_twiddles(m);
    upload(d->tw64, tw.data(), tw.size() * 8, st);
    if (d->fp64) {
        upload(d->tw, tw.data(), tw.size() * 8, st);
        upload(d->k1, k1.data(), k1.size() * 8, st);
        upload(d->hs, hs.data(), hs.size() * 8, st);
    } else {
        auto twf = narrow<float>(tw), k1f = narrow<float>(k1), hsf = narrow<float>(hs);
        upload(d->tw, twf.data(), twf.size() * 4, st);
        upload(d->k1, k1f.data(), k1f.size() * 4, st);
        upload(d->hs, hsf.data(), hsf.size() * 4, st);
        cuda_ok(cudaStreamSynchronize(st), "sync");
    }
    upload(d->fsp0, g.f_sp0.v.data(), g.f_sp0.v.size() * 8, st);
    upload(d->gsp0, g.g_sp0.v.data(), g.g_sp0.v.size() * 8, st);
    d->fk_full.ensure(static_cast<size_t>(m) * m * 16);
    d->fk.ensure(static_cast<size_t>(m) * hp * cb);
    d->gtab.ensure(static_cast<size_t>(n + 1) * hp * rb);
    d->fg.ensure(static_cast<size_t>(m) * hp * 4 * rb);
    cuda_ok(gtd_greens_tables(static_cast<const double*>(d->fsp0.p), static_cast<const double*>(d->gsp0.p),
                              g.phi, n, hp, d->fp64, d->tw64.p, d->fk_full.p, d->fk.p, d->gtab.p, d->fg.p, g.alpha,
                              st),
            "greens tables");
    {
        DBuf flag;
        flag.ensure(sizeof(int));
        d->fgm.ensure(static_cast<size_t>(m) * hp * 4 * rb);
        cuda_ok(gtd_greens_fgm(d->fk_full.p, static_cast<const double*>(d->gsp0.p), n, hp, d->fp64, g.alpha,
                               g.mu * g.beta, d->fgm.p, flag.as<int>(), st),
                "fixed-mu table");
        int f = 0;
        cuda_ok(cudaMemcpyAsync(&f, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st), "flag");
        cuda_ok(cudaStreamSynchronize(st), "greens tables sync");
        d->d.det_flags = f ? GTD_ST_RUNAWAY_DET : 0;
    }
    d->d.n = n;
    d->d.m = m;
    d->d.h = n + 1;
    d->d.hp = hp;
    d->d.fp64 = d->fp64;
    d->d.fk = d->fk.p;
    d->d.gtab = d->gtab.p;
    d->d.k1 = d->k1.p;
    d->d.tw = d->tw.p;
    d->d.fg = d->fg.p;
    d->d.fgm = d->fgm.p;
    d->d.hs = d->hs.p;
    d->d.alpha = g.alpha;
    d->d.beta = g.beta;
    d->d.rand_scale = g.rand_scale;
    d->d.mu_fixed = g.mu;
    return d;
}


}  // namespace gth
