// host.cpp — host data model (files, grids, GreensSet directories).
// File formats follow the reference byte-for-byte on write and accept what the
// reference accepts on read:
//   grid file     : "n pitch unit" header then n rows of n values, 17 significant
//                   digits (reference field.cpp:89-129)
//   key-value file: "key value" per line, '#' comments, '=' accepted as a
//                   separator, keys written sorted (reference kvfile.cpp:12-44,124-129)
//   GreensSet dir : manifest.txt, calibration.txt, f_sp0/g_sp0/f_det/f_rand/p_var.map,
//                   tran_###.map (reference greens.cpp:464-548)
#include "host.hpp"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>

namespace gth {

void fail(Status s, const std::string& stage, const std::string& msg) { throw Error(s, stage, msg); }

const char* unit_str(Unit u) {
    switch (u) {
        case Unit::Watts: return "watts";
        case Unit::Kelvin: return "kelvin";
        case Unit::KelvinPerWatt: return "kelvin_per_watt";
        default: return "dimensionless";
    }
}

Unit parse_unit(const std::string& s) {
    static const std::pair<const char*, Unit> table[] = {{"watts", Unit::Watts},
                                                         {"kelvin", Unit::Kelvin},
                                                         {"kelvin_per_watt", Unit::KelvinPerWatt},
                                                         {"dimensionless", Unit::Dimensionless}};
    for (const auto& [name, u] : table)
        if (s == name) return u;
    fail(ST_CONFIG, "field-io", "unknown field unit '" + s + "'");
}

Field::Field(int n_, double pitch_, Unit u, double fill) : n(n_), pitch(pitch_), unit(u) {
    if (n_ < 2) fail(ST_CONFIG, "field", "grid side must be >= 2, got " + std::to_string(n_));
    if (!(pitch_ > 0.0)) fail(ST_CONFIG, "field", "pitch must be positive");
    v.assign(static_cast<size_t>(n_) * n_, fill);
}

double Field::max() const { return *std::max_element(v.begin(), v.end()); }
double Field::min() const { return *std::min_element(v.begin(), v.end()); }

double Field::sum() const {
    double s = 0.0, lost = 0.0;
    for (double x : v) {
        const double t = s + x;
        lost += std::abs(s) >= std::abs(x) ? (s - t) + x : (x - t) + s;
        s = t;
    }
    return s + lost;
}

std::pair<int, int> Field::argmax() const {
    size_t k = static_cast<size_t>(std::max_element(v.begin(), v.end()) - v.begin());
    return {static_cast<int>(k) / n, static_cast<int>(k) % n};
}

void Field::check_finite(const char* what) const {
    for (double x : v)
        if (!std::isfinite(x)) fail(ST_VALIDATION, "field", std::string(what) + ": non-finite entry");
}

// Binary sidecar "<path>.bin": the 17-digit text stays the
// interchange format; a raw little-endian copy next to it makes re-reads of large
// maps (one 8192^2 map is ~1.7 GB of text) a memcpy. The sidecar is used only if
// it is at least as new as the text and records the text's byte size and a
// fingerprint of its content (FNV-1a over the first and last 4 KiB: the header line
// and the last rows), so a text rewritten by another tool -- same size, same
// timestamp granularity, or mtimes copied by cp -p / rsync / tar -- falls back to
// parsing. GT_NO_BINARY_SIDECAR=1 disables it.
namespace {
struct SidecarHeader {
    char magic[8];
    int32_t n, unit;
    double pitch;
    uint64_t text_bytes;
    uint64_t text_hash;
};
constexpr char kMagic[8] = {'G', 'T', 'F', 'B', '2', 0, 0, 0};
uint64_t text_fingerprint(const std::string& path, uint64_t size) {
    std::ifstream is(path, std::ios::binary);
    uint64_t h = 1469598103934665603ull ^ size;
    auto mix = [&](const char* p, std::streamsize k) {
        for (std::streamsize i = 0; i < k; ++i) h = (h ^ static_cast<unsigned char>(p[i])) * 1099511628211ull;
    };
    char buf[4096];
    is.read(buf, sizeof buf);
    mix(buf, is.gcount());
    if (size > 2 * sizeof buf) {
        is.clear();
        is.seekg(static_cast<std::streamoff>(size - sizeof buf));
        is.read(buf, sizeof buf);
        mix(buf, is.gcount());
    }
    return h;
}
bool sidecars_enabled() {
    const char* e = std::getenv("GT_NO_BINARY_SIDECAR");
    return !(e && *e && *e != '0');
}
bool read_sidecar(const std::string& path, Field* out) {
    namespace fs = std::filesystem;
    const std::string bin = path + ".bin";
    std::error_code ec;
    if (!sidecars_enabled() || !fs::exists(bin, ec) || !fs::exists(path, ec)) return false;
    if (fs::last_write_time(bin, ec) < fs::last_write_time(path, ec) || ec) return false;
    std::ifstream is(bin, std::ios::binary);
    SidecarHeader h{};
    if (!is.read(reinterpret_cast<char*>(&h), sizeof h)) return false;
    if (std::memcmp(h.magic, kMagic, 8) != 0 || h.n < 2 || h.unit < 0 || h.unit > 3) return false;
    const uint64_t size = static_cast<uint64_t>(fs::file_size(path, ec));
    if (ec || h.text_bytes != size || h.text_hash != text_fingerprint(path, size)) return false;
    Field f(h.n, h.pitch, static_cast<Unit>(h.unit));
    if (!is.read(reinterpret_cast<char*>(f.v.data()), static_cast<std::streamsize>(f.v.size() * sizeof(double))))
        return false;
    *out = std::move(f);
    return true;
}
void write_sidecar(const Field& f, const std::string& path) {
    namespace fs = std::filesystem;
    if (!sidecars_enabled()) return;
    std::error_code ec;
    SidecarHeader h{};
    std::memcpy(h.magic, kMagic, 8);
    h.n = f.n;
    h.unit = static_cast<int32_t>(f.unit);
    h.pitch = f.pitch;
    h.text_bytes = static_cast<uint64_t>(fs::file_size(path, ec));
    if (ec) return;
    h.text_hash = text_fingerprint(path, h.text_bytes);
    std::ofstream os(path + ".bin", std::ios::binary | std::ios::trunc);
    os.write(reinterpret_cast<const char*>(&h), sizeof h);
    os.write(reinterpret_cast<const char*>(f.v.data()), static_cast<std::streamsize>(f.v.size() * sizeof(double)));
    if (!os) {
        os.close();
        fs::remove(path + ".bin", ec);  // a partial sidecar must not be picked up
    }
}
}  // namespace

Field read_field(const std::string& path) {
    {
        Field f(2, 1.0, Unit::Watts);
        if (read_sidecar(path, &f)) {
            f.check_finite(path.c_str());
            return f;
        }
    }
    std::ifstream is(path);
    if (!is) fail(ST_CONFIG, "field-io", "cannot open '" + path + "'");
    int n = 0;
    double pitch = 0.0;
    std::string unit;
    if (!(is >> n >> pitch >> unit))
        fail(ST_CONFIG, "field-io", path + ": malformed header (want 'n pitch unit')");
    if (n < 2) fail(ST_CONFIG, "field-io", path + ": grid side must be >= 2");
    Field f(n, pitch, parse_unit(unit));
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            if (!(is >> f.at(i, j)))
                fail(ST_CONFIG, "field-io", path + ": truncated value grid at row " + std::to_string(i));
    f.check_finite(path.c_str());
    return f;
}

void write_field(const Field& f, const std::string& path) {
    std::ofstream os(path);
    if (!os) fail(ST_CONFIG, "field-io", "cannot open '" + path + "' for writing");
    os.precision(17);
    os << f.n << ' ' << f.pitch << ' ' << unit_str(f.unit) << '\n';
    for (int i = 0; i < f.n; ++i) {
        for (int j = 0; j < f.n; ++j) os << (j ? " " : "") << f.at(i, j);
        os << '\n';
    }
    if (!os) fail(ST_CONFIG, "field-io", "write failed for '" + path + "'");
    os.close();
    write_sidecar(f, path);
}

// ------------------------------------------------------------------- Kv
Kv Kv::parse(const std::string& path) {
    std::ifstream is(path);
    if (!is) fail(ST_CONFIG, "config", "cannot open '" + path + "'");
    Kv kv;
    kv.origin_ = path;
    std::string line;
    int no = 0;
    while (std::getline(is, line)) {
        ++no;
        if (auto p = line.find('#'); p != std::string::npos) line.resize(p);
        for (char& ch : line)
            if (ch == '=') ch = ' ';
        std::istringstream ls(line);
        std::string key;
        if (!(ls >> key)) continue;
        std::string rest;
        std::getline(ls, rest);
        const auto b = rest.find_first_not_of(" \t");
        if (b == std::string::npos)
            fail(ST_CONFIG, "config", path + ":" + std::to_string(no) + ": key '" + key + "' has no value");
        const auto e = rest.find_last_not_of(" \t\r");
        kv.m_[key] = rest.substr(b, e - b + 1);
    }
    return kv;
}

std::string Kv::str(const std::string& k) const {
    auto it = m_.find(k);
    if (it == m_.end()) fail(ST_CONFIG, "config", origin_ + ": missing required key '" + k + "'");
    return it->second;
}

double Kv::num(const std::string& k) const {
    const std::string s = str(k);
    size_t used = 0;
    double v = 0.0;
    try {
        v = std::stod(s, &used);
    } catch (const std::exception&) {
        used = 0;
    }
    if (used == 0 || used != s.size())
        fail(ST_CONFIG, "config", origin_ + ": key '" + k + "' is not a number: '" + s + "'");
    return v;
}

long long Kv::integer(const std::string& k) const {
    const std::string s = str(k);
    size_t used = 0;
    long long v = 0;
    try {
        v = std::stoll(s, &used);
    } catch (const std::exception&) {
        used = 0;
    }
    if (used == 0 || used != s.size())
        fail(ST_CONFIG, "config", origin_ + ": key '" + k + "' is not an integer: '" + s + "'");
    return v;
}

std::vector<double> Kv::list(const std::string& k) const {
    std::string s = str(k);
    std::replace(s.begin(), s.end(), ',', ' ');
    std::istringstream is(s);
    std::vector<double> out;
    for (double x; is >> x;) out.push_back(x);
    if (out.empty()) fail(ST_CONFIG, "config", origin_ + ": key '" + k + "' holds no numbers");
    return out;
}

void Kv::put_num(const std::string& k, double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    m_[k] = buf;
}

void Kv::known(const std::vector<std::string>& keys) const {
    for (const auto& kv : m_)
        if (std::find(keys.begin(), keys.end(), kv.first) == keys.end())
            fail(ST_CONFIG, "config", origin_ + ": unknown key '" + kv.first + "'");
}

void Kv::save(const std::string& path) const {
    std::ofstream os(path);
    if (!os) fail(ST_CONFIG, "config", "cannot open '" + path + "' for writing");
    for (const auto& kv : m_) os << kv.first << ' ' << kv.second << '\n';
    if (!os) fail(ST_CONFIG, "config", "write failed for '" + path + "'");
}

// --------------------------------------------------------------- GreensSet
void Greens::validate() const {
    if (n < 2 || f_sp0.n != n || f_det.n != n)
        fail(ST_CONFIG, "greens", "GreensSet maps are inconsistent with n");
    if (f_sp0.min() < 0.0) fail(ST_VALIDATION, "greens", "f_sp0 has negative entries");
    const auto [pi, pj] = f_sp0.argmax();
    if (pi != center() || pj != center())
        fail(ST_VALIDATION, "greens", "f_sp0 peak is not at the source cell");
    f_det.check_finite("f_det");
    f_rand.check_finite("f_rand");
}

static std::string tran_file(size_t i) {
    char b[32];
    std::snprintf(b, sizeof b, "tran_%03zu.map", i);
    return b;
}

static std::string join_list(const std::vector<double>& xs) {
    std::string out;
    char b[40];
    for (size_t i = 0; i < xs.size(); ++i) {
        std::snprintf(b, sizeof b, "%.17g", xs[i]);
        out += (i ? "," : "");
        out += b;
    }
    return out;
}

Greens load_greens_dir(const std::string& dir) {
    const Kv man = Kv::parse(dir + "/manifest.txt");
    Greens g;
    g.n = static_cast<int>(man.integer("n"));
    g.pitch = man.num("pitch");
    g.phi = man.num("phi");
    g.kappa_inf = man.num("kappa_inf");
    g.alpha = man.num("alpha");
    g.beta = man.num("beta");
    g.mu = man.num("mu");
    g.capacitance = man.num("capacitance");
    g.rand_scale = man.num("rand_scale", 1.0);
    g.f_sp0 = read_field(dir + "/f_sp0.map");
    g.g_sp0 = read_field(dir + "/g_sp0.map");
    g.f_det = read_field(dir + "/f_det.map");
    g.f_rand = read_field(dir + "/f_rand.map");
    g.p_var = read_field(dir + "/p_var.map");
    const long long cnt = man.integer("tran_count");
    if (cnt > 0) {
        g.t_samples = man.list("t_samples");
        if (static_cast<long long>(g.t_samples.size()) != cnt)
            fail(ST_CONFIG, "greens", dir + ": t_samples does not match tran_count");
        for (long long i = 0; i < cnt; ++i) g.tran.push_back(read_field(dir + "/" + tran_file(i)));
    }
    g.validate();
    const Kv cal = Kv::parse(dir + "/calibration.txt");
    g.c_prime = cal.num("c_prime");
    g.fit_r2 = cal.num("fit_r2");
    g.c = cal.num("c");
    g.rep_alpha = cal.num("alpha");
    g.cap_residual = cal.num("cap_residual", 0.0);
    if (cal.has("sweep_conductivity")) {
        auto ks = cal.list("sweep_conductivity"), ps = cal.list("sweep_peak");
        for (size_t i = 0; i < std::min(ks.size(), ps.size()); ++i) g.sweep.emplace_back(ks[i], ps[i]);
    }
    return g;
}

void save_greens_dir(const Greens& g, const std::string& dir) {
    std::filesystem::create_directories(dir);
    Kv man;
    man.put_int("n", g.n);
    man.put_num("pitch", g.pitch);
    man.put_num("phi", g.phi);
    man.put_num("kappa_inf", g.kappa_inf);
    man.put_num("alpha", g.alpha);
    man.put_num("beta", g.beta);
    man.put_num("mu", g.mu);
    man.put_num("capacitance", g.capacitance);
    man.put_num("rand_scale", g.rand_scale);
    man.put_int("tran_count", static_cast<long long>(g.tran.size()));
    if (!g.t_samples.empty()) man.put("t_samples", join_list(g.t_samples));
    man.save(dir + "/manifest.txt");
    Kv cal;
    cal.put_num("c_prime", g.c_prime);
    cal.put_num("fit_r2", g.fit_r2);
    cal.put_num("c", g.c);
    cal.put_num("alpha", g.rep_alpha);
    cal.put_num("cap_residual", g.cap_residual);
    if (!g.sweep.empty()) {
        std::vector<double> ks, ps;
        for (const auto& [k, p] : g.sweep) {
            ks.push_back(k);
            ps.push_back(p);
        }
        cal.put("sweep_conductivity", join_list(ks));
        cal.put("sweep_peak", join_list(ps));
    }
    cal.save(dir + "/calibration.txt");
    write_field(g.f_sp0, dir + "/f_sp0.map");
    write_field(g.g_sp0, dir + "/g_sp0.map");
    write_field(g.f_det, dir + "/f_det.map");
    write_field(g.f_rand, dir + "/f_rand.map");
    write_field(g.p_var, dir + "/p_var.map");
    for (size_t i = 0; i < g.tran.size(); ++i) write_field(g.tran[i], dir + "/" + tran_file(i));
}

// ------------------------------------------------------- stack / variation
void Stack::validate() const {
    if (n < 2) fail(ST_CONFIG, "stack", "grid side must be >= 2");
    if (n % 2 != 0) fail(ST_CONFIG, "stack", "grid side must be even (center impulse)");
    if (!(die_edge > 0.0)) fail(ST_CONFIG, "stack", "die_edge must be positive");
    if (!(ambient > 0.0)) fail(ST_CONFIG, "stack", "ambient must be positive");
    if (!(sink_resistance > 0.0)) fail(ST_CONFIG, "stack", "sink_resistance must be positive");
    const std::pair<const char*, const Layer*> ls[] = {{"die", &die}, {"tim", &tim}, {"spreader", &spreader}};
    for (const auto& [name, l] : ls) {
        if (!(l->thickness > 0.0)) fail(ST_CONFIG, "stack", std::string("layer '") + name + "': thickness must be positive");
        if (!(l->conductivity > 0.0)) fail(ST_CONFIG, "stack", std::string("layer '") + name + "': conductivity must be positive");
        if (!(l->heat_capacity > 0.0)) fail(ST_CONFIG, "stack", std::string("layer '") + name + "': heat capacity must be positive");
    }
}

Stack load_stack_file(const std::string& path) {
    const Kv kv = Kv::parse(path);
    kv.known({"n", "die_edge", "die_thickness", "die_conductivity", "die_heat_capacity", "tim_thickness",
              "tim_conductivity", "tim_heat_capacity", "spreader_thickness", "spreader_conductivity",
              "spreader_heat_capacity", "ambient", "sink_resistance"});
    Stack s;
    s.n = static_cast<int>(kv.integer("n", s.n));
    s.die_edge = kv.num("die_edge", s.die_edge);
    auto layer = [&](const char* name, Layer& l) {
        const std::string p = name;
        l.thickness = kv.num(p + "_thickness", l.thickness);
        l.conductivity = kv.num(p + "_conductivity", l.conductivity);
        l.heat_capacity = kv.num(p + "_heat_capacity", l.heat_capacity);
    };
    layer("die", s.die);
    layer("tim", s.tim);
    layer("spreader", s.spreader);
    s.ambient = kv.num("ambient", s.ambient);
    s.sink_resistance = kv.num("sink_resistance", s.sink_resistance);
    s.validate();
    return s;
}

void save_stack_file(const Stack& s, const std::string& path) {
    Kv kv;
    kv.put_int("n", s.n);
    kv.put_num("die_edge", s.die_edge);
    const std::pair<const char*, const Layer*> ls[] = {{"die", &s.die}, {"tim", &s.tim}, {"spreader", &s.spreader}};
    for (const auto& [name, l] : ls) {
        const std::string p = name;
        kv.put_num(p + "_thickness", l->thickness);
        kv.put_num(p + "_conductivity", l->conductivity);
        kv.put_num(p + "_heat_capacity", l->heat_capacity);
    }
    kv.put_num("ambient", s.ambient);
    kv.put_num("sink_resistance", s.sink_resistance);
    kv.save(path);
}

void VarParams::validate() const {
    if (sigma_sys < 0.0 || sigma_rand < 0.0) fail(ST_CONFIG, "variation", "sigmas must be non-negative");
    if (!(corr_range > 0.0 && corr_range <= 1.0)) fail(ST_CONFIG, "variation", "corr_range must lie in (0, 1]");
    if (!(dopant_spread >= 0.0)) fail(ST_CONFIG, "variation", "dopant_spread must be non-negative");
    if (!(cond_clamp > 0.0 && cond_clamp < 1.0)) fail(ST_CONFIG, "variation", "cond_clamp must lie in (0, 1)");
}

VarParams load_var_file(const std::string& path) {
    const Kv kv = Kv::parse(path);
    kv.known({"sigma_sys", "sigma_rand", "corr_range", "seed", "beta", "beta_L", "beta_tox", "dopant_spread",
              "eta", "cond_clamp", "exponent_cap"});
    VarParams p;
    p.sigma_sys = kv.num("sigma_sys", p.sigma_sys);
    p.sigma_rand = kv.num("sigma_rand", p.sigma_rand);
    p.corr_range = kv.num("corr_range", p.corr_range);
    p.seed = static_cast<uint64_t>(kv.integer("seed", static_cast<long long>(p.seed)));
    p.beta = kv.num("beta", p.beta);
    p.beta_l = kv.num("beta_L", p.beta_l);
    p.beta_tox = kv.num("beta_tox", p.beta_tox);
    p.dopant_spread = kv.num("dopant_spread", p.dopant_spread);
    p.eta = kv.num("eta", p.eta);
    p.cond_clamp = kv.num("cond_clamp", p.cond_clamp);
    p.exponent_cap = kv.num("exponent_cap", p.exponent_cap);
    p.validate();
    return p;
}

void save_var_file(const VarParams& p, const std::string& path) {
    Kv kv;
    kv.put_num("sigma_sys", p.sigma_sys);
    kv.put_num("sigma_rand", p.sigma_rand);
    kv.put_num("corr_range", p.corr_range);
    kv.put_int("seed", static_cast<long long>(p.seed));
    kv.put_num("beta", p.beta);
    kv.put_num("beta_L", p.beta_l);
    kv.put_num("beta_tox", p.beta_tox);
    kv.put_num("dopant_spread", p.dopant_spread);
    kv.put_num("eta", p.eta);
    kv.put_num("cond_clamp", p.cond_clamp);
    kv.put_num("exponent_cap", p.exponent_cap);
    kv.save(path);
}

}  // namespace gth
