// host.hpp — host-side data model of the drop-in library: grids, key-value
// files, GreensSet directories and the error taxonomy, mirroring the
// reference's L1 layer (field.hpp:23-69, kvfile.hpp:14-43, greens.hpp:18-39,
// errors.hpp:12-45) so the C ABI reads and writes the reference's own files.
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace gth {

// gt_status values (reference greentherm.h:16-22).
enum Status { ST_OK = 0, ST_CONFIG = 2, ST_SOLVER = 3, ST_VALIDATION = 4, ST_INTERNAL = 5 };

// One exception type carrying the status class and the pipeline stage
// (the reference uses a class hierarchy mapped by capi.cpp:25-34).
struct Error : std::runtime_error {
    Status status;
    std::string stage;
    Error(Status s, std::string st, const std::string& msg)
        : std::runtime_error(msg), status(s), stage(std::move(st)) {}
};
[[noreturn]] void fail(Status s, const std::string& stage, const std::string& msg);

enum class Unit { Watts, Kelvin, KelvinPerWatt, Dimensionless };
const char* unit_str(Unit u);
Unit parse_unit(const std::string& s);

struct Field {
    int n = 0;
    double pitch = 0.0;
    Unit unit = Unit::Dimensionless;
    std::vector<double> v;

    Field() = default;
    Field(int n_, double pitch_, Unit u, double fill = 0.0);
    double& at(int i, int j) { return v[static_cast<size_t>(i) * n + j]; }
    double at(int i, int j) const { return v[static_cast<size_t>(i) * n + j]; }
    double max() const;
    double min() const;
    double sum() const;  // Neumaier compensated (reference field.cpp:45-57)
    std::pair<int, int> argmax() const;
    bool same_shape(const Field& o) const { return n == o.n && pitch == o.pitch; }
    void check_finite(const char* what) const;
};

Field read_field(const std::string& path);
void write_field(const Field& f, const std::string& path);

class Kv {
public:
    static Kv parse(const std::string& path);
    bool has(const std::string& k) const { return m_.count(k) != 0; }
    std::string str(const std::string& k) const;
    double num(const std::string& k) const;
    double num(const std::string& k, double dflt) const { return has(k) ? num(k) : dflt; }
    long long integer(const std::string& k) const;
    long long integer(const std::string& k, long long dflt) const { return has(k) ? integer(k) : dflt; }
    std::vector<double> list(const std::string& k) const;
    void put(const std::string& k, const std::string& v) { m_[k] = v; }
    void put_num(const std::string& k, double v);
    void put_int(const std::string& k, long long v) { m_[k] = std::to_string(v); }
    void known(const std::vector<std::string>& keys) const;
    void save(const std::string& path) const;

private:
    std::string origin_;
    std::map<std::string, std::string> m_;
};

struct Greens {
    int n = 0;
    double pitch = 0.0;
    Field f_sp0, g_sp0, f_det, f_rand, p_var;
    double phi = 0.0, kappa_inf = 0.0, alpha = 0.0, beta = 0.0, mu = 0.0;
    double capacitance = 0.0, rand_scale = 1.0;
    std::vector<double> t_samples;
    std::vector<Field> tran;
    // calibration report (reference greens.hpp:41-48)
    double c_prime = 0.0, fit_r2 = 0.0, c = 0.0, rep_alpha = 0.0, cap_residual = 0.0;
    std::vector<std::pair<double, double>> sweep;

    int center() const { return n / 2; }
    void validate() const;  // reference greens.cpp:96-106
};

Greens load_greens_dir(const std::string& dir);
void save_greens_dir(const Greens& g, const std::string& dir);

// Reference stack / variation parameter files (stack.hpp:17-26, variation.hpp:13-27).
struct Layer {
    double thickness, conductivity, heat_capacity;
};
struct Stack {
    double die_edge = 0.01;
    Layer die{0.15e-3, 130.0, 1.75e6}, tim{0.02e-3, 4.0, 4.0e6}, spreader{3.5e-3, 400.0, 3.55e6};
    double ambient = 318.15, sink_resistance = 0.25;
    int n = 64;
    double pitch() const { return die_edge / n; }
    void validate() const;
};
Stack load_stack_file(const std::string& path);
void save_stack_file(const Stack& s, const std::string& path);

struct VarParams {
    double sigma_sys = 0.025, sigma_rand = 0.015, corr_range = 0.5;
    uint64_t seed = 1;
    double beta = 0.0275, beta_l = -10.0, beta_tox = -5.0, dopant_spread = 0.05, eta = 1.3;
    double cond_clamp = 0.3, exponent_cap = 6.0;
    void validate() const;
};
VarParams load_var_file(const std::string& path);
void save_var_file(const VarParams& p, const std::string& path);

}  // namespace gth
