// gt_ops.h — host orchestration of the reference-API solves (steady, step,
// trace, Monte Carlo, calibration) over the device kernels.
#pragma once

#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "host.hpp"

// Prepared device GreensSet of one gt_greens handle (the reference rebuilds its
// PreparedGreens on every gt_solve_* call, capi.cpp:196,210,247; here it is built on
// the first call and reused). Calls on one handle serialise on `mu`.
struct GtSolveCache;
struct GtSolveSlot {
    std::mutex mu;
    std::shared_ptr<GtSolveCache> cache;
};

void gt_ops_modal_kernel(const gth::Stack& s, double* out_host);
gth::Field gt_ops_oracle_steady(const gth::Stack& stack, const gth::VarParams* var, const gth::Field& p_dyn,
                                const gth::Field* nominal_leak, int temp_dep_leakage, int temp_dep_conductivity,
                                int* outer_iterations);
std::vector<gth::Field> gt_ops_oracle_transient(const gth::Stack& stack, const gth::VarParams* var,
                                                const gth::Field& p_dyn, const gth::Field* nominal_leak,
                                                int temp_dep_leakage, const std::vector<double>& times, double dt);
gth::Greens gt_ops_calibrate_modal(const gth::Stack& s, const gth::VarParams& v, const gth::Field* nominal_leak,
                                   double leak_total);
gth::Field gt_ops_steady(const gth::Greens& g, GtSolveSlot& slot, const gth::Field& p_dyn, bool with_rand,
                         double* online_ms);
std::vector<gth::Field> gt_ops_step(const gth::Greens& g, GtSolveSlot& slot, const gth::Field& p_dyn,
                                    const std::vector<double>& times, bool with_rand, double* online_ms);
void gt_ops_check_trace(double dt, const std::vector<gth::Field>& frames);
std::vector<gth::Field> gt_ops_trace(const gth::Greens& g, GtSolveSlot& slot, double dt,
                                     const std::vector<gth::Field>& frames, int window, bool with_rand,
                                     std::vector<double>* times, double* online_ms);
void gt_ops_monte_carlo(const gth::Greens& g, const gth::VarParams& v, const gth::Field& nominal_leak,
                        const gth::Field& p_dyn, const std::vector<unsigned long long>& seeds, int jobs,
                        const std::string& csv_path, double* mean_max, double* std_max);
