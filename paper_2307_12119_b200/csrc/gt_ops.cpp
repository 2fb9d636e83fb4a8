// gt_ops.cpp — host orchestration of the reference-API solves.
#include "gt_ops.h"

using namespace gth;

void gt_ops_check_trace(double dt, const std::vector<Field>& frames) {
    // reference solver.cpp:74-83
    if (frames.empty()) fail(ST_CONFIG, "solver", "power trace is empty");
    if (!(dt > 0.0)) fail(ST_CONFIG, "solver", "power trace dt must be positive");
    for (const Field& f : frames) {
        if (!f.same_shape(frames.front())) fail(ST_CONFIG, "solver", "power trace frames differ in shape");
        f.check_finite("trace frame");
        if (f.min() < 0.0) fail(ST_CONFIG, "solver", "trace powers must be >= 0");
    }
}

Greens gt_ops_calibrate_modal(const Stack&, const VarParams&, const Field*, double) {
    fail(ST_INTERNAL, "calibrate", "device calibration not built yet");
}
Field gt_ops_steady(const Greens&, const Field&, bool, double*) {
    fail(ST_INTERNAL, "solver", "steady path not built yet");
}
std::vector<Field> gt_ops_step(const Greens&, const Field&, const std::vector<double>&, bool, double*) {
    fail(ST_INTERNAL, "solver", "step path not built yet");
}
std::vector<Field> gt_ops_trace(const Greens&, double, const std::vector<Field>&, int, bool, std::vector<double>*,
                                double*) {
    fail(ST_INTERNAL, "solver", "trace path not built yet");
}
void gt_ops_monte_carlo(const Greens&, const VarParams&, const Field&, const Field&,
                        const std::vector<unsigned long long>&, int, const std::string&, double*, double*) {
    fail(ST_INTERNAL, "solver", "monte carlo path not built yet");
}
