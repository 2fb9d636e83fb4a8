// dropin_demo.cpp -- a host program written against the reference C ABI only
// (include/greentherm.h, the reference's own header surface), built twice by
// tests/test_dropin_gpu.py: linked against the reference library compiled from its
// unchanged sources (oracle/_ref/libgreentherm_ref.so) and against
// libgreentherm_b200.so. Same source, same calls, no code change: the outputs must agree.
//
// usage: dropin_demo GREENS_DIR VARIATION_FILE POWER_MAP OUT_PREFIX
#include <cstdio>
#include <cstdlib>
#include <string>

#include "greentherm.h"

static int check(gt_status s, const char* what) {
    if (s != GT_OK) {
        std::fprintf(stderr, "error stage=%s status=%s msg=\"%s\" (%s)\n", gt_last_error_stage(), gt_status_name(s),
                     gt_last_error(), what);
        std::exit(1);
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 5) return 2;
    const std::string prefix = argv[4];
    gt_greens* g = nullptr;
    check(gt_greens_load(argv[1], &g), "greens load");
    gt_field* p = nullptr;
    check(gt_field_load(argv[3], &p), "power load");
    double online = 0.0;
    for (int with_rand = 0; with_rand < 2; ++with_rand) {
        gt_field* t = nullptr;
        check(gt_solve_steady(g, p, with_rand, &t, &online), "steady");
        check(gt_field_save(t, (prefix + (with_rand ? "steady_rand.map" : "steady.map")).c_str()), "save");
        const int n = gt_field_n(t);
        std::printf("steady with_rand=%d max=%.12f mean=%.12f\n", with_rand, gt_field_max(t),
                    gt_field_sum(t) / (double(n) * n));
        gt_field_free(t);
    }
    const unsigned long long seeds[6] = {1, 2, 3, 5, 8, 13};
    double mean_max = 0.0, std_max = 0.0;
    check(gt_monte_carlo(g, argv[2], nullptr, 20.0, p, seeds, 6, 4, (prefix + "mc.csv").c_str(), &mean_max, &std_max),
          "monte carlo");
    std::printf("monte_carlo mean_max=%.12f std_max=%.12f\n", mean_max, std_max);
    gt_field_free(p);
    gt_greens_free(g);
    return 0;
}
