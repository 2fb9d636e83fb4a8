// kirchhoff.cuh — inverse Kirchhoff transform of the mode-B / config-4 row passes.
//
// For k = k_ref (T/T0)^-eta (restate.cpp fixed_point_impl, after the reference's
// conductivity refresh, fdm.cpp:187): with ka = T0^(1-eta), kb = (1-eta) T0^-eta and
// br = ka + kb theta, T = br^(1/(1-eta)). Written as
//     T - T0 = T0 expm1(kexp log1p(kc theta)),   kc = kb / ka = (1-eta) / T0,
// it costs log1p + expm1 instead of pow (about a third of the instructions in fp32) and
// returns the rise without the cancellation of br^kexp - T0. br > 0 <=> kc theta > -1.
#pragma once
#include "gt_device.h"

#ifndef GT_KIRCH_POW
#define GT_KIRCH_POW 0
#endif

namespace gtb {

template <typename T>
__device__ __forceinline__ T kirchhoff_rise(T theta, T kc, T kexp, T t_ambient, int& bad) {
    const T u = kc * theta;
    if (!(u > T(-1))) bad |= GTD_ST_KIRCHHOFF;
#if GT_KIRCH_POW  // A/B timing switch: the pow form of the first version
    return pow(T(1) + u, kexp) * t_ambient - t_ambient;
#else
    return t_ambient * expm1(kexp * log1p(u));
#endif
}

}  // namespace gtb
