// passplan/detail/arrival_math.hpp -- the reference's scalar arrival-time
// math (proj/include/passplan/detail/arrival_math.hpp:15-69) under its own
// names, forwarding to the one shared restatement in pp_math.hpp (the same
// expression trees the sm_100a kernels evaluate; host code is compiled with
// -ffp-contract=off, so the results are bit-identical to the reference's).
#pragma once

#include "passplan/detail/pp_math.hpp"

namespace passplan::detail {

inline double rest_to_rest_time(double L, double a, double b, double vmax) {
  return pp::rest_to_rest_time(L, a, b, vmax).v;
}

inline double one_d_time_to_rest(double v0, double dist, double a, double b, double vmax) {
  return pp::one_d_time_to_rest(v0, dist, a, b, vmax).v;
}

inline double arrival_given(double qx, double qy, double d2, double vx, double vy, double a,
                            double b, double vmax, double radius) {
  return pp::arrival_given(qx, qy, d2, vx, vy, a, b, vmax, radius).v;
}

inline double arrival_to_point(double tx, double ty, double px, double py, double vx, double vy,
                               double a, double b, double vmax, double radius) {
  return pp::arrival_to_point(tx, ty, px, py, vx, vy, a, b, vmax, radius).v;
}

}  // namespace passplan::detail
