// passplan/kernels/kernel.hpp -- the reference's per-pair scan plug-in point
// (proj/include/passplan/kernels/kernel.hpp:10-60): the same RobotKin /
// ScanBatch types, the same inline sample_feasible (through the shared
// restatement pp_math.hpp), and a backend registry whose one entry is the
// B200 backend "sm100a": its scan_first runs on the GPU (pp_scan_first, one
// warp per pair).  The planner itself never calls through this interface --
// a call is one (trajectory, robot) pair, far below a kernel launch -- run_dpps
// replaces the layer above it and reports this backend's name in
// DppsTelemetry::kernel.  The reference's CPU backends (scalar_kernel,
// avx2_kernel) are not provided: there is no CPU path.
#pragma once

#include <vector>

#include "passplan/detail/arrival_math.hpp"

namespace passplan::kernels {

struct RobotKin {
  double px = 0.0, py = 0.0;
  double vx = 0.0, vy = 0.0;
  double accel = 0.0, decel = 0.0, vmax = 0.0;
  double radius = 0.0;
  double vbound = 0.0;  // max(vmax, |v|)
};

struct ScanBatch {
  const double* ts = nullptr;
  const double* ss = nullptr;
  int k_begin = 0;
  int k_end = 0;  // exclusive
  double ox = 0.0, oy = 0.0;
  double ux = 0.0, uy = 0.0;
};

// The reference's exact sample test (kernel.hpp:33-44): the quick reject on
// radius + vbound t, then arrival_given <= t.
inline bool sample_feasible(const ScanBatch& b, const RobotKin& r, int k) {
  const double t = b.ts[k];
  const double s = b.ss[k];
  const pp::xd px = pp::xd(b.ox) + pp::xd(b.ux) * s, py = pp::xd(b.oy) + pp::xd(b.uy) * s;
  const pp::xd qx = px - r.px, qy = py - r.py;
  const pp::xd d2 = qx * qx + qy * qy;
  const pp::xd reach = pp::xd(r.radius) + pp::xd(r.vbound) * t;
  if (d2 > reach * reach) return false;
  return detail::arrival_given(qx.v, qy.v, d2.v, r.vx, r.vy, r.accel, r.decel, r.vmax,
                               r.radius) <= t;
}

// Smallest k in [k_begin, k_end) whose sample the robot can intercept, or -1.
using ScanFn = int (*)(const ScanBatch&, const RobotKin&);

struct KernelBackend {
  const char* name;
  ScanFn scan_first;
};

const KernelBackend& sm100a_kernel();                     // the B200 backend
const KernelBackend& active_kernel();                     // == sm100a_kernel()
std::vector<const KernelBackend*> available_kernels();  // {&sm100a_kernel()}

}  // namespace passplan::kernels
