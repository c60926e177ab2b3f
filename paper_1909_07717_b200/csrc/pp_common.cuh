// pp_common.cuh -- Frame / parameter layouts shared by every kernel, the exact-safe FP32
// filters (ReachBound, ArrivalLB, TrajF) and the bit-exact division helpers.
#pragma once

#include <cstdint>
#include <cstdio>

#include "passplan_b200.h"
#include <math_constants.h>

#include "passplan/detail/pp_math.hpp"

namespace pp {

// Device-side bounds checks of the checked build (-DPP_CHECKED, a verification
// variant: tools/build_variants.sh checked -DPP_CHECKED): a failed check
// prints its site and traps, so a test run on that build fails loudly at the
// first out-of-range index.  Compiled out of the product.
#ifdef PP_CHECKED
#define PP_CHECK(cond)                                                                  \
  do {                                                                                  \
    if (!(cond)) {                                                                      \
      printf("PP_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__,    \
             #cond, static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));        \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
#else
#define PP_CHECK(cond) \
  do {                 \
  } while (0)
#endif

constexpr int kMaxRobots = 32;  // 16 ours + 16 theirs (world.hpp:62)
constexpr int kTheirs = 16;     // slot offset of the opponents

// One world state as the kernels see it.  Teams are id-sorted (dpps.cpp:79-92)
// so slot order == id order; ours at [0,16), theirs at [16,32).
struct __align__(16) FrameDev {
  double px[kMaxRobots], py[kMaxRobots], vx[kMaxRobots], vy[kMaxRobots];
  int32_t id[kMaxRobots];
  double ball_x, ball_y;
  double L, W, gw, dd, dw;
  int32_t n_ours, n_theirs, kicker_slot, n_scan;
  int8_t scan_slot[kMaxRobots];  // robots scanned: ours minus kicker, then theirs
};

struct DevParams {
  double slide, roll, ratio, chip_frac;
  double dt, radius, safety, margin_cap;
  double a_o, b_o, vmax_o, a_t, b_t, vmax_t;
  double pw_t, pw_s, pw_d, pw_r, pw_m;
  double len_upper_cfg, ang_upper;
  double power_min, power_max;
  // Exact squared thresholds (see sqrt_threshold in pp_cabi.cu):
  //   sqrt_rn(x) <  radius        <=>  x <  r_lt2
  //   sqrt_rn(x) <= radius + 1e-9 <=>  x <= mb_le2
  double r_lt2, mb_le2;
  float dtf, radf;  // FP32 copies of dt and radius for the filters
  int32_t n_dirs, n_pows, n_kt, kt_chip0, kt_chip1, n_ptiles, n_tiles;
  // leftover rounds (16- and 8-warp scan shapes): lane-per-cell steps before
  // a (robot, cell) goes to scan_leftovers, and its steps per round there
  int32_t scan_steps, scan_round_steps;
  // Verification switch (pp_ctx_set_option PP_OPT_EXACT_ONLY): every FP32
  // filter passes through -- no reach / lower-bound rejects, no skip-ahead,
  // no upper-bound accepts, no FP32 window prunes, no FP32 / band shortcuts
  // in goal_view -- so every in-window sample takes the exact FP64 test.
  int32_t exact_only;
  // World-independent tables built on the host (pp_cabi.cu ensure_tables):
  const double4* dirs;      // [n_dirs] raw (x, y) and unit (x, y), dpps.cpp:37-48, 120-122
  const struct PowRow* pows;  // [n_kt][n_pows] trajectory per kick slot and power
  // The frames' RobotK[kMaxRobots] each (robot_consts: on the host with a
  // single frame, by robot_consts_kernel for batches), else nullptr
  // (computed per tile).
  const void* rk_pre;
  // Single-frame launches: queue entries written per value chunk (scan ->
  // value streaming: a chunk's CTA starts once its 32 entries are in, while
  // the scan's last tiles still run), else nullptr (value waits for the grid).
  unsigned* chunk_fill;
  // 1: the single frame and its robots' filter constants come in the
  // kernels' FrameArg parameter (no copy: the call graph updates the kernel
  // nodes' parameters), 0: from `frames` / rk_pre in global memory.
  int32_t frame_in_arg;
  // scan_warp_kernel: CTAs per frame (each runs every scan_groups-th tile)
  int32_t scan_groups;
  // Batches: cross_cap(k) for k < n_xcap (xcap_table_kernel), else nullptr
  const int32_t* xcap;
  int32_t n_xcap, pad4;
  // Batches: the frame fold writes this compact per-frame result (indexed
  // like the launch's frames) instead of the full pp_dpps_summary.
  pp_frame_summary* compact;
};

// resolve_kick(power_table[p], kick type) and its sample counts, computed on
// the host with the same correctly rounded FP64 operations (ball_model.cpp:
// 12-43, dpps.cpp:50-62, intercept.cpp:47-69): the scan window start `kb`
// (chip: first sample past the airborne stretch) and `count` samples to rest.
struct PowRow {
  double speed, v1, t_se, d_se, t_stop, d_stop;
  int32_t count, kb;
};

struct CellOut {
  double* our_time;
  double* opp_time;
  double* rx;
  double* ry;
  float* score;
  int8_t* our_slot;
  int8_t* opp_slot;
  uint8_t* feasible;
};

// Best (score, cell) per kick slot 0 / 1 of one value chunk, with the
// winner's PassFeatures.
struct __align__(16) Partial {
  double score[2];
  int64_t cell[2];
  double feat[2][5];
  int64_t n_feasible[2];
};

// ---------------------------------------------------------------------------
// Approximate FP32 square root on the MUFU reciprocal square root (~2 ulp).
// Only used inside the slack-protected bounds below: IEEE sqrtf / division
// cost 60-75 cycles of dependent latency on sm_100a, MUFU.RSQ about 40.
// MUFU reciprocal / reciprocal square root without the denormal rescaling
// rsqrtf / __fdividef add (every operand here is a normal number or is
// guarded; values below 1e-30 only ever move a bound by < 1e-15).
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_ftz(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float sqrt_a(float x) { return x > 1e-30f ? x * rsqrt_ftz(x) : 0.f; }

// FP32 reach bound used to skip samples that cannot be feasible.
//
// arrival_given >= t_along = one_d_time_to_rest(va, deff) with |va| <= u = |v|.
// Over va in [-u, u] that time is minimised at va = min(sqrt(2 b deff), u)
// (decreasing in va up to the exact-stop speed, increasing past it), giving
//   m(deff) = sqrt(2 deff / b)              if 2 b deff <= u^2
//           = one_d_time_to_rest(u, deff)   otherwise.
// reach(t) = m^-1(t) is the farthest target the robot could reach AND stop at
// by time t.  d > radius + reach(t) implies arrival > t, so such samples are
// infeasible.  FP32 evaluation error is covered by the 1e-4 relative and 1e-4 m
// absolute slack the caller adds (FP32 sample positions are within ~2e-5 m).
struct ReachBound {
  float u, b, vmax, t_brake, t_c0, d_used, k_tri, c_tri, half_b, u2_2b, inv_2k;
  ReachBound() = default;
  PP_HD ReachBound(float u_, float a, float b_, float vmax_)
      : u(u_), b(b_), vmax(vmax_) {
    t_brake = u / b;
    half_b = 0.5f * b;
    u2_2b = u * u / (2.f * b);
    // triangle profile from v0 = u: t = (peak - u)/a + peak/b
    k_tri = a * b / (a + b);  // peak = (t + u/a) * k_tri
    inv_2k = 1.f / (2.f * k_tri);
    c_tri = u / a;
    t_c0 = (vmax - u) / a + vmax / b;  // peak reaches vmax
    d_used = (vmax * vmax - u * u) / (2.f * a) + vmax * vmax / (2.f * b);
  }
  // Branch-free (lanes of a warp sit in different pieces): every piece is a
  // couple of FMAs, then selects.
  __device__ __forceinline__ float reach(float t) const {
    const float brake = half_b * t * t;
    const float capped = fmaf(vmax, t - t_brake, u2_2b);  // brake to the cap, cruise
    const float peak = (t + c_tri) * k_tri;
    // D = ((a+b) peak^2 - b u^2) / (2ab) = peak^2 / (2 k_tri) - u^2 / (2a)
    const float tri = fmaf(peak * peak, inv_2k, -u * c_tri * 0.5f);
    const float cruise = fmaf(vmax, t - t_c0, d_used);
    const float free_run = t <= t_c0 ? tri : cruise;
    return t <= t_brake ? brake : (u > vmax ? capped : free_run);
  }
};

// Rigorous FP32 lower bound on arrival_given (arrival_math.hpp:49-62).
//
// arrival_given = max(one_d_time_to_rest(va, deff), |vc| / b).  With FP32
// inputs the true va / deff lie in [v_lo, v_hi] x [d_lo, d_hi] (position
// error <= kPosErr, direction error <= 2 kPosErr / d).  one_d_time_to_rest is
// decreasing in v0 and increasing in dist on the forward side of the
// exact-stop line v0^2 = 2 b dist and increasing in v0, decreasing in dist on
// the overshoot side, so its minimum over the box is:
//   box entirely "moving away" (v_hi < 0): at (v_hi, d_lo);
//   box entirely overshooting (v_lo^2 > 2 b d_hi): at (v_lo, d_hi);
//   otherwise >= min_{v0 <= max(v_hi,0)} one_d(v0, d_lo)
//             = sqrt(2 d_lo / b) if it can stop exactly, else forward(U, d_lo).
// The result is scaled by (1 - 3e-5) and shifted by 2e-5 s to absorb the FP32
// evaluation error of these few operations, so L <= exact arrival always.
constexpr float kPosErr = 1e-4f;  // |FP32 sample position error| bound [m]

struct ArrivalLB {
  float vx, vy, u, b, vmax, ia, ib, ivmax, c_peak_d, c_peak_v, half_ib, half_ia, vm2, rr_dused,
      t_vab;
  ArrivalLB() = default;
  PP_HD ArrivalLB(float vx_, float vy_, float u_, float a, float b_,
                                       float vmax_)
      : vx(vx_), vy(vy_), u(u_), b(b_), vmax(vmax_) {
    ia = 1.f / a;
    ib = 1.f / b;
    ivmax = 1.f / vmax;
    c_peak_d = 2.f * a * b / (a + b);  // peak^2 = c_peak_d * dist + c_peak_v * v0^2
    c_peak_v = b / (a + b);
    half_ib = 0.5f * ib;
    half_ia = 0.5f * ia;
    vm2 = vmax * vmax;
    rr_dused = vm2 * half_ia + vm2 * half_ib;
    t_vab = vmax * ia + vmax * ib;
  }
  __device__ __forceinline__ float rest_to_rest(float L) const {
    const float peak = sqrt_a(c_peak_d * L);
    if (peak <= vmax) return peak * (ia + ib);
    return t_vab + (L - rr_dused) * ivmax;
  }
  // min over v0 <= U (U >= 0) of one_d_time_to_rest(v0, d)
  __device__ __forceinline__ float forward_min(float U, float d) const {
    if (U * U >= 2.f * b * d) return sqrt_a(2.f * d * ib);
    const float peak = sqrt_a(fmaf(c_peak_d, d, c_peak_v * U * U));
    if (peak <= vmax) return (peak - U) * ia + peak * ib;
    if (U <= vmax) {
      const float d_used = (vm2 - U * U) * half_ia + vm2 * half_ib;
      return (vmax - U) * ia + vmax * ib + (d - d_used) * ivmax;
    }
    return U * ib + (d - U * U * half_ib) * ivmax;
  }
  // d = |q| and inv_d = 1/|q| (approximate) from the caller's single rsqrt.
  __device__ __forceinline__ float lower_bound(float qx, float qy, float d, float inv_d,
                                               float radius) const {
    const float d_lo = fmaxf(d * (1.f - 1e-6f) - kPosErr - radius, 0.f);
    const float d_hi = fmaxf(d * (1.f + 1e-6f) + kPosErr - radius, 0.f);
    float va = 0.f, vc = 0.f, dv = u;  // unknown direction near the robot
    if (d > 10.f * kPosErr) {
      va = (vx * qx + vy * qy) * inv_d;
      vc = (vx * qy - vy * qx) * inv_d;
      dv = u * (2.f * kPosErr * inv_d + 1e-5f) + 1e-6f;
    }
    const float v_lo = va - dv, v_hi = va + dv;
    float t_along;
    // rest_to_rest is increasing in its argument and ~sqrt near 0, so the
    // arguments are rounded DOWN by a relative + absolute slack first.
    if (v_hi < 0.f) {
      const float g = fmaf(v_hi * v_hi, half_ib, d_lo);
      t_along = -v_hi * ib + rest_to_rest(fmaxf(fmaf(g, -1e-5f, g) - 1e-6f, 0.f));
    } else if (v_lo > 0.f && v_lo * v_lo > 2.f * b * d_hi) {
      const float e2 = v_lo * v_lo * half_ib;
      const float g = e2 - d_hi - 1e-5f * (e2 + d_hi) - 1e-6f;
      t_along = v_lo * ib + rest_to_rest(fmaxf(g, 0.f));
    } else {
      t_along = forward_min(v_hi, d_lo);
    }
    const float t_cross = fmaxf(fabsf(vc) - dv, 0.f) * ib;
    return fmaf(fmaxf(t_along, t_cross), 1.f - 3e-5f, -2e-5f);
  }
  // forward-regime time one_d_time_to_rest(v0, d) for 0 <= v0, v0^2 <= 2 b d
  __device__ __forceinline__ float forward(float v0, float d) const {
    const float peak = sqrt_a(fmaf(c_peak_d, d, c_peak_v * v0 * v0));
    if (peak <= vmax) return (peak - v0) * ia + peak * ib;
    if (v0 <= vmax) {
      const float d_used = (vm2 - v0 * v0) * half_ia + vm2 * half_ib;
      return (vmax - v0) * ia + vmax * ib + (d - d_used) * ivmax;
    }
    return v0 * ib + (d - v0 * v0 * half_ib) * ivmax;
  }
  // Rigorous upper bound (mirror of lower_bound): the maximum of
  // one_d_time_to_rest over the same box is attained at (v_lo, d_hi) on the
  // wrong-way and forward sides and at (v_hi, d_lo) on the overshoot side.
  __device__ __forceinline__ float upper_bound(float qx, float qy, float d, float inv_d,
                                               float radius) const {
    if (!(d > 10.f * kPosErr)) return 1e30f;  // direction unknown: no claim
    const float d_lo = fmaxf(d * (1.f - 1e-6f) - kPosErr - radius, 0.f);
    const float d_hi = fmaxf(d * (1.f + 1e-6f) + kPosErr - radius, 0.f);
    const float va = (vx * qx + vy * qy) * inv_d;
    const float vc = (vx * qy - vy * qx) * inv_d;
    const float dv = u * (2.f * kPosErr * inv_d + 1e-5f) + 1e-6f;
    const float v_lo = va - dv, v_hi = va + dv;
    float t = 0.f;
    if (v_lo < 0.f) {  // wrong way: |v0|/b + rest_to_rest(v0^2/2b + d), max at (v_lo, d_hi)
      const float g = fmaf(v_lo * v_lo, half_ib, d_hi);
      t = fmaxf(t, -v_lo * ib + rest_to_rest(fmaf(g, 1e-5f, g) + 1e-6f));
    }
    const float vf = fmaxf(v_lo, 0.f);
    if (vf * vf <= 2.f * b * d_hi) t = fmaxf(t, forward(vf, d_hi));
    if (v_hi > 0.f && v_hi * v_hi > 2.f * b * d_lo) {  // overshoot, max at (v_hi, d_lo)
      const float e2 = v_hi * v_hi * half_ib;
      const float g = e2 - d_lo + 1e-5f * (e2 + d_lo) + 1e-6f;
      t = fmaxf(t, v_hi * ib + rest_to_rest(g));
    }
    const float t_cross = (fabsf(vc) + dv) * ib;
    return fmaf(fmaxf(t, t_cross), 1.f + 3e-5f, 2e-5f);
  }
};

// FP32 copy of the trajectory for the filter's sample positions.
struct TrajF {
  float speed, v1, t_se, d_se, t_stop, d_stop, hs, hr;
  TrajF() = default;
  __device__ __forceinline__ TrajF(const Traj& tr, float slide, float roll)
      : speed(static_cast<float>(tr.speed.v)), v1(static_cast<float>(tr.v1.v)),
        t_se(static_cast<float>(tr.t_se.v)), d_se(static_cast<float>(tr.d_se.v)),
        t_stop(static_cast<float>(tr.t_stop.v)), d_stop(static_cast<float>(tr.d_stop.v)),
        hs(0.5f * slide), hr(0.5f * roll) {}
  // Both pieces, then selects (lanes of a warp sit in different pieces:
  // C5 batch scan -0.6 % against the branches).
  __device__ __forceinline__ float speed_at(float t) const {  // ball_model.cpp:77-81
    const float a = speed - 2.f * hs * t, b = v1 - 2.f * hr * (t - t_se);
    return t < t_se ? a : (t < t_stop ? b : 0.f);
  }
  __device__ __forceinline__ float distance_at(float t) const {
    const float w = t - t_se;
    const float a = t * (speed - hs * t), b = d_se + w * (v1 - hr * w);
    return t < t_se ? a : (t < t_stop ? b : d_stop);
  }
};

}  // namespace pp
