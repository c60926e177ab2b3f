// pp_intercept.cuh -- intercept_kernel / shot_kernel: intercept_all over one trajectory
// (intercept.cpp:154-196) for possession and decide_shot.
#pragma once

#include "pp_value.cuh"

namespace pp {

// ---------------------------------------------------------------------------
// Standalone interception of one trajectory: intercept_time / intercept_all
// (intercept.cpp:154-196), used by possession (pass_eval.cpp:271-298) and
// decide_shot (pass_eval.cpp:194-233).  One warp per robot; the 32 lanes test
// 32 consecutive samples per step (possession samples at 1 ms, thousands of
// samples per robot), the first sample not rejected by the FP32 filters gets
// the exact FP64 test, and the rest rule applies when none hits
// (intercept.cpp:121-150).
// BallPath / make_path: passplan/detail/pp_math.hpp (shared with the host).

// scan_window (intercept.cpp:47-69) of a path sampled at dt.
__device__ __forceinline__ void path_window(const BallPath& B, const FrameDev& F, xd dt,
                                            int* kb_out, int* ke_out, bool* rif_out) {
  const Traj& tr = B.tr;
  const xd slide = B.slide, roll = B.roll;
  const int count = static_cast<int>(floor((tr.t_stop / dt + xd(1e-9)).v)) + 1;
  const xd d_exit = ray_exit_distance(F.L, F.W, B.ox, B.oy, B.ux, B.uy);
  int kb = 0, ke = 0;
  bool rif = false;
  if (!isnan(d_exit.v)) {
    ke = count;
    if (d_exit < tr.d_stop) {
      const xd t_exit = travel_time_to_distance(tr, slide, roll, d_exit);
      const int k_last =
          !isnan(t_exit.v) ? static_cast<int>(floor((t_exit / dt + xd(1e-9)).v)) : count - 1;
      ke = ke < k_last + 1 ? ke : k_last + 1;
    } else {
      rif = true;
    }
    if (tr.from.v > 0.0) {
      const xd t_air = travel_time_to_distance(tr, slide, roll, tr.from);
      if (!isnan(t_air.v)) kb = static_cast<int>(ceil((t_air / dt - xd(1e-9)).v));
    }
  }
  *kb_out = kb;
  *ke_out = ke;
  *rif_out = rif;
}

struct InterceptOut {
  int32_t finite, pad;
  double time, px, py;
};

// intercept_with (intercept.cpp:121-150) for scanned robot `ri` of F, whole
// warp.  Result valid in every lane.
__device__ __forceinline__ InterceptOut intercept_warp(const BallPath& B, int kb, int ke, bool rif,
                                                       const FrameDev& F, const DevParams& P,
                                                       const RobotK& rk, int ri, xd dt) {
  const int lane = threadIdx.x & 31;
  const xd slide = B.slide, roll = B.roll, radius = P.radius;
  const int slot = F.scan_slot[ri];
  const bool theirs = slot >= kTheirs;
  const xd rpx = F.px[slot], rpy = F.py[slot], rvx = F.vx[slot], rvy = F.vy[slot];
  const xd a = theirs ? P.a_t : P.a_o;
  const xd b = theirs ? P.b_t : P.b_o;
  const xd vmax = theirs ? P.vmax_t : P.vmax_o;
  const xd vbound = rk.vbound;
  const ReachBound& rb = rk.rb;
  const ArrivalLB& lb = rk.lb;
  const Traj& tr = B.tr;
  const xd ox = B.ox, oy = B.oy, ux = B.ux, uy = B.uy;
  const float dtf = static_cast<float>(dt.v);
  const float radf = static_cast<float>(radius.v);
  const float vbf = static_cast<float>(vbound.v);
  const float bxf = static_cast<float>((ox - rpx).v);
  const float byf = static_cast<float>((oy - rpy).v);
  const float uxf = static_cast<float>(ux.v), uyf = static_cast<float>(uy.v);
  const float s0 = -(bxf * uxf + byf * uyf);
  const TrajF trf(tr, static_cast<float>(slide.v), static_cast<float>(roll.v));
  int hit = -1;
  int k0 = kb;
  int guard = 0;
  while (k0 < ke) {
    // lane j: sample k0 + j.  0 rejected (next sample to look at in nx),
    // 1 window end, 2 certainly feasible, 3 needs the exact test.
    const int kk = k0 + lane;
    int code = 1, nx = kk + 1;
    if (kk < ke && P.exact_only) {
      code = 3;  // verification switch: the exact test for every sample
    } else if (kk < ke) {
      const float tf = static_cast<float>(kk) * dtf;
      const float sf = trf.distance_at(tf);
      const float qxf = fmaf(uxf, sf, bxf);
      const float qyf = fmaf(uyf, sf, byf);
      const float d2f = fmaf(qxf, qxf, qyf * qyf);
      const float thr = radf + fmaf(rb.reach(tf), 1.0001f, 1e-4f);
      const float inv_d = rsqrt_ftz(fmaxf(d2f, 1e-30f));
      const float df = d2f * inv_d;
      if (d2f > thr * thr) {
        const float gap = df - thr;
        const float approach = sf < s0 + 1e-3f ? trf.speed_at(tf) : 0.f;
        const float rate = (approach + vbf) * dtf * 1.0001f;
        const float j = floorf(gap * rcp_ftz(rate) * 0.9999f);
        nx = kk + 1 + (j > 1.f ? (j < 1048576.f ? static_cast<int>(j) - 1 : 1048575) : 0);
        code = 0;
      } else if (lb.lower_bound(qxf, qyf, df, inv_d, radf) > fmaf(tf, 1.000001f, 1e-6f)) {
        code = 0;
      } else if (lb.upper_bound(qxf, qyf, df, inv_d, radf) < fmaf(tf, 0.999999f, -1e-6f)) {
        code = 2;
      } else {
        code = 3;
      }
    }
    const unsigned nonrej = __ballot_sync(0xffffffffu, code != 0);
    if (nonrej == 0u) {  // all 32 rejected: continue past everything they certified
      int far = nx;
      for (int o = 16; o > 0; o >>= 1) far = max(far, __shfl_xor_sync(0xffffffffu, far, o));
      k0 = far;
    } else {
      const int f = __ffs(nonrej) - 1;
      const int cf = __shfl_sync(0xffffffffu, code, f);
      const int kf = k0 + f;
      if (cf == 1) break;
      if (cf == 2) {
        hit = kf;
        break;
      }
      // exact reference test (kernel.hpp:33-44), one lane
      int pass = 0;
      if (lane == f) {
        const xd t = xd(double(kf)) * dt;
        const xd sx = distance_at(tr, slide, roll, t);
        const xd qx = (ox + ux * sx) - rpx;
        const xd qy = (oy + uy * sx) - rpy;
        const xd d2 = qx * qx + qy * qy;
        const xd reach = radius + vbound * t;
        pass = !(d2 > reach * reach) && arrival_given(qx, qy, d2, rvx, rvy, a, b, vmax, radius) <= t;
      }
      pass = __shfl_sync(0xffffffffu, pass, f);
      if (pass) {
        hit = kf;
        break;
      }
      k0 = kf + 1;
    }
    if (++guard > (1 << 24)) __trap();
  }
  InterceptOut r{0, 0, 0.0, 0.0, 0.0};
  if (hit >= 0) {
    const xd t = xd(double(hit)) * dt;
    const xd s = distance_at(tr, slide, roll, t);
    r.finite = 1;
    r.time = t.v;
    r.px = (ox + ux * s).v;
    r.py = (oy + uy * s).v;
  } else if (rif) {
    const xd rx = ox + ux * tr.d_stop, ry = oy + uy * tr.d_stop;
    const xd arr = arrival_to_point(rx, ry, rpx, rpy, rvx, rvy, a, b, vmax, radius);
    r.finite = 1;
    r.time = (arr > tr.t_stop ? arr : tr.t_stop).v;
    r.px = rx.v;
    r.py = ry.v;
  }
  return r;
}

// intercept_all: every scanned robot of the frame against one path.
__global__ void __launch_bounds__(1024) intercept_kernel(const FrameDev* __restrict__ frame,
                                                         DevParams P, BallPath B, double dt,
                                                         InterceptOut* __restrict__ out) {
  __shared__ FrameDev F;
  __shared__ RobotK rk[kMaxRobots];
  load_frame(&F, frame);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0)
    for (int ri = lane; ri < F.n_scan; ri += 32) robot_consts(F, P, ri, &rk[ri]);
  __syncthreads();
  int kb, ke;
  bool rif;
  path_window(B, F, dt, &kb, &ke, &rif);
  for (int ri = warp; ri < F.n_scan; ri += blockDim.x >> 5) {
    const InterceptOut r = intercept_warp(B, kb, ke, rif, F, P, rk[ri], ri, dt);
    PP_CHECK(ri < kMaxRobots);
    if (lane == 0) out[ri] = r;
  }
}

// decide_shot (pass_eval.cpp:194-233): goal view from the origin, flat shot
// at shot_speed toward the view target, opponents (the frame's scan list)
// intercept it at sbip_dt before it reaches the line?
__global__ void __launch_bounds__(512) shot_kernel(const FrameDev* __restrict__ frame,
                                                   DevParams P, double ox, double oy,
                                                   double shot_speed, double angle_threshold,
                                                   pp_shot_decision* __restrict__ out) {
  __shared__ FrameDev F;
  __shared__ RobotK rk[kMaxRobots];
  __shared__ View view;
  __shared__ __align__(16) unsigned char b_raw[sizeof(BallPath)];  // (xd has a constructor)
  BallPath& B = *reinterpret_cast<BallPath*>(b_raw);
  __shared__ double t_goal;
  __shared__ int stage;  // 0 go on, 1 decided
  __shared__ double t_min;
  load_frame(&F, frame);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    view = goal_view_thread(ox, oy, F, P.radius, P.r_lt2, P.mb_le2, P.exact_only != 0);
    const xd gx = xd(0.5) * xd(F.L);
    pp_shot_decision d{};
    d.shot_angle = view.angle;
    d.target_x = gx.v;
    d.target_y = view.ty;
    stage = 0;
    t_min = CUDART_INF;
    if (view.angle < angle_threshold || view.angle <= 0.0) {
      d.reason = 0;  // ShotReason::angle_too_small
      d.blocked = 1;
      stage = 1;
    } else {
      B = make_path(ox, oy, gx - xd(ox), xd(view.ty) - xd(oy), shot_speed, false, true, P.slide,
                    P.roll, P.ratio, P.chip_frac);
      const xd goal_dist = dist2d(ox, oy, gx, view.ty);
      t_goal = travel_time_to_distance(B.tr, B.slide, B.roll, goal_dist).v;
      if (isnan(t_goal)) {  // the shot dies before the line
        d.reason = 1;       // ShotReason::interceptable
        d.blocked = 1;
        stage = 1;
      }
    }
    *out = d;
  }
  if (warp == 1)
    for (int ri = lane; ri < F.n_scan; ri += 32) robot_consts(F, P, ri, &rk[ri]);
  __syncthreads();
  if (stage) return;
  int kb, ke;
  bool rif;
  path_window(B, F, P.dt, &kb, &ke, &rif);
  for (int ri = warp; ri < F.n_scan; ri += blockDim.x >> 5) {
    const InterceptOut r = intercept_warp(B, kb, ke, rif, F, P, rk[ri], ri, P.dt);
    if (lane == 0 && r.finite) atomicMin(reinterpret_cast<unsigned long long*>(&t_min),
                                         static_cast<unsigned long long>(__double_as_longlong(r.time)));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // any opponent strictly earlier than the ball at the line (times >= 0, so
    // the unsigned bit-pattern minimum is the numeric minimum)
    if (t_min < t_goal) {
      out->reason = 1;
      out->blocked = 1;
    } else {
      out->shoot = 1;
      out->reason = 2;  // ShotReason::clear
    }
  }
}

}  // namespace pp
