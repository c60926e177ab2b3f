// pp_runmap.cuh -- runmap_kernel: the running-point map and best_running_points
// (offball.cpp:17-258).
#pragma once

#include "pp_intercept.cuh"

namespace pp {

// ---------------------------------------------------------------------------
// Running-point map (offball.cpp:17-258).

struct RunZone {
  double x0, y0, ydir;  // lattice anchors: x = x0 + i*step, y = y0 + ydir*(j*step)
  int32_t nx, ny;
  int64_t offset;       // first vertex in the map
  int32_t selected;     // zone takes part in best_running_points
  int32_t in_map;       // zone is rasterised into the per-vertex map
};

struct RunParams {
  double step, L, W, dd, dw, gw;
  double ball_x, ball_y;
  double a_t, b_t, vmax_t, cap;
  double w_dg, w_db, w_angle, w_guard, w_exp;
  double len_upper;
  double band_full_lo, band_peak_lo, band_peak_hi, band_full_hi;
  double nearest_opp;          // min_opp |opp - ball| (point independent)
  double g_px[2], g_py[2], g_vx[2], g_vy[2];  // the two ranked guards
  int32_t n_guards;
  int32_t blocks_per_zone[4];
  int32_t pad;
  RunZone zone[4];
};

struct __align__(16) RunPartial {
  double score;
  int64_t index;  // linear (i*ny + j) within the zone; -1 = none
  double px, py;
  double feat[5];
};

__device__ __forceinline__ xd band_value(const RunParams& R, xd a) {
  const xd full_lo = R.band_full_lo, peak_lo = R.band_peak_lo, peak_hi = R.band_peak_hi,
           full_hi = R.band_full_hi;
  if (a < full_lo || a > full_hi) return 0.0;
  if (a < peak_lo) {
    const xd w = peak_lo - full_lo;
    return w.v > 0.0 ? (a - full_lo) / w : xd(1.0);
  }
  if (a > peak_hi) {
    const xd w = full_hi - peak_hi;
    return w.v > 0.0 ? (full_hi - a) / w : xd(1.0);
  }
  return 1.0;
}

// entry_param (offball.cpp:31-51)
__device__ __forceinline__ xd entry_param(xd bx0, xd bx1, xd by0, xd by1, xd ax, xd ay, xd bx,
                                          xd by) {
  xd t_enter = -CUDART_INF, t_exit = CUDART_INF;
  const xd lo[2] = {bx0, by0};
  const xd hi[2] = {bx1, by1};
  const xd p[2] = {ax, ay};
  const xd d[2] = {bx - ax, by - ay};
  for (int axis = 0; axis < 2; ++axis) {
    if (d[axis].v == 0.0) {
      if (p[axis] < lo[axis] || p[axis] > hi[axis]) return 1.0;
      continue;
    }
    xd t0 = (lo[axis] - p[axis]) / d[axis];
    xd t1 = (hi[axis] - p[axis]) / d[axis];
    if (t0 > t1) {
      const xd tmp = t0;
      t0 = t1;
      t1 = tmp;
    }
    if (t0 > t_enter) t_enter = t0;
    if (t1 < t_exit) t_exit = t1;
  }
  if (t_enter > t_exit || t_enter.v > 1.0) return 1.0;
  return t_enter.v > 0.0 ? t_enter : xd(0.0);
}

// guard_points + guard_time (offball.cpp:125-174) for a point outside the
// area's interior; gpq (optional) receives P.x, P.y, Q.x, Q.y.
__device__ __forceinline__ xd guard_time_at(const RunParams& R, xd x, xd y, double* gpq) {
  const xd hl = xd(0.5) * xd(R.L);
  const xd dx0 = hl - xd(R.dd);
  const xd hdw = xd(0.5) * xd(R.dw);
  const xd gx = hl;
  const xd ghh = xd(0.5) * xd(R.gw);
  const xd tp = entry_param(dx0, hl, -hdw, hdw, x, y, gx, ghh);
  const xd tq = entry_param(dx0, hl, -hdw, hdw, x, y, gx, -ghh);
  const xd gpx = x + (gx - x) * tp, gpy = y + (ghh - y) * tp;
  const xd gqx = x + (gx - x) * tq, gqy = y + (-ghh - y) * tq;
  const xd cap = R.cap;
  xd total;
  if (R.n_guards >= 2) {
    const xd a0p = arrival_time(R.g_px[0], R.g_py[0], R.g_vx[0], R.g_vy[0], gpx, gpy, R.a_t,
                                R.b_t, R.vmax_t);
    const xd a0q = arrival_time(R.g_px[0], R.g_py[0], R.g_vx[0], R.g_vy[0], gqx, gqy, R.a_t,
                                R.b_t, R.vmax_t);
    const xd a1p = arrival_time(R.g_px[1], R.g_py[1], R.g_vx[1], R.g_vy[1], gpx, gpy, R.a_t,
                                R.b_t, R.vmax_t);
    const xd a1q = arrival_time(R.g_px[1], R.g_py[1], R.g_vx[1], R.g_vy[1], gqx, gqy, R.a_t,
                                R.b_t, R.vmax_t);
    const xd s1 = a0p + a1q, s2 = a0q + a1p;
    total = s2 < s1 ? s2 : s1;  // std::min
  } else if (R.n_guards == 1) {
    const xd ap = arrival_time(R.g_px[0], R.g_py[0], R.g_vx[0], R.g_vy[0], gpx, gpy, R.a_t,
                               R.b_t, R.vmax_t);
    const xd aq = arrival_time(R.g_px[0], R.g_py[0], R.g_vx[0], R.g_vy[0], gqx, gqy, R.a_t,
                               R.b_t, R.vmax_t);
    total = (aq < ap ? aq : ap) + cap;
  } else {
    total = xd(2.0) * cap;
  }
  if (gpq) {
    gpq[0] = gpx.v;
    gpq[1] = gpy.v;
    gpq[2] = gqx.v;
    gpq[3] = gqy.v;
  }
  return total < cap ? total : cap;
}

// score_running_point (offball.cpp:176-201); false where it would throw.
__device__ __forceinline__ bool score_running_point(const RunParams& R, xd x, xd y, double* score,
                                                    double* feat) {
  const xd hl = xd(0.5) * xd(R.L);
  if (!(x.v >= 0.0 && x <= hl && xfabs(y) <= xd(0.5) * xd(R.W))) return false;
  // strictly_in_their_defense_area -> guard_points throws (offball.cpp:126-128)
  const xd dx0 = hl - xd(R.dd);
  const xd hdw = xd(0.5) * xd(R.dw);
  if (x > dx0 && x < hl && y > -hdw && y < hdw) return false;
  const xd gx = hl;
  const xd dist_goal = dist2d(x, y, gx, 0.0);
  const xd dist_ball = dist2d(x, y, R.ball_x, R.ball_y);
  const xd angle = atan2(xfabs(y - xd(0.0)).v, (gx - x).v);
  const xd guard = guard_time_at(R, x, y, nullptr);
  const xd exposure = dist_ball.v > R.nearest_opp ? xd(1.0) : xd(0.0);
  const xd len = R.len_upper;
  const xd s = xd(R.w_dg) * -clamp01(dist_goal / len) + xd(R.w_db) * clamp01(dist_ball / len) +
               xd(R.w_angle) * band_value(R, angle) + xd(R.w_guard) * guard +
               xd(R.w_exp) * -exposure;
  *score = s.v;
  feat[0] = dist_goal.v;
  feat[1] = dist_ball.v;
  feat[2] = angle.v;
  feat[3] = guard.v;
  feat[4] = exposure.v;
  return true;
}

// score_running_point at explicit points (thread per point); ok = 0 where the
// reference throws (outside the front field / strictly inside the area).
__global__ void __launch_bounds__(256) run_points_kernel(RunParams R, int64_t n,
                                                        const double* __restrict__ px,
                                                        const double* __restrict__ py,
                                                        double* __restrict__ out7) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  double score = 0.0, feat[5] = {0, 0, 0, 0, 0};
  const bool ok = score_running_point(R, px[q], py[q], &score, feat);
  out7[7 * q] = ok ? 1.0 : 0.0;
  out7[7 * q + 1] = score;
  for (int k = 0; k < 5; ++k) out7[7 * q + 2 + k] = feat[k];
}

// guard_points / guard_time at explicit points (thread per point, any point
// of the plane); out6 = ok, P.x, P.y, Q.x, Q.y, guard time.  ok = 0 where the
// reference throws (strictly inside the defense area, offball.cpp:126-128).
__global__ void __launch_bounds__(256) guard_points_kernel(RunParams R, int64_t n,
                                                          const double* __restrict__ px,
                                                          const double* __restrict__ py,
                                                          double* __restrict__ out6) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const xd x = px[q], y = py[q];
  const xd hl = xd(0.5) * xd(R.L);
  const xd hdw = xd(0.5) * xd(R.dw);
  const bool inside = x > hl - xd(R.dd) && x < hl && y > -hdw && y < hdw;
  double gpq[4] = {0.0, 0.0, 0.0, 0.0};
  const xd t = inside ? xd(0.0) : guard_time_at(R, x, y, gpq);
  out6[6 * q] = inside ? 0.0 : 1.0;
  for (int k = 0; k < 4; ++k) out6[6 * q + 1 + k] = gpq[k];
  out6[6 * q + 5] = t.v;
}

struct RunOut {
  double* px;
  double* py;
  double* score;
  pp_run_features* features;
  uint8_t* scorable;
};

__device__ __forceinline__ bool run_better(double s_new, int64_t i_new, double s_old,
                                           int64_t i_old) {
  if (i_old < 0) return i_new >= 0;
  if (i_new < 0) return false;
  return s_new > s_old || (s_new == s_old && i_new < i_old);
}

// blockIdx.y = zone, blockIdx.x = vertex block of the zone.
template <bool kMap>
__global__ void __launch_bounds__(256) runmap_kernel(RunParams R, RunOut out,
                                                     RunPartial* __restrict__ partials,
                                                     unsigned* __restrict__ counter,
                                                     pp_runmap_summary* __restrict__ summary) {
  const int z = blockIdx.y;
  const RunZone& Z = R.zone[z];
  const int64_t nv = static_cast<int64_t>(Z.nx) * Z.ny;
  const int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double score = 0.0;
  double feat[5] = {0, 0, 0, 0, 0};
  int64_t cand = -1;
  bool scorable = false;  // a map vertex score_running_point accepts
  if (v < nv && ((kMap && Z.in_map) || Z.selected)) {
    const int i = static_cast<int>(v / Z.ny);
    const int j = static_cast<int>(v % Z.ny);
    const xd step = R.step;
    const xd x = xd(Z.x0) + xd(1.0) * (xd(double(i)) * step);
    const xd y = xd(Z.y0) + xd(Z.ydir) * (xd(double(j)) * step);
    const bool ok = score_running_point(R, x, y, &score, feat);
    if (kMap && Z.in_map) {
      const int64_t o = Z.offset + v;
      out.px[o] = x.v;
      out.py[o] = y.v;
      out.score[o] = ok ? score : CUDART_NAN;
      out.features[o] =
          ok ? pp_run_features{feat[0], feat[1], feat[2], feat[3], feat[4]} : pp_run_features{0, 0, 0, 0, 0};
      out.scorable[o] = ok;
      scorable = ok;
    }
    // best_running_points candidates: interior, outside the INCLUSIVE area.
    const xd hl = xd(0.5) * xd(R.L);
    const xd hdw = xd(0.5) * xd(R.dw);
    const bool in_area = x >= hl - xd(R.dd) && x <= hl && y >= -hdw && y <= hdw;
    if (Z.selected && ok && i >= 1 && i + 1 < Z.nx && j >= 1 && j + 1 < Z.ny && !in_area) cand = v;
  }
  // CTA argmax (score desc, index asc).
  __shared__ RunPartial red[256];
  red[threadIdx.x].score = score;
  red[threadIdx.x].index = cand;
  __syncthreads();
  for (int stride = blockDim.x / 2; stride > 0; stride >>= 1) {
    if (threadIdx.x < stride) {
      RunPartial& a = red[threadIdx.x];
      const RunPartial& b = red[threadIdx.x + stride];
      if (run_better(b.score, b.index, a.score, a.index)) {
        a.score = b.score;
        a.index = b.index;
      }
    }
    __syncthreads();
  }
  __shared__ unsigned last;
  const int n_ok = __syncthreads_count(scorable);
  if (threadIdx.x == 0) {
    RunPartial p = red[0];
    p.px = p.py = 0.0;
    const int64_t base = static_cast<int64_t>(z) * gridDim.x;
    partials[base + blockIdx.x] = p;
    if (n_ok) atomicAdd(reinterpret_cast<unsigned long long*>(counter + 2), n_ok);
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x * gridDim.y - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 4) {
    const int zz = threadIdx.x;
    const RunZone& ZZ = R.zone[zz];
    RunPartial best;
    best.score = 0.0;
    best.index = -1;
    const int64_t base = static_cast<int64_t>(zz) * gridDim.x;
    for (int b = 0; b < R.blocks_per_zone[zz]; ++b) {
      const volatile RunPartial* p = partials + base + b;
      const double ps = p->score;
      const int64_t pi = p->index;
      if (run_better(ps, pi, best.score, best.index)) {
        best.score = ps;
        best.index = pi;
      }
    }
    pp_running_point& o = summary->best[zz];
    o.zone = zz;
    o.valid = 0;
    if (best.index >= 0 && ZZ.selected) {
      const int i = static_cast<int>(best.index / ZZ.ny);
      const int j = static_cast<int>(best.index % ZZ.ny);
      const xd x = xd(ZZ.x0) + xd(1.0) * (xd(double(i)) * xd(R.step));
      const xd y = xd(ZZ.y0) + xd(ZZ.ydir) * (xd(double(j)) * xd(R.step));
      double s, f[5];
      score_running_point(R, x, y, &s, f);
      o.valid = 1;
      o.px = x.v;
      o.py = y.v;
      o.score = s;
      o.features = pp_run_features{f[0], f[1], f[2], f[3], f[4]};
    }
  }
  if (threadIdx.x == 0) {
    unsigned long long* n_sc = reinterpret_cast<unsigned long long*>(counter + 2);
    summary->n_scorable = static_cast<int64_t>(*reinterpret_cast<volatile unsigned long long*>(n_sc));
    *n_sc = 0ull;  // self-cleaning for the next launch
    *counter = 0;
  }
}

}  // namespace pp
