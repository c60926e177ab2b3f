/*
 * pp_oracle.c -- TEST INFRASTRUCTURE ONLY: plain-C FP64 restatement of the
 * reference hot path.  Each function cites the reference file:line it
 * follows (paths relative to /root/reference/proj).  Compile with
 * -ffp-contract=off (proj/CMakeLists.txt:12-14) so every expression rounds
 * exactly like the reference's.  Single-threaded; run_dpps's worker pool is
 * result-neutral (dpps.cpp:281-283) so the serial loop is the oracle.
 */
#include "pp_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "passplan_b200_layout.h"

#define OR_PI 3.14159265358979323846 /* std::numbers::pi */

static void put(char* msg, size_t len, const char* s) {
  if (msg && len) snprintf(msg, len, "%s", s);
}

/* ---- vec2.hpp:45-56 ---------------------------------------------------- */
static double dist2(double ax, double ay, double bx, double by) {
  const double dx = ax - bx, dy = ay - by;
  return sqrt(dx * dx + dy * dy);
}

static double seg_dist(double px, double py, double ax, double ay, double bx, double by) {
  const double abx = bx - ax, aby = by - ay;
  const double len2 = abx * abx + aby * aby;
  if (len2 == 0.0) return dist2(px, py, ax, ay);
  double t = ((px - ax) * abx + (py - ay) * aby) / len2;
  if (t < 0.0) t = 0.0;
  if (t > 1.0) t = 1.0;
  return dist2(px, py, ax + abx * t, ay + aby * t);
}

/* ---- detail/arrival_math.hpp:15-69 -------------------------------------- */
static double rest_to_rest(double L, double a, double b, double vmax) {
  const double peak2 = ((2.0 * a) * b * L) / (a + b);
  const double peak = sqrt(peak2);
  if (peak <= vmax) return peak / a + peak / b;
  const double d_used = (vmax * vmax) / (2.0 * a) + (vmax * vmax) / (2.0 * b);
  return vmax / a + vmax / b + (L - d_used) / vmax;
}

static double one_d(double v0, double dist, double a, double b, double vmax) {
  const double brake_dist = (v0 * v0) / (2.0 * b);
  if (v0 < 0.0 || brake_dist > dist) {
    const double gap = brake_dist - copysign(dist, v0);
    return fabs(v0) / b + rest_to_rest(gap, a, b, vmax);
  }
  const double peak2 = ((2.0 * a) * b * dist + b * (v0 * v0)) / (a + b);
  const double peak = sqrt(peak2);
  if (peak <= vmax) return (peak - v0) / a + peak / b;
  if (v0 <= vmax) {
    const double d_used = (vmax * vmax - v0 * v0) / (2.0 * a) + (vmax * vmax) / (2.0 * b);
    return (vmax - v0) / a + vmax / b + (dist - d_used) / vmax;
  }
  const double d_used = (v0 * v0 - vmax * vmax) / (2.0 * b) + (vmax * vmax) / (2.0 * b);
  return (v0 - vmax) / b + vmax / b + (dist - d_used) / vmax;
}

static double arrival_given(double qx, double qy, double d2, double vx, double vy, double a,
                            double b, double vmax, double radius) {
  const double d = sqrt(d2);
  const double deff_raw = d - radius;
  const double deff = deff_raw > 0.0 ? deff_raw : 0.0;
  const double denom = d > 1e-30 ? d : 1e-30;
  const double ex = qx / denom;
  const double ey = qy / denom;
  const double va = vx * ex + vy * ey;
  const double vc = vx * ey - vy * ex;
  const double t_along = one_d(va, deff, a, b, vmax);
  const double t_cross = fabs(vc) / b;
  return t_along > t_cross ? t_along : t_cross;
}

static double arrival_to_point(double tx, double ty, double px, double py, double vx, double vy,
                               double a, double b, double vmax, double radius) {
  const double qx = tx - px;
  const double qy = ty - py;
  return arrival_given(qx, qy, qx * qx + qy * qy, vx, vy, a, b, vmax, radius);
}

/* motion.cpp:16-29 */
static double arrival_time(double px, double py, double vx, double vy, double tx, double ty,
                           const pp_motion_limits* m) {
  const double qx = tx - px;
  const double qy = ty - py;
  const double d2 = qx * qx + qy * qy;
  if (d2 <= 1e-24) {
    const double speed = sqrt(vx * vx + vy * vy);
    return one_d(speed, 0.0, m->max_accel, m->max_decel, m->max_speed);
  }
  return arrival_given(qx, qy, d2, vx, vy, m->max_accel, m->max_decel, m->max_speed, 0.0);
}

/* ---- ball_model.cpp:12-43, 83-107 --------------------------------------- */
typedef struct {
  double ox, oy, ux, uy, speed, v1, slide, roll, t_se, d_se, t_stop, d_stop, from;
} traj_t;

/* slide_phase 0 = BallTrajectory::free_roll (ball_model.cpp:72-75) */
static traj_t resolve_phase(double ox, double oy, double dx, double dy, double speed, int chip,
                            const pp_ball_model* bm, int slide_phase);

static traj_t resolve(double ox, double oy, double dx, double dy, double speed, int chip,
                      const pp_ball_model* bm) {
  return resolve_phase(ox, oy, dx, dy, speed, chip, bm, 1);
}

static traj_t resolve_phase(double ox, double oy, double dx, double dy, double speed, int chip,
                            const pp_ball_model* bm, int slide_phase) {
  traj_t t;
  memset(&t, 0, sizeof(t));
  t.ox = ox;
  t.oy = oy;
  t.speed = speed;
  t.slide = bm->slide_decel;
  t.roll = bm->roll_decel;
  const double n = sqrt(dx * dx + dy * dy);
  if (n == 0.0) {
    t.ux = 1.0;
    t.uy = 0.0;
  } else {
    t.ux = dx / n;
    t.uy = dy / n;
  }
  t.v1 = slide_phase ? bm->transition_ratio * speed : speed;
  if (slide_phase) {
    t.t_se = (speed - t.v1) / bm->slide_decel;
    t.d_se = (speed * speed - t.v1 * t.v1) / (2.0 * bm->slide_decel);
  }
  t.t_stop = t.t_se + t.v1 / bm->roll_decel;
  t.d_stop = t.d_se + (t.v1 * t.v1) / (2.0 * bm->roll_decel);
  t.from = chip ? bm->chip_flight_fraction * t.d_stop : 0.0;
  return t;
}

static double distance_at(const traj_t* tr, double t) {
  if (t < tr->t_se) return tr->speed * t - 0.5 * tr->slide * t * t;
  if (t < tr->t_stop) {
    const double u = t - tr->t_se;
    return tr->d_se + tr->v1 * u - 0.5 * tr->roll * u * u;
  }
  return tr->d_stop;
}

/* returns 0 for nullopt */
static int travel_time(const traj_t* tr, double d, double* out) {
  if (d == 0.0) {
    *out = 0.0;
    return 1;
  }
  if (d > tr->d_stop) return 0;
  if (d <= tr->d_se) {
    const double rad = tr->speed * tr->speed - 2.0 * tr->slide * d;
    *out = 2.0 * d / (tr->speed + sqrt(rad < 0.0 ? 0.0 : rad));
    return 1;
  }
  const double rem = d - tr->d_se;
  const double rad = tr->v1 * tr->v1 - 2.0 * tr->roll * rem;
  *out = tr->t_se + 2.0 * rem / (tr->v1 + sqrt(rad < 0.0 ? 0.0 : rad));
  return 1;
}

/* ---- intercept.cpp:27-69 ------------------------------------------------- */
static int contains(const pp_field* f, double x, double y) { /* world.hpp:20-23 */
  return x >= -0.5 * f->length && x <= 0.5 * f->length && y >= -0.5 * f->width &&
         y <= 0.5 * f->width;
}

static int ray_exit(const pp_field* f, double ox, double oy, double ux, double uy, double* out) {
  if (!contains(f, ox, oy)) return 0;
  const double hx = 0.5 * f->length;
  const double hy = 0.5 * f->width;
  double s = INFINITY, c;
  if (ux > 0.0) {
    c = (hx - ox) / ux;
    if (c < s) s = c;
  } else if (ux < 0.0) {
    c = (-hx - ox) / ux;
    if (c < s) s = c;
  }
  if (uy > 0.0) {
    c = (hy - oy) / uy;
    if (c < s) s = c;
  } else if (uy < 0.0) {
    c = (-hy - oy) / uy;
    if (c < s) s = c;
  }
  *out = s < 0.0 ? 0.0 : s;
  return 1;
}

typedef struct {
  int kb, ke, rif;
} window_t;

static window_t scan_window(const traj_t* tr, int count, double dt, int has_exit, double d_exit) {
  window_t w = {0, 0, 0};
  if (!has_exit) return w;
  w.ke = count;
  if (d_exit < tr->d_stop) {
    double t_exit;
    const int k_last = travel_time(tr, d_exit, &t_exit) ? (int)floor(t_exit / dt + 1e-9) : count - 1;
    w.ke = w.ke < k_last + 1 ? w.ke : k_last + 1;
    w.rif = 0;
  } else {
    w.rif = 1;
  }
  if (tr->from > 0.0) {
    double t_air;
    if (travel_time(tr, tr->from, &t_air)) w.kb = (int)ceil(t_air / dt - 1e-9);
  }
  return w;
}

typedef struct {
  double px, py, vx, vy, a, b, vmax, radius, vbound;
  int id;
} kin_t;

/* make_kin, intercept.cpp:71-85 */
static kin_t make_kin(const pp_robot* r, const pp_motion_limits* m, double radius) {
  kin_t k;
  k.px = r->px;
  k.py = r->py;
  k.vx = r->vx;
  k.vy = r->vy;
  k.a = m->max_accel;
  k.b = m->max_decel;
  k.vmax = m->max_speed;
  k.radius = radius;
  const double speed = sqrt(r->vx * r->vx + r->vy * r->vy);
  k.vbound = speed > m->max_speed ? speed : m->max_speed;
  k.id = r->id;
  return k;
}

/* sample_feasible, kernels/kernel.hpp:33-44 */
static int sample_feasible(const traj_t* tr, double dt, const kin_t* r, int k, or_counts* c) {
  const double t = k * dt;
  const double s = distance_at(tr, t);
  const double px = tr->ox + tr->ux * s;
  const double py = tr->oy + tr->uy * s;
  const double qx = px - r->px;
  const double qy = py - r->py;
  const double d2 = qx * qx + qy * qy;
  const double reach = r->radius + r->vbound * t;
  if (d2 > reach * reach) {
    c->quick_rejects++;
    return 0;
  }
  c->full_tests++;
  return arrival_given(qx, qy, d2, r->vx, r->vy, r->a, r->b, r->vmax, r->radius) <= t;
}

/* scan_robot, intercept.cpp:87-115 + scan_first_scalar, kernel_scalar.cpp:7-12 */
static int scan_robot(const traj_t* tr, double dt, int kb, int ke, const kin_t* kin, or_counts* c) {
  if (kb >= ke) return -1;
  const double t_hi = (ke - 1) * dt;
  const double s_lo = distance_at(tr, kb * dt);
  const double s_hi = distance_at(tr, (ke - 1) * dt);
  const double ax = tr->ox + tr->ux * s_lo, ay = tr->oy + tr->uy * s_lo;
  const double bx = tr->ox + tr->ux * s_hi, by = tr->oy + tr->uy * s_hi;
  const double dmin = seg_dist(kin->px, kin->py, ax, ay, bx, by);
  if (dmin - kin->radius > kin->vbound * t_hi) return -1;
  int k0 = kb;
  if (kin->vbound > 0.0) {
    const double t_lo = (dmin - kin->radius - 1e-9) / kin->vbound;
    if (t_lo > 0.0) {
      /* std::lower_bound over ts[k] = k*dt */
      int k = kb;
      while (k < ke && k * dt < t_lo) ++k;
      k0 = k;
      if (k0 >= ke) return -1;
    }
  }
  for (int k = k0; k < ke; ++k)
    if (sample_feasible(tr, dt, kin, k, c)) return k;
  return -1;
}

/* ---- dpps.cpp:30-62 ------------------------------------------------------ */
void or_direction_table(int32_t n, double* xy) {
  for (int k = 0; k <= n / 2; ++k) {
    const double theta = -OR_PI + k * (2.0 * OR_PI / n);
    double c = cos(theta), s = sin(theta);
    if (k == 0) {
      c = -1.0;
      s = 0.0;
    }
    xy[2 * k] = c;
    xy[2 * k + 1] = s;
    const int m = (n - k) % n;
    if (m != k) {
      xy[2 * m] = c;
      xy[2 * m + 1] = -s;
    }
  }
}

static double power_of(int j, int n, double pmin, double pmax) {
  if (n == 1) return pmin;
  const double span = pmax - pmin;
  return pmin + (j * span) / (n - 1);
}

void or_params_default(pp_params* p) { /* config.hpp, weights.hpp, dpps.hpp defaults */
  memset(p, 0, sizeof(*p));
  p->ball.slide_decel = 3.4;
  p->ball.roll_decel = 0.5;
  p->ball.transition_ratio = 5.0 / 7.0;
  p->ball.power_min = 1.0;
  p->ball.power_max = 6.5;
  p->ball.chip_flight_fraction = 0.5;
  p->motion_ours.max_speed = p->motion_theirs.max_speed = 3.25;
  p->motion_ours.max_accel = p->motion_theirs.max_accel = 3.0;
  p->motion_ours.max_decel = p->motion_theirs.max_decel = 3.0;
  p->grid.n_directions = 128;
  p->grid.n_powers = 64;
  p->grid.power_min = 1.0;
  p->grid.power_max = 6.5;
  p->grid.flat = p->grid.chip = 1;
  p->pass_weights.teammate_time = 1.0;
  p->pass_weights.shoot_angle = 2.0;
  p->pass_weights.dist_goal = 1.0;
  p->pass_weights.refraction = 0.5;
  p->pass_weights.margin = 1.0;
  p->run_weights.dist_goal = 1.0;
  p->run_weights.dist_ball = 0.3;
  p->run_weights.angle = 1.0;
  p->run_weights.guard_time = 0.3;
  p->run_weights.exposure = 0.5;
  p->norm.length_upper = 0.0;
  p->norm.angle_upper = OR_PI;
  p->angle_band.full_lo = 0.0;
  p->angle_band.peak_lo = 15.0 * OR_PI / 180.0;
  p->angle_band.peak_hi = 45.0 * OR_PI / 180.0;
  p->angle_band.full_hi = 90.0 * OR_PI / 180.0;
  pp_thresholds* t = &p->thresholds;
  t->sbip_dt = 1.0 / 60.0;
  t->robot_radius = 0.09;
  t->safety_margin = 0.3;
  t->buffer_time = 0.3;
  t->possession_radius = 0.15;
  t->angle_threshold = 0.1;
  t->shot_power = 0.0;
  t->margin_cap = 10.0;
  t->possession_dt = 1e-3;
  t->contest_epsilon = 1e-3;
  t->grid_step = 0.1;
  t->min_zone_width = 1.0;
  t->guard_time_cap = 10.0;
  t->drag_v_min = 1.0;
  t->marking_radius = 0.6;
}

/* SearchGrid::validate (dpps.cpp:22-28) */
static const char* grid_error(const pp_search_grid* g) {
  if (g->n_directions < 1) return "grid.n_directions must be >= 1";
  if (g->n_powers < 1) return "grid.n_powers must be >= 1";
  if (!(g->power_min > 0.0) || !(g->power_min <= g->power_max))
    return "grid requires 0 < power_min <= power_max";
  return NULL;
}

/* PlannerConfig::validate (config.cpp:172-200) minus SvgStyle */
static const char* config_error(const pp_params* p) {
  const pp_ball_model* b = &p->ball;
  if (!(b->slide_decel > b->roll_decel) || !(b->roll_decel > 0.0))
    return "ball model requires slide_decel > roll_decel > 0";
  if (!(b->transition_ratio > 0.0) || !(b->transition_ratio < 1.0))
    return "transition_ratio must lie in (0,1)";
  if (!(b->power_min > 0.0) || !(b->power_min < b->power_max))
    return "ball model requires 0 < power_min < power_max";
  if (!(b->chip_flight_fraction > 0.0) || !(b->chip_flight_fraction < 1.0))
    return "chip_flight_fraction must lie in (0,1)";
  const pp_motion_limits* ms[2] = {&p->motion_ours, &p->motion_theirs};
  for (int i = 0; i < 2; ++i)
    if (!(ms[i]->max_speed > 0.0) || !(ms[i]->max_accel > 0.0) || !(ms[i]->max_decel > 0.0))
      return "motion limits must all be positive";
  const char* g = grid_error(&p->grid);
  if (g) return g;
  const pp_thresholds* t = &p->thresholds;
  if (!(t->sbip_dt > 0.0)) return "thresholds.sbip_dt must be > 0";
  if (!(t->possession_dt > 0.0)) return "thresholds.possession_dt must be > 0";
  if (!(t->robot_radius >= 0.0)) return "thresholds.robot_radius must be >= 0";
  if (!(t->safety_margin >= 0.0)) return "thresholds.safety_margin must be >= 0";
  if (!(t->buffer_time >= 0.0)) return "thresholds.buffer_time must be >= 0";
  if (!(t->possession_radius > 0.0)) return "thresholds.possession_radius must be > 0";
  if (!(t->angle_threshold >= 0.0)) return "thresholds.angle_threshold must be >= 0";
  if (!(t->shot_power >= 0.0)) return "thresholds.shot_power must be >= 0";
  if (!(t->margin_cap > 0.0)) return "thresholds.margin_cap must be > 0";
  if (!(t->contest_epsilon >= 0.0)) return "thresholds.contest_epsilon must be >= 0";
  if (!(t->grid_step > 0.0)) return "thresholds.grid_step must be > 0";
  if (!(t->min_zone_width > 0.0)) return "thresholds.min_zone_width must be > 0";
  if (!(t->guard_time_cap > 0.0)) return "thresholds.guard_time_cap must be > 0";
  if (!(t->drag_v_min >= 0.0)) return "thresholds.drag_v_min must be >= 0";
  if (!(t->marking_radius > 0.0)) return "thresholds.marking_radius must be > 0";
  if (!(p->norm.length_upper >= 0.0)) return "norm.length_upper must be >= 0";
  if (!(p->norm.angle_upper > 0.0)) return "norm.angle_upper must be > 0";
  const pp_angle_band* a = &p->angle_band;
  if (!(a->full_lo <= a->peak_lo && a->peak_lo <= a->peak_hi && a->peak_hi <= a->full_hi))
    return "angle_band knots must be non-decreasing";
  return NULL;
}

/* id-sorted slot order (dpps.cpp:79-92), stable insertion sort */
static int id_order(const pp_robot* r, int n, int* idx) {
  for (int i = 0; i < n; ++i) {
    int j = i;
    while (j > 0 && r[idx[j - 1]].id > r[i].id) {
      idx[j] = idx[j - 1];
      --j;
    }
    idx[j] = i;
  }
  return n;
}

int32_t or_nearest_teammate(const pp_world* w) {
  int32_t id = w->n_ours > 0 ? w->ours[0].id : -1;
  double best = INFINITY;
  for (int i = 0; i < w->n_ours; ++i) {
    const double d = dist2(w->ours[i].px, w->ours[i].py, w->ball_px, w->ball_py);
    if (d < best) {
      best = d;
      id = w->ours[i].id;
    }
  }
  return id;
}

/* ---- pass_eval.cpp:15-126 (goal_view) ------------------------------------ */
typedef struct {
  double angle, lo, hi, ty;
} view_t;

static int blocks(double px, double py, double gx, double y, double cx, double cy, double r) {
  return seg_dist(cx, cy, px, py, gx, y) < r;
}

static int may_block(double px, double py, double glx, double gly, double grx, double gry,
                     double cx, double cy, double r) {
  const double margin = r + 1e-9;
  if (seg_dist(cx, cy, px, py, glx, gly) <= margin) return 1;
  if (seg_dist(cx, cy, px, py, grx, gry) <= margin) return 1;
  if (seg_dist(cx, cy, glx, gly, grx, gry) <= margin) return 1;
  const double c1 = (glx - px) * (cy - py) - (gly - py) * (cx - px);
  const double c2 = (grx - glx) * (cy - gly) - (gry - gly) * (cx - glx);
  const double c3 = (px - grx) * (cy - gry) - (py - gry) * (cx - grx);
  return (c1 >= 0.0 && c2 >= 0.0 && c3 >= 0.0) || (c1 <= 0.0 && c2 <= 0.0 && c3 <= 0.0);
}

static double bisect_edge(double px, double py, double gx, double cx, double cy, double r,
                          double yb, double yf) {
  for (int i = 0; i < 60; ++i) {
    const double mid = 0.5 * (yb + yf);
    if (blocks(px, py, gx, mid, cx, cy, r))
      yb = mid;
    else
      yf = mid;
  }
  return 0.5 * (yb + yf);
}

static view_t goal_view(double px, double py, const pp_world* w, double r) {
  const pp_field* f = &w->field;
  const double gx = 0.5 * f->length;
  const double gh = 0.5 * f->goal_width;
  view_t v = {0.0, 0.0, 0.0, 0.0}; /* target = their_goal_center */
  if (gx - px < 1e-9) return v;
  int n_half = (int)ceil(f->goal_width / (r < 1e-3 ? 1e-3 : r));
  n_half = n_half < 24 ? 24 : (n_half > 1024 ? 1024 : n_half);
  const int nh = 2 * n_half + 1;
  double* h = (double*)malloc(sizeof(double) * nh);
  int at = 0;
  for (int j = n_half; j >= 1; --j) h[at++] = j == n_half ? -gh : -((j * gh) / n_half);
  h[at++] = 0.0;
  for (int j = 1; j <= n_half; ++j) h[at++] = j == n_half ? gh : (j * gh) / n_half;
  double lo_s[PP_MAX_TEAM], hi_s[PP_MAX_TEAM];
  int n_iv = 0;
  for (int o = 0; o < w->n_theirs; ++o) {
    const double cx = w->theirs[o].px, cy = w->theirs[o].py;
    if (dist2(cx, cy, px, py) < r) {
      free(h);
      return v;
    }
    if (!may_block(px, py, gx, 0.5 * f->goal_width, gx, -0.5 * f->goal_width, cx, cy, r)) continue;
    int first = -1, last = -1;
    for (int i = 0; i < nh; ++i)
      if (blocks(px, py, gx, h[i], cx, cy, r)) {
        if (first < 0) first = i;
        last = i;
      }
    if (first < 0) continue;
    const double lo = first == 0 ? -gh : bisect_edge(px, py, gx, cx, cy, r, h[first], h[first - 1]);
    const double hi = last == nh - 1 ? gh : bisect_edge(px, py, gx, cx, cy, r, h[last], h[last + 1]);
    /* std::sort by lo; equal-lo order cannot change the sweep */
    int k = n_iv;
    while (k > 0 && lo_s[k - 1] > lo) {
      lo_s[k] = lo_s[k - 1];
      hi_s[k] = hi_s[k - 1];
      --k;
    }
    lo_s[k] = lo;
    hi_s[k] = hi;
    ++n_iv;
  }
  free(h);
  const double x_off = gx - px;
  double cursor = -gh, best_lo = 0.0, best_hi = 0.0, best_w = -1.0;
#define OR_CONSIDER(LO, HI)                                                     \
  do {                                                                          \
    const double w_ = atan2((HI) - py, x_off) - atan2((LO) - py, x_off);        \
    if (w_ > best_w) {                                                          \
      best_w = w_;                                                              \
      best_lo = (LO);                                                           \
      best_hi = (HI);                                                           \
    }                                                                           \
  } while (0)
  for (int q = 0; q < n_iv; ++q) {
    if (lo_s[q] > cursor) OR_CONSIDER(cursor, lo_s[q]);
    if (hi_s[q] > cursor) cursor = hi_s[q];
  }
  if (cursor < gh) OR_CONSIDER(cursor, gh);
#undef OR_CONSIDER
  if (best_w <= 0.0) return v;
  v.angle = best_w;
  v.lo = best_lo;
  v.hi = best_hi;
  v.ty = 0.5 * (best_lo + best_hi);
  return v;
}

static double clamp01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }

/* score_pass, pass_eval.cpp:148-173 (angle_between :137-144) */
static double score_pass(double rx, double ry, double our_t, double opp_t, const pp_world* w,
                         const pp_params* p, pp_pass_features* ft) {
  const view_t v = goal_view(rx, ry, w, p->thresholds.robot_radius);
  const double gx = 0.5 * w->field.length;
  const double dist_goal = dist2(rx, ry, gx, 0.0);
  const double ax = rx + (rx - w->ball_px), ay = ry + (ry - w->ball_py);
  const double ux = ax - rx, uy = ay - ry;
  const double vx = gx - rx, vy = v.ty - ry;
  const double cross = ux * vy - uy * vx;
  const double dot = ux * vx + uy * vy;
  const double refr = (cross == 0.0 && dot == 0.0) ? 0.0 : fabs(atan2(cross, dot));
  const double margin = isinf(opp_t) ? p->thresholds.margin_cap : opp_t - our_t;
  const double len_upper = p->norm.length_upper > 0.0 ? p->norm.length_upper : w->field.length;
  const double ang_upper = p->norm.angle_upper;
  const pp_pass_weights* pw = &p->pass_weights;
  const double score = pw->teammate_time * (-our_t) + pw->shoot_angle * clamp01(v.angle / ang_upper) +
                       pw->dist_goal * (-clamp01(dist_goal / len_upper)) +
                       pw->refraction * (-clamp01(refr / ang_upper)) + pw->margin * margin;
  if (ft) {
    ft->teammate_intercept_time = our_t;
    ft->shoot_angle_at_receive = v.angle;
    ft->dist_receive_to_goal = dist_goal;
    ft->refraction_angle = refr;
    ft->intercept_margin = margin;
  }
  return score;
}

/* ---- dpps.cpp:106-309 (run_dpps_serial) + best_pass ×3 -------------------- */
typedef struct {
  double bound;
  int slot;
} order_t;

static int cmp_order(const void* a, const void* b) {
  const order_t* x = (const order_t*)a;
  const order_t* y = (const order_t*)b;
  if (x->bound < y->bound) return -1;
  if (x->bound > y->bound) return 1;
  return x->slot - y->slot;
}

/* best_of, dpps.cpp:140-202 */
static void best_of(const kin_t* team, int n, int skip, const traj_t* tr, double dt, window_t win,
                    int* best_slot, double* best_t, int* best_id, double* bx, double* by,
                    or_counts* c) {
  int best_k = win.ke;
  order_t order[PP_MAX_TEAM];
  int n_ord = 0;
  const double rest_x = tr->ox + tr->ux * tr->d_stop, rest_y = tr->oy + tr->uy * tr->d_stop;
  for (int i = 0; i < n; ++i) {
    if (i == skip) continue;
    double bound = 0.0;
    if (win.kb < win.ke && team[i].vbound > 0.0) {
      const double s_lo = distance_at(tr, win.kb * dt);
      const double s_hi = distance_at(tr, (win.ke - 1) * dt);
      bound = (seg_dist(team[i].px, team[i].py, tr->ox + tr->ux * s_lo, tr->oy + tr->uy * s_lo,
                        tr->ox + tr->ux * s_hi, tr->oy + tr->uy * s_hi) -
               team[i].radius) /
              team[i].vbound;
      c->bounds++;
    }
    order[n_ord].bound = bound;
    order[n_ord].slot = i;
    ++n_ord;
  }
  qsort(order, (size_t)n_ord, sizeof(order_t), cmp_order);
  for (int o = 0; o < n_ord; ++o) {
    const kin_t* kin = &team[order[o].slot];
    c->scans++;
    const int ke = win.ke < best_k + 1 ? win.ke : best_k + 1;
    const int k = scan_robot(tr, dt, win.kb, ke, kin, c);
    double time = INFINITY, px = 0.0, py = 0.0;
    if (k >= 0) {
      time = k * dt;
      const double s = distance_at(tr, time);
      px = tr->ox + tr->ux * s;
      py = tr->oy + tr->uy * s;
      if (k < best_k) best_k = k;
    } else if (win.rif) {
      c->rest_evals++;
      const double arr = arrival_to_point(rest_x, rest_y, kin->px, kin->py, kin->vx, kin->vy,
                                          kin->a, kin->b, kin->vmax, kin->radius);
      time = arr > tr->t_stop ? arr : tr->t_stop;
      px = rest_x;
      py = rest_y;
    }
    if (time < *best_t || (time == *best_t && kin->id < *best_id)) {
      *best_t = time;
      *best_id = kin->id;
      *best_slot = order[o].slot;
      *bx = px;
      *by = py;
    }
  }
  if (skip >= 0 && skip < n) {
    c->scans++;
    const int ke = win.ke < best_k + 1 ? win.ke : best_k + 1;
    (void)scan_robot(tr, dt, win.kb, ke, &team[skip], c);
  }
}

int or_dpps_counted(const pp_world* w, const pp_params* p, const pp_search_grid* grid_in,
                    int32_t kicker_id, void* block, or_counts* counts, char* msg, size_t msg_len) {
  const pp_search_grid* g = grid_in ? grid_in : &p->grid;
  const char* err = grid_error(g);
  if (err) {
    put(msg, msg_len, err);
    return PP_CONFIG;
  }
  err = config_error(p);
  if (err) {
    put(msg, msg_len, err);
    return PP_CONFIG;
  }
  int found = 0;
  for (int i = 0; i < w->n_ours; ++i) found |= w->ours[i].id == kicker_id;
  if (!found) {
    char b[96];
    snprintf(b, sizeof(b), "kicker id %d is not on team ours", kicker_id);
    put(msg, msg_len, b);
    return PP_VALIDATION;
  }
  or_counts local;
  memset(&local, 0, sizeof(local));
  or_counts* c = counts ? counts : &local;
  memset(c, 0, sizeof(*c));
  const int n_kt = (g->flat ? 1 : 0) + (g->chip ? 1 : 0);
  const int nd = g->n_directions, np = g->n_powers;
  const int64_t n = (int64_t)n_kt * nd * np;
  pp_grid_view v;
  pp_grid_view_of_(block, n, &v);
  pp_dpps_summary* s = v.summary;
  memset(s, 0, sizeof(*s));
  s->n_cells = n;
  s->n_kick_types = n_kt;
  s->kick_types[0] = g->flat ? 0 : 1;
  s->kick_types[1] = 1;
  s->n_directions = nd;
  s->n_powers = np;
  s->kicker_id = kicker_id;
  s->n_ours = w->n_ours;
  s->n_theirs = w->n_theirs;
  int so[PP_MAX_TEAM], st[PP_MAX_TEAM];
  id_order(w->ours, w->n_ours, so);
  id_order(w->theirs, w->n_theirs, st);
  kin_t ours[PP_MAX_TEAM], theirs[PP_MAX_TEAM];
  int kicker_slot = -1;
  for (int i = 0; i < PP_MAX_TEAM; ++i) {
    s->ours_ids[i] = i < w->n_ours ? w->ours[so[i]].id : -1;
    s->theirs_ids[i] = i < w->n_theirs ? w->theirs[st[i]].id : -1;
  }
  for (int i = 0; i < w->n_ours; ++i) {
    ours[i] = make_kin(&w->ours[so[i]], &p->motion_ours, p->thresholds.robot_radius);
    if (ours[i].id == kicker_id) kicker_slot = i;
  }
  for (int i = 0; i < w->n_theirs; ++i)
    theirs[i] = make_kin(&w->theirs[st[i]], &p->motion_theirs, p->thresholds.robot_radius);
  s->kicker_slot = kicker_slot;
  {
    const pp_robot* k = NULL;
    for (int i = 0; i < w->n_ours && !k; ++i)
      if (w->ours[i].id == kicker_id) k = &w->ours[i];
    s->kicker_in_possession =
        dist2(w->ball_px, w->ball_py, k->px, k->py) <= p->thresholds.possession_radius;
  }
  for (int k = 0; k < 3; ++k) s->best_cell[k] = -1;
  if (n == 0) return PP_OK;
  double* dirs = (double*)malloc(sizeof(double) * 2 * nd);
  or_direction_table(nd, dirs);
  const double dt = p->thresholds.sbip_dt;
  int64_t cell = 0;
  for (int kt = 0; kt < n_kt; ++kt) {
    const int chip = (kt == 0 && g->flat) ? 0 : 1;
    for (int d = 0; d < nd; ++d) {
      double d_exit = 0.0;
      const int has_exit = ray_exit(&w->field, w->ball_px, w->ball_py, dirs[2 * d], dirs[2 * d + 1],
                                    &d_exit);
      for (int j = 0; j < np; ++j, ++cell) {
        const double speed = power_of(j, np, g->power_min, g->power_max);
        const traj_t tr = resolve(w->ball_px, w->ball_py, dirs[2 * d], dirs[2 * d + 1], speed,
                                  chip, &p->ball);
        const int count = (int)floor(tr.t_stop / dt + 1e-9) + 1;
        const window_t win = scan_window(&tr, count, dt, has_exit, d_exit);
        int os = -1, oid = -1, ts = -1, tid = -1;
        double ot = INFINITY, pt = INFINITY, rx = 0.0, ry = 0.0, dx, dy;
        best_of(ours, w->n_ours, kicker_slot, &tr, dt, win, &os, &ot, &oid, &rx, &ry, c);
        best_of(theirs, w->n_theirs, -1, &tr, dt, win, &ts, &pt, &tid, &dx, &dy, c);
        v.our_time[cell] = ot;
        v.opp_time[cell] = pt;
        v.our_slot[cell] = (int8_t)os;
        v.opp_slot[cell] = (int8_t)ts;
        v.rx[cell] = 0.0;
        v.ry[cell] = 0.0;
        uint8_t feas = 0;
        if (ot < INFINITY) {
          v.rx[cell] = rx;
          v.ry[cell] = ry;
          feas = isinf(pt) || ot + p->thresholds.safety_margin <= pt;
        }
        v.feasible[cell] = feas;
        v.score[cell] = -INFINITY;
        if (feas) {
          pp_pass_features ft;
          const double sc = score_pass(rx, ry, ot, pt, w, p, &ft);
          v.score[cell] = (float)sc;
          const int row = chip ? 2 : 1;
          s->n_feasible[0]++;
          s->n_feasible[row]++;
          /* best_pass: first strict max in cell order (pass_eval.cpp:178-185) */
          if (s->best_cell[row] < 0 || sc > s->best_score[row]) {
            s->best_cell[row] = cell;
            s->best_score[row] = sc;
            s->best_features[row] = ft;
          }
          if (s->best_cell[0] < 0 || sc > s->best_score[0]) {
            s->best_cell[0] = cell;
            s->best_score[0] = sc;
            s->best_features[0] = ft;
          }
        }
      }
    }
  }
  free(dirs);
  s->sbip_calls = (uint64_t)n * (uint64_t)(w->n_ours + w->n_theirs);
  return PP_OK;
}

int or_dpps(const pp_world* w, const pp_params* p, const pp_search_grid* grid, int32_t kicker_id,
            void* block, char* msg, size_t msg_len) {
  return or_dpps_counted(w, p, grid, kicker_id, block, NULL, msg, msg_len);
}

int or_score_cells(const pp_world* w, const pp_params* p, int64_t n, const double* rx,
                   const double* ry, const double* our_time, const double* opp_time,
                   const uint8_t* feasible, double* score_out, pp_pass_features* feat_out,
                   char* msg, size_t msg_len) {
  for (int64_t i = 0; i < n; ++i) {
    if (!feasible[i]) {
      put(msg, msg_len, "score_pass: candidate is not feasible");
      return PP_DOMAIN;
    }
    score_out[i] = score_pass(rx[i], ry[i], our_time[i], opp_time[i], w, p,
                              feat_out ? &feat_out[i] : NULL);
  }
  return PP_OK;
}

int or_goal_views(const pp_world* w, double radius, int64_t n, const double* px, const double* py,
                  double* angle, double* lo, double* hi, double* ty) {
  for (int64_t i = 0; i < n; ++i) {
    const view_t v = goal_view(px[i], py[i], w, radius);
    angle[i] = v.angle;
    lo[i] = v.lo;
    hi[i] = v.hi;
    ty[i] = v.ty;
  }
  return PP_OK;
}

/* ---- offball.cpp:17-258 -------------------------------------------------- */
typedef struct {
  double x0, x1, y0, y1;
} box_t;

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

static double entry_param(box_t b, double ax, double ay, double bx, double by) {
  double t_enter = -INFINITY, t_exit = INFINITY;
  const double lo[2] = {b.x0, b.y0}, hi[2] = {b.x1, b.y1};
  const double p[2] = {ax, ay}, d[2] = {bx - ax, by - ay};
  for (int axis = 0; axis < 2; ++axis) {
    if (d[axis] == 0.0) {
      if (p[axis] < lo[axis] || p[axis] > hi[axis]) return 1.0;
      continue;
    }
    double t0 = (lo[axis] - p[axis]) / d[axis];
    double t1 = (hi[axis] - p[axis]) / d[axis];
    if (t0 > t1) {
      const double tmp = t0;
      t0 = t1;
      t1 = tmp;
    }
    if (t0 > t_enter) t_enter = t0;
    if (t1 < t_exit) t_exit = t1;
  }
  if (t_enter > t_exit || t_enter > 1.0) return 1.0;
  return t_enter > 0.0 ? t_enter : 0.0;
}

static double band_value(const pp_angle_band* b, double a) {
  if (a < b->full_lo || a > b->full_hi) return 0.0;
  if (a < b->peak_lo) {
    const double w = b->peak_lo - b->full_lo;
    return w > 0.0 ? (a - b->full_lo) / w : 1.0;
  }
  if (a > b->peak_hi) {
    const double w = b->full_hi - b->peak_hi;
    return w > 0.0 ? (b->full_hi - a) / w : 1.0;
  }
  return 1.0;
}

typedef struct {
  double dist;
  int id, idx;
} cand_t;

static int cmp_cand(const void* a, const void* b) {
  const cand_t* x = (const cand_t*)a;
  const cand_t* y = (const cand_t*)b;
  if (x->dist != y->dist) return x->dist < y->dist ? -1 : 1;
  return (x->id > y->id) - (x->id < y->id);
}

/* score_running_point (offball.cpp:176-201); 0 where it throws */
static int score_running_point(double x, double y, const pp_world* w, const pp_params* p,
                               double* score, pp_run_features* ft) {
  const pp_field* f = &w->field;
  if (!(x >= 0.0 && x <= 0.5 * f->length && fabs(y) <= 0.5 * f->width)) return 0;
  /* guard_points throws strictly inside the defense area (offball.cpp:126-128) */
  if (x > 0.5 * f->length - f->defense_depth && x < 0.5 * f->length &&
      y > -0.5 * f->defense_width && y < 0.5 * f->defense_width)
    return 0;
  const double gx = 0.5 * f->length;
  const double dg = dist2(x, y, gx, 0.0);
  const double db = dist2(x, y, w->ball_px, w->ball_py);
  const double angle = atan2(fabs(y - 0.0), gx - x);
  const box_t box = {0.5 * f->length - f->defense_depth, 0.5 * f->length, -0.5 * f->defense_width,
                     0.5 * f->defense_width};
  const double lpx = 0.5 * f->length, lpy = 0.5 * f->goal_width;
  const double rpx = 0.5 * f->length, rpy = -0.5 * f->goal_width;
  const double tp = entry_param(box, x, y, lpx, lpy);
  const double tq = entry_param(box, x, y, rpx, rpy);
  const double gpx = x + (lpx - x) * tp, gpy = y + (lpy - y) * tp;
  const double gqx = x + (rpx - x) * tq, gqy = y + (rpy - y) * tq;
  /* guard_time (offball.cpp:137-174) */
  cand_t cands[PP_MAX_TEAM];
  const int nt = w->n_theirs;
  for (int i = 0; i < nt; ++i) {
    const pp_robot* r = &w->theirs[i];
    const double cx = clampd(r->px, box.x0, box.x1), cy = clampd(r->py, box.y0, box.y1);
    cands[i].dist = dist2(r->px, r->py, cx, cy);
    cands[i].id = r->id;
    cands[i].idx = i;
  }
  qsort(cands, (size_t)nt, sizeof(cand_t), cmp_cand);
  const double cap = p->thresholds.guard_time_cap;
  const pp_motion_limits* m = &p->motion_theirs;
  double total;
  if (nt >= 2) {
    const pp_robot* r0 = &w->theirs[cands[0].idx];
    const pp_robot* r1 = &w->theirs[cands[1].idx];
    const double a0p = arrival_time(r0->px, r0->py, r0->vx, r0->vy, gpx, gpy, m);
    const double a0q = arrival_time(r0->px, r0->py, r0->vx, r0->vy, gqx, gqy, m);
    const double a1p = arrival_time(r1->px, r1->py, r1->vx, r1->vy, gpx, gpy, m);
    const double a1q = arrival_time(r1->px, r1->py, r1->vx, r1->vy, gqx, gqy, m);
    const double s1 = a0p + a1q, s2 = a0q + a1p;
    total = s2 < s1 ? s2 : s1;
  } else if (nt == 1) {
    const pp_robot* r0 = &w->theirs[cands[0].idx];
    const double ap = arrival_time(r0->px, r0->py, r0->vx, r0->vy, gpx, gpy, m);
    const double aq = arrival_time(r0->px, r0->py, r0->vx, r0->vy, gqx, gqy, m);
    total = (aq < ap ? aq : ap) + cap;
  } else {
    total = 2.0 * cap;
  }
  const double guard = total < cap ? total : cap;
  double nearest = INFINITY;
  for (int i = 0; i < nt; ++i) {
    const double d = dist2(w->theirs[i].px, w->theirs[i].py, w->ball_px, w->ball_py);
    nearest = d < nearest ? d : nearest; /* std::min(nearest, d) */
  }
  const double exposure = db > nearest ? 1.0 : 0.0;
  const double len = p->norm.length_upper > 0.0 ? p->norm.length_upper : f->length;
  const pp_run_weights* rw = &p->run_weights;
  *score = rw->dist_goal * -clamp01(dg / len) + rw->dist_ball * clamp01(db / len) +
           rw->angle * band_value(&p->angle_band, angle) + rw->guard_time * guard +
           rw->exposure * -exposure;
  ft->dist_to_goal = dg;
  ft->dist_to_ball = db;
  ft->angle_to_goal = angle;
  ft->guard_time = guard;
  ft->defense_exposure = exposure;
  return 1;
}

static int axis_count(double span, double step) {
  const int n = (int)floor(span / step + 1e-9) + 1;
  return n > 0 ? n : 0;
}

typedef struct {
  double x0, x1, y0, y1;
  double xa, ya, ydir;
  int nx, ny;
} zone_t;

static int partition(const pp_world* w, const pp_params* p, zone_t z[4], double* cut_x,
                     double* cut_y) {
  const pp_field* f = &w->field;
  const double mzw = p->thresholds.min_zone_width;
  if (!(mzw > 0.0) || 2.0 * mzw > f->width) return 0;
  *cut_x = 0.25 * f->length;
  *cut_y = clampd(w->ball_py, -0.5 * f->width + mzw, 0.5 * f->width - mzw);
  const double xm = 0.5 * f->length, yt = 0.5 * f->width;
  const double b[4][4] = {{0.0, *cut_x, *cut_y, yt},
                          {0.0, *cut_x, -yt, *cut_y},
                          {*cut_x, xm, *cut_y, yt},
                          {*cut_x, xm, -yt, *cut_y}};
  const double step = p->thresholds.grid_step;
  for (int i = 0; i < 4; ++i) {
    z[i].x0 = b[i][0];
    z[i].x1 = b[i][1];
    z[i].y0 = b[i][2];
    z[i].y1 = b[i][3];
    const int upper = i == 0 || i == 2; /* zone_ys, offball.cpp:79-83 */
    z[i].xa = z[i].x0;
    z[i].ya = upper ? z[i].y0 : z[i].y1;
    z[i].ydir = upper ? 1.0 : -1.0;
    z[i].nx = axis_count(z[i].x1 - z[i].x0, step);
    z[i].ny = axis_count(z[i].y1 - z[i].y0, step);
  }
  return 1;
}

int64_t or_runmap_count(const pp_world* w, const pp_params* p, uint32_t zone_mask) {
  zone_t z[4];
  double cx, cy;
  if (!partition(w, p, z, &cx, &cy)) return -1;
  int64_t n = 0;
  for (int i = 0; i < 4; ++i)
    if (zone_mask & (1u << i)) n += (int64_t)z[i].nx * z[i].ny;
  return n;
}

int or_runmap(const pp_world* w, const pp_params* p, const pp_runmap_request* req, void* block,
              int64_t block_vertices, char* msg, size_t msg_len) {
  zone_t z[4];
  double cut_x, cut_y;
  if (!partition(w, p, z, &cut_x, &cut_y)) {
    put(msg, msg_len, "min_zone_width must be positive and at most half the field width");
    return PP_CONFIG;
  }
  const double step = p->thresholds.grid_step;
  pp_runmap_view v;
  pp_runmap_view_of_(block, block_vertices, &v);
  pp_runmap_summary* s = v.summary;
  memset(s, 0, sizeof(*s));
  s->cut_x = cut_x;
  s->cut_y = cut_y;
  int64_t at = 0;
  for (int i = 0; i < 4; ++i) {
    s->zone_offset[i] = at;
    if (!(req->zone_mask & (1u << i))) continue;
    s->zone_nx[i] = z[i].nx;
    s->zone_ny[i] = z[i].ny;
    for (int a = 0; a < z[i].nx; ++a) {
      for (int b = 0; b < z[i].ny; ++b, ++at) {
        if (at >= block_vertices) {
          put(msg, msg_len, "runmap block too small");
          return PP_INTERNAL;
        }
        const double x = z[i].xa + 1.0 * (a * step);
        const double y = z[i].ya + z[i].ydir * (b * step);
        v.px[at] = x;
        v.py[at] = y;
        double sc;
        pp_run_features ft;
        if (score_running_point(x, y, w, p, &sc, &ft)) {
          v.score[at] = sc;
          v.features[at] = ft;
          v.scorable[at] = 1;
          s->n_scorable++;
        } else {
          v.score[at] = NAN;
          memset(&v.features[at], 0, sizeof(pp_run_features));
          v.scorable[at] = 0;
        }
      }
    }
  }
  s->n_vertices = at;
  /* best_running_points (offball.cpp:215-258) */
  uint32_t excluded = req->occupied_mask;
  if (req->has_best_pass_point) {
    const double px = req->best_pass_px, py = req->best_pass_py;
    if (!(px < z[0].x0 || px > z[2].x1 || py < z[1].y0 || py > z[0].y1)) {
      const int lab = px >= cut_x ? (py >= cut_y ? 2 : 3) : (py >= cut_y ? 0 : 1);
      excluded |= 1u << lab;
    }
  }
  uint32_t selected = 0;
  int n_sel = 0;
  const int prio[4] = {2, 3, 0, 1};
  for (int q = 0; q < 4; ++q) {
    if (n_sel >= req->n_runners) break;
    if (!(excluded & (1u << prio[q]))) {
      selected |= 1u << prio[q];
      ++n_sel;
    }
  }
  const pp_field* f = &w->field;
  for (int i = 0; i < 4; ++i) {
    s->best_order[i] = -1;
    if (!(selected & (1u << i))) continue;
    int have = 0;
    pp_running_point best;
    memset(&best, 0, sizeof(best));
    for (int a = 1; a + 1 < z[i].nx; ++a) {
      for (int b = 1; b + 1 < z[i].ny; ++b) {
        const double x = z[i].xa + 1.0 * (a * step);
        const double y = z[i].ya + z[i].ydir * (b * step);
        if (x >= 0.5 * f->length - f->defense_depth && x <= 0.5 * f->length &&
            y >= -0.5 * f->defense_width && y <= 0.5 * f->defense_width)
          continue; /* in_their_defense_area, inclusive */
        double sc;
        pp_run_features ft;
        if (!score_running_point(x, y, w, p, &sc, &ft)) continue;
        if (!have || sc > best.score) {
          best.zone = i;
          best.valid = 1;
          best.px = x;
          best.py = y;
          best.score = sc;
          best.features = ft;
          have = 1;
        }
      }
    }
    if (have) {
      s->best[i] = best;
      s->best_order[s->n_best++] = i;
    }
  }
  return PP_OK;
}

/* ==== SURVEY §8(f): interception, possession, shot, free kick ============ */

static const char* ball_error(const pp_ball_model* b) { /* ball_model.cpp:47-60 */
  if (!(b->slide_decel > b->roll_decel) || !(b->roll_decel > 0.0))
    return "ball model requires slide_decel > roll_decel > 0";
  if (!(b->transition_ratio > 0.0) || !(b->transition_ratio < 1.0))
    return "transition_ratio must lie in (0,1)";
  if (!(b->power_min > 0.0) || !(b->power_min < b->power_max))
    return "ball model requires 0 < power_min < power_max";
  if (!(b->chip_flight_fraction > 0.0) || !(b->chip_flight_fraction < 1.0))
    return "chip_flight_fraction must lie in (0,1)";
  return NULL;
}

/* BallTrajectory::{flat_kick, chip_kick, free_roll} with resolve's checks
 * (ball_model.cpp:12-75). */
static int kick_traj(const pp_kick* k, const pp_ball_model* b, traj_t* out, char* msg,
                     size_t len) {
  const char* e = ball_error(b);
  if (e) {
    put(msg, len, e);
    return PP_CONFIG;
  }
  const int roll = k->kind == 2;
  const double speed = roll ? sqrt(k->dir_x * k->dir_x + k->dir_y * k->dir_y) : k->speed;
  if (!(speed >= 0.0) || !isfinite(speed)) {
    put(msg, len, "kick speed must be finite and non-negative");
    return PP_DOMAIN;
  }
  if (sqrt(k->dir_x * k->dir_x + k->dir_y * k->dir_y) == 0.0 && speed > 0.0) {
    put(msg, len, "kick direction must be non-zero");
    return PP_DOMAIN;
  }
  *out = resolve_phase(k->origin_x, k->origin_y, k->dir_x, k->dir_y, speed, k->kind == 1, b, !roll);
  return PP_OK;
}

/* intercept_with (intercept.cpp:121-150) */
static pp_intercept intercept_with(const traj_t* tr, double dt, window_t win, const kin_t* kin) {
  or_counts c;
  memset(&c, 0, sizeof(c));
  pp_intercept r;
  memset(&r, 0, sizeof(r));
  r.robot_id = kin->id;
  const int k = scan_robot(tr, dt, win.kb, win.ke, kin, &c);
  if (k >= 0) {
    const double s = distance_at(tr, k * dt);
    r.finite = 1;
    r.time = k * dt;
    r.point_x = tr->ox + tr->ux * s;
    r.point_y = tr->oy + tr->uy * s;
  } else if (win.rif) {
    const double rx = tr->ox + tr->ux * tr->d_stop, ry = tr->oy + tr->uy * tr->d_stop;
    const double arr = arrival_to_point(rx, ry, kin->px, kin->py, kin->vx, kin->vy, kin->a, kin->b,
                                        kin->vmax, kin->radius);
    r.finite = 1;
    r.time = arr > tr->t_stop ? arr : tr->t_stop;
    r.point_x = rx;
    r.point_y = ry;
  }
  return r;
}

/* TrajectorySamples count + scan_window along the unit direction
 * (intercept.cpp:12-25, 154-170) */
static window_t traj_window(const traj_t* tr, const pp_field* f, double dt) {
  const int count = (int)floor(tr->t_stop / dt + 1e-9) + 1;
  double d_exit = 0.0;
  const int has_exit = ray_exit(f, tr->ox, tr->oy, tr->ux, tr->uy, &d_exit);
  return scan_window(tr, count, dt, has_exit, d_exit);
}

int or_intercept_all(const pp_world* w, const pp_params* p, const pp_kick* k, double dt,
                     pp_intercept* out, char* msg, size_t msg_len) {
  if (!(dt > 0.0)) {
    put(msg, msg_len, "intercept_all: dt must be > 0");
    return PP_DOMAIN;
  }
  traj_t tr;
  const int st = kick_traj(k, &p->ball, &tr, msg, msg_len);
  if (st != PP_OK) return st;
  const window_t win = traj_window(&tr, &w->field, dt);
  int n = 0;
  for (int team = 0; team < 2; ++team) { /* intercept.cpp:176-195 */
    const pp_robot* r = team ? w->theirs : w->ours;
    const int nr = team ? w->n_theirs : w->n_ours;
    int idx[PP_MAX_TEAM];
    id_order(r, nr, idx);
    for (int i = 0; i < nr; ++i) {
      const kin_t kin = make_kin(&r[idx[i]], team ? &p->motion_theirs : &p->motion_ours,
                                 p->thresholds.robot_radius);
      out[n] = intercept_with(&tr, dt, win, &kin);
      out[n].team = team;
      ++n;
    }
  }
  return PP_OK;
}

int or_possession(const pp_world* w, const pp_params* p, pp_possession_report* out, char* msg,
                  size_t msg_len) {
  const pp_kick roll = {w->ball_px, w->ball_py, w->ball_vx, w->ball_vy, 0.0, 2, 0};
  pp_intercept all[2 * PP_MAX_TEAM];
  const int st = or_intercept_all(w, p, &roll, p->thresholds.possession_dt, all, msg, msg_len);
  if (st != PP_OK) return st;
  memset(out, 0, sizeof(*out));
  for (int i = 0; i < w->n_ours + w->n_theirs; ++i) { /* pass_eval.cpp:279-283 */
    if (!all[i].finite) continue;
    int32_t* has = all[i].team == 0 ? &out->has_our : &out->has_their;
    double* t = all[i].team == 0 ? &out->our_time : &out->their_time;
    if (!*has || all[i].time < *t) {
      *has = 1;
      *t = all[i].time;
    }
  }
  if (!out->has_our && !out->has_their) {
    out->side = 2;
  } else if (!out->has_their) {
    out->side = 0;
  } else if (!out->has_our) {
    out->side = 1;
  } else {
    const double delta = out->our_time - out->their_time;
    out->side = fabs(delta) <= p->thresholds.contest_epsilon ? 2 : (delta < 0.0 ? 0 : 1);
  }
  return PP_OK;
}

int or_decide_shot(const pp_world* w, const pp_params* p, int32_t shooter_id,
                   pp_shot_decision* out, char* msg, size_t msg_len) {
  const pp_robot* sh = NULL;
  for (int i = 0; i < w->n_ours; ++i)
    if (w->ours[i].id == shooter_id) sh = &w->ours[i];
  if (!sh) {
    put(msg, msg_len, "kicker id not on team ours");
    return PP_VALIDATION;
  }
  memset(out, 0, sizeof(*out));
  const int has_ball = dist2(sh->px, sh->py, w->ball_px, w->ball_py) <= p->thresholds.possession_radius;
  const double ox = has_ball ? w->ball_px : sh->px, oy = has_ball ? w->ball_py : sh->py;
  const double r = p->thresholds.robot_radius;
  const view_t v = goal_view(ox, oy, w, r);
  const double gx = 0.5 * w->field.length;
  out->shot_angle = v.angle;
  out->target_x = gx;
  out->target_y = v.ty;
  if (v.angle < p->thresholds.angle_threshold || v.angle <= 0.0) {
    out->reason = 0;
    out->blocked = 1;
    return PP_OK;
  }
  const double speed = p->thresholds.shot_power > 0.0 ? p->thresholds.shot_power : p->ball.power_max;
  const pp_kick kick = {ox, oy, gx - ox, v.ty - oy, speed, 0, 0};
  traj_t tr;
  const int st = kick_traj(&kick, &p->ball, &tr, msg, msg_len);
  if (st != PP_OK) return st;
  double t_goal;
  if (!travel_time(&tr, dist2(ox, oy, gx, v.ty), &t_goal)) {
    out->reason = 1;
    out->blocked = 1;
    return PP_OK;
  }
  const double dt = p->thresholds.sbip_dt;
  const window_t win = traj_window(&tr, &w->field, dt);
  for (int i = 0; i < w->n_theirs; ++i) { /* world.theirs in input order */
    const kin_t kin = make_kin(&w->theirs[i], &p->motion_theirs, r);
    const pp_intercept ir = intercept_with(&tr, dt, win, &kin);
    if (ir.finite && ir.time < t_goal) {
      out->reason = 1;
      out->blocked = 1;
      return PP_OK;
    }
  }
  out->shoot = 1;
  out->reason = 2;
  return PP_OK;
}

int or_plan_free_kick(const pp_world* w, const pp_params* p, int32_t kicker_id,
                      const pp_candidate* c, pp_free_kick_plan* out, char* msg, size_t msg_len) {
  char buf[160];
  if (!c->feasible) {
    put(msg, msg_len, "plan_free_kick: target candidate is not feasible");
    return PP_DOMAIN;
  }
  const pp_robot* kk = NULL;
  const pp_robot* rcv = NULL;
  for (int i = 0; i < w->n_ours; ++i) {
    if (w->ours[i].id == kicker_id) kk = &w->ours[i];
    if (w->ours[i].id == c->our_id && !rcv) rcv = &w->ours[i];
  }
  if (!kk) {
    snprintf(buf, sizeof(buf), "plan_free_kick: kicker id %d is not on team ours", kicker_id);
    put(msg, msg_len, buf);
    return PP_VALIDATION;
  }
  if (!rcv) {
    snprintf(buf, sizeof(buf), "plan_free_kick: receiver id %d is not on team ours", c->our_id);
    put(msg, msg_len, buf);
    return PP_VALIDATION;
  }
  const pp_search_grid* g = &p->grid;
  if (c->power_index < 0 || c->power_index >= g->n_powers) {
    put(msg, msg_len, "plan_free_kick: candidate power index outside the configured grid");
    return PP_DOMAIN;
  }
  const double power = power_of(c->power_index, g->n_powers, g->power_min, g->power_max);
  const double dx = c->receive_x - w->ball_px, dy = c->receive_y - w->ball_py;
  const pp_kick kick = {w->ball_px, w->ball_py, dx, dy, power, c->kick_type == 1 ? 1 : 0, 0};
  traj_t tr;
  const int st = kick_traj(&kick, &p->ball, &tr, msg, msg_len);
  if (st != PP_OK) return st;
  double t_ball;
  if (!travel_time(&tr, sqrt(dx * dx + dy * dy), &t_ball)) {
    put(msg, msg_len, "plan_free_kick: receive point beyond the ball's rollout");
    return PP_DOMAIN;
  }
  memset(out, 0, sizeof(*out));
  out->t_ball = t_ball;
  out->t_robot = arrival_time(rcv->px, rcv->py, rcv->vx, rcv->vy, c->receive_x, c->receive_y,
                              &p->motion_ours);
  out->order = out->t_robot <= out->t_ball ? 1 : 0;
  out->kick_delay = out->t_robot - out->t_ball > 0.0 ? out->t_robot - out->t_ball : 0.0;
  return PP_OK;
}
