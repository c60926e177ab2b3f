// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Compiled together with the UNMODIFIED reference sources under
// /root/reference/proj/src (see oracle/Makefile) into oracle/_ref/libpassplan_ref.so.
// It exposes the reference's own hot-path entry points behind the same POD
// structs as include/passplan_b200.h, so tests/golden/make_golden.py can dump
// golden vectors and bench.py's reference arm can time the stock CPU path.
// Nothing here is product code and the product never links it.
//
// Reference entry points wrapped (proj/include/passplan/...):
//   run_dpps / run_dpps_serial      dpps.hpp:90-96
//   best_pass (+ only)              pass_eval.hpp:55-60
//   score_pass / goal_view          pass_eval.hpp:34-44
//   score_running_point, best_running_points, zone_lattice, partition_zones
//                                   offball.hpp:46-99
//   oracles::random_world / lattice_world   tests/oracles.hpp:228-289
//   load_world_snapshot             snapshot.hpp:14

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "oracles.hpp"
#include "passplan/config.hpp"
#include "passplan/csv.hpp"
#include "passplan/intercept.hpp"
#include "passplan/dpps.hpp"
#include "passplan/errors.hpp"
#include "passplan/kernels/kernel.hpp"
#include "passplan/offball.hpp"
#include "passplan/pass_eval.hpp"
#include "passplan/snapshot.hpp"
#include "passplan_b200.h"
#include "passplan_b200_layout.h"

using namespace passplan;

namespace {

using Clock = std::chrono::steady_clock;

void put_msg(char* msg, size_t len, const std::string& s) {
  if (msg == nullptr || len == 0) return;
  std::snprintf(msg, len, "%s", s.c_str());
}

int status_of(ErrorCategory c) {
  switch (c) {
    case ErrorCategory::schema: return PP_SCHEMA;
    case ErrorCategory::validation: return PP_VALIDATION;
    case ErrorCategory::config: return PP_CONFIG;
    case ErrorCategory::domain: return PP_DOMAIN;
    case ErrorCategory::internal: return PP_INTERNAL;
  }
  return PP_INTERNAL;
}

template <typename F>
int guarded(char* msg, size_t len, F&& f) {
  try {
    f();
    return PP_OK;
  } catch (const Error& e) {
    put_msg(msg, len, e.what());
    return status_of(e.category());
  } catch (const std::exception& e) {
    put_msg(msg, len, e.what());
    return PP_INTERNAL;
  }
}

RobotState to_robot(const pp_robot& r) {
  RobotState s;
  s.id = r.id;
  s.position = {r.px, r.py};
  s.velocity = {r.vx, r.vy};
  s.theta = r.theta;
  return s;
}

pp_robot from_robot(const RobotState& s) {
  pp_robot r{};
  r.id = s.id;
  r.px = s.position.x;
  r.py = s.position.y;
  r.vx = s.velocity.x;
  r.vy = s.velocity.y;
  r.theta = s.theta;
  return r;
}

WorldState to_world(const pp_world& w) {
  WorldState s;
  s.field.length = w.field.length;
  s.field.width = w.field.width;
  s.field.goal_width = w.field.goal_width;
  s.field.defense_depth = w.field.defense_depth;
  s.field.defense_width = w.field.defense_width;
  s.ball.position = {w.ball_px, w.ball_py};
  s.ball.velocity = {w.ball_vx, w.ball_vy};
  for (int i = 0; i < w.n_ours; ++i) s.ours.push_back(to_robot(w.ours[i]));
  for (int i = 0; i < w.n_theirs; ++i) s.theirs.push_back(to_robot(w.theirs[i]));
  return s;
}

void from_world(const WorldState& s, pp_world* w) {
  std::memset(w, 0, sizeof(*w));
  w->field = {s.field.length, s.field.width, s.field.goal_width, s.field.defense_depth,
              s.field.defense_width};
  w->ball_px = s.ball.position.x;
  w->ball_py = s.ball.position.y;
  w->ball_vx = s.ball.velocity.x;
  w->ball_vy = s.ball.velocity.y;
  w->n_ours = static_cast<int32_t>(s.ours.size());
  w->n_theirs = static_cast<int32_t>(s.theirs.size());
  for (size_t i = 0; i < s.ours.size() && i < PP_MAX_TEAM; ++i) w->ours[i] = from_robot(s.ours[i]);
  for (size_t i = 0; i < s.theirs.size() && i < PP_MAX_TEAM; ++i)
    w->theirs[i] = from_robot(s.theirs[i]);
}

SearchGrid to_grid(const pp_search_grid& g) {
  SearchGrid s;
  s.n_directions = g.n_directions;
  s.n_powers = g.n_powers;
  s.power_min = g.power_min;
  s.power_max = g.power_max;
  s.flat = g.flat != 0;
  s.chip = g.chip != 0;
  return s;
}

PlannerConfig to_config(const pp_params& p) {
  PlannerConfig c;
  c.ball.slide_decel = p.ball.slide_decel;
  c.ball.roll_decel = p.ball.roll_decel;
  c.ball.transition_ratio = p.ball.transition_ratio;
  c.ball.power_min = p.ball.power_min;
  c.ball.power_max = p.ball.power_max;
  c.ball.chip_flight_fraction = p.ball.chip_flight_fraction;
  c.motion_ours = {p.motion_ours.max_speed, p.motion_ours.max_accel, p.motion_ours.max_decel};
  c.motion_theirs = {p.motion_theirs.max_speed, p.motion_theirs.max_accel,
                     p.motion_theirs.max_decel};
  c.grid = to_grid(p.grid);
  const pp_pass_weights& pw = p.pass_weights;
  c.weights.pass = {pw.teammate_time, pw.shoot_angle, pw.dist_goal, pw.refraction, pw.margin};
  const pp_run_weights& rw = p.run_weights;
  c.weights.run = {rw.dist_goal, rw.dist_ball, rw.angle, rw.guard_time, rw.exposure};
  c.weights.norm = {p.norm.length_upper, p.norm.angle_upper};
  c.angle_band = {p.angle_band.full_lo, p.angle_band.peak_lo, p.angle_band.peak_hi,
                  p.angle_band.full_hi};
  const pp_thresholds& t = p.thresholds;
  PlannerThresholds& o = c.thresholds;
  o.sbip_dt = t.sbip_dt;
  o.robot_radius = t.robot_radius;
  o.safety_margin = t.safety_margin;
  o.buffer_time = t.buffer_time;
  o.possession_radius = t.possession_radius;
  o.angle_threshold = t.angle_threshold;
  o.shot_power = t.shot_power;
  o.margin_cap = t.margin_cap;
  o.possession_dt = t.possession_dt;
  o.contest_epsilon = t.contest_epsilon;
  o.grid_step = t.grid_step;
  o.min_zone_width = t.min_zone_width;
  o.guard_time_cap = t.guard_time_cap;
  o.drag_v_min = t.drag_v_min;
  o.marking_radius = t.marking_radius;
  return c;
}

pp_pass_features to_features(const PassFeatures& f) {
  return {f.teammate_intercept_time, f.shoot_angle_at_receive, f.dist_receive_to_goal,
          f.refraction_angle, f.intercept_margin};
}

int slot_of(const std::vector<RobotState>& team, int id, int32_t* sorted_ids, int* n_out) {
  std::vector<int> ids;
  for (const auto& r : team) ids.push_back(r.id);
  std::sort(ids.begin(), ids.end());
  int slot = -1;
  for (size_t i = 0; i < ids.size(); ++i) {
    if (sorted_ids != nullptr && i < PP_MAX_TEAM) sorted_ids[i] = ids[i];
    if (ids[i] == id) slot = static_cast<int>(i);
  }
  if (n_out != nullptr) *n_out = static_cast<int>(ids.size());
  return slot;
}

void fill_grid_block(const CandidateGrid& g, const WorldState& w, const PlannerConfig& cfg,
                     void* block) {
  const int64_t n = static_cast<int64_t>(g.cells.size());
  pp_grid_view v;
  pp_grid_view_of_(block, n, &v);
  pp_dpps_summary& s = *v.summary;
  std::memset(&s, 0, sizeof(s));
  s.n_cells = n;
  s.n_kick_types = static_cast<int32_t>(g.kick_types.size());
  for (size_t i = 0; i < g.kick_types.size(); ++i)
    s.kick_types[i] = g.kick_types[i] == KickType::flat ? 0 : 1;
  s.n_directions = g.grid.n_directions;
  s.n_powers = g.grid.n_powers;
  s.kicker_id = g.kicker_id;
  int n_ours = 0, n_theirs = 0;
  s.kicker_slot = slot_of(w.ours, g.kicker_id, s.ours_ids, &n_ours);
  slot_of(w.theirs, -1, s.theirs_ids, &n_theirs);
  s.n_ours = n_ours;
  s.n_theirs = n_theirs;
  s.kicker_in_possession = g.telemetry.kicker_in_possession ? 1 : 0;
  s.sbip_calls = g.telemetry.sbip_calls;
  s.device_ms = g.telemetry.wall_ms;
  auto slot_for = [](const int32_t* ids, int n_ids, int id) -> int8_t {
    if (id < 0) return -1;
    for (int i = 0; i < n_ids; ++i)
      if (ids[i] == id) return static_cast<int8_t>(i);
    return -1;
  };
  for (int64_t i = 0; i < n; ++i) {
    const PassCandidate& c = g.cells[i];
    v.our_time[i] = c.our_time;
    v.opp_time[i] = c.opp_time;
    v.rx[i] = c.receive_point.x;
    v.ry[i] = c.receive_point.y;
    v.our_slot[i] = slot_for(s.ours_ids, n_ours, c.our_id);
    v.opp_slot[i] = slot_for(s.theirs_ids, n_theirs, c.opp_id);
    v.feasible[i] = c.feasible ? 1 : 0;
    v.score[i] = -std::numeric_limits<float>::infinity();
    if (c.feasible) {
      v.score[i] = static_cast<float>(score_pass(c, w, cfg).first);
      s.n_feasible[0]++;
      s.n_feasible[c.kick_type == KickType::flat ? 1 : 2]++;
    }
  }
  const std::optional<KickType> which[3] = {std::nullopt, KickType::flat, KickType::chip};
  for (int k = 0; k < 3; ++k) {
    s.best_cell[k] = -1;
    const auto b = best_pass(g, w, cfg, which[k]);
    if (!b) continue;
    int slot = 0;
    for (size_t t = 0; t < g.kick_types.size(); ++t)
      if (g.kick_types[t] == b->candidate.kick_type) slot = static_cast<int>(t);
    s.best_cell[k] = g.cell_index(slot, b->candidate.dir_index, b->candidate.power_index);
    s.best_score[k] = b->score;
    s.best_features[k] = to_features(b->features);
  }
}

int nearest_teammate(const WorldState& w) {
  int id = w.ours.empty() ? -1 : w.ours[0].id;
  double best = std::numeric_limits<double>::infinity();
  for (const RobotState& r : w.ours) {
    const double d = distance(r.position, w.ball.position);
    if (d < best) {
      best = d;
      id = r.id;
    }
  }
  return id;
}

int axis_count(double span, double step) {
  const int n = static_cast<int>(std::floor(span / step + 1e-9)) + 1;
  return n > 0 ? n : 0;
}

}  // namespace

extern "C" {

const char* ref_kernel_name(void) { return kernels::active_kernel().name; }

int ref_dpps(const pp_world* world, const pp_params* params, const pp_search_grid* grid,
             int32_t kicker_id, int32_t workers, void* block, char* msg, size_t msg_len) {
  return guarded(msg, msg_len, [&] {
    const WorldState w = to_world(*world);
    const PlannerConfig cfg = to_config(*params);
    const SearchGrid sg = to_grid(grid ? *grid : params->grid);
    const CandidateGrid g = workers <= 0 ? run_dpps_serial(w, kicker_id, sg, cfg)
                                         : run_dpps(w, kicker_id, sg, cfg, workers);
    fill_grid_block(g, w, cfg, block);
  });
}

int ref_score_cells(const pp_world* world, const pp_params* params, int64_t n, const double* rx,
                    const double* ry, const double* our_time, const double* opp_time,
                    const uint8_t* feasible, double* score_out, pp_pass_features* feat_out,
                    char* msg, size_t msg_len) {
  return guarded(msg, msg_len, [&] {
    const WorldState w = to_world(*world);
    const PlannerConfig cfg = to_config(*params);
    for (int64_t i = 0; i < n; ++i) {
      PassCandidate c;
      c.receive_point = {rx[i], ry[i]};
      c.our_time = our_time[i];
      c.opp_time = opp_time[i];
      c.feasible = feasible[i] != 0;
      const auto [score, f] = score_pass(c, w, cfg);
      score_out[i] = score;
      if (feat_out) feat_out[i] = to_features(f);
    }
  });
}

int ref_goal_views(const pp_world* world, double radius, int64_t n, const double* px,
                   const double* py, double* angle, double* lo, double* hi, double* ty) {
  return guarded(nullptr, 0, [&] {
    const WorldState w = to_world(*world);
    for (int64_t i = 0; i < n; ++i) {
      const GoalView v = goal_view({px[i], py[i]}, w, radius);
      angle[i] = v.angle;
      lo[i] = v.window_lo;
      hi[i] = v.window_hi;
      ty[i] = v.target.y;
    }
  });
}

int64_t ref_runmap_count(const pp_world* world, const pp_params* params, uint32_t zone_mask) {
  const WorldState w = to_world(*world);
  const PlannerConfig cfg = to_config(*params);
  const ZonePartition part =
      partition_zones(w.field, w.ball.position, cfg.thresholds.min_zone_width);
  int64_t total = 0;
  for (int z = 0; z < 4; ++z) {
    if (!(zone_mask & (1u << z))) continue;
    total += static_cast<int64_t>(
        zone_lattice(part.zones[z], cfg.thresholds.grid_step).size());
  }
  return total;
}

int ref_runmap(const pp_world* world, const pp_params* params, const pp_runmap_request* req,
               void* block, int64_t block_vertices, char* msg, size_t msg_len) {
  return guarded(msg, msg_len, [&] {
    const WorldState w = to_world(*world);
    const PlannerConfig cfg = to_config(*params);
    const ZonePartition part =
        partition_zones(w.field, w.ball.position, cfg.thresholds.min_zone_width);
    pp_runmap_view v;
    pp_runmap_view_of_(block, block_vertices, &v);
    pp_runmap_summary& s = *v.summary;
    std::memset(&s, 0, sizeof(s));
    s.cut_x = part.cut_x;
    s.cut_y = part.cut_y;
    int64_t at = 0;
    for (int z = 0; z < 4; ++z) {
      s.zone_offset[z] = at;
      if (!(req->zone_mask & (1u << z))) continue;
      const Zone& zone = part.zones[z];
      s.zone_nx[z] = axis_count(zone.x1 - zone.x0, cfg.thresholds.grid_step);
      s.zone_ny[z] = axis_count(zone.y1 - zone.y0, cfg.thresholds.grid_step);
      const std::vector<Vec2> lat = zone_lattice(zone, cfg.thresholds.grid_step);
      for (const Vec2& p : lat) {
        if (at >= block_vertices) throw internal_error("runmap block too small");
        v.px[at] = p.x;
        v.py[at] = p.y;
        try {
          const auto [score, ft] = score_running_point(p, w, cfg);
          v.score[at] = score;
          v.features[at] = {ft.dist_to_goal, ft.dist_to_ball, ft.angle_to_goal, ft.guard_time,
                            ft.defense_exposure};
          v.scorable[at] = 1;
          s.n_scorable++;
        } catch (const Error&) {
          v.score[at] = std::numeric_limits<double>::quiet_NaN();
          v.features[at] = {0, 0, 0, 0, 0};
          v.scorable[at] = 0;
        }
        ++at;
      }
    }
    s.n_vertices = at;
    std::set<ZoneLabel> occupied;
    for (int z = 0; z < 4; ++z)
      if (req->occupied_mask & (1u << z)) occupied.insert(static_cast<ZoneLabel>(z));
    std::optional<Vec2> bp;
    if (req->has_best_pass_point) bp = Vec2{req->best_pass_px, req->best_pass_py};
    const auto best = best_running_points(w, occupied, cfg, req->n_runners, bp);
    s.n_best = static_cast<int32_t>(best.size());
    for (size_t i = 0; i < best.size(); ++i) {
      const RunningPoint& rp = best[i];
      const int z = static_cast<int>(rp.zone);
      s.best_order[i] = z;
      pp_running_point& o = s.best[z];
      o.zone = z;
      o.valid = 1;
      o.px = rp.point.x;
      o.py = rp.point.y;
      o.score = rp.score;
      o.features = {rp.features.dist_to_goal, rp.features.dist_to_ball, rp.features.angle_to_goal,
                    rp.features.guard_time, rp.features.defense_exposure};
    }
  });
}

int ref_random_world(uint64_t seed, int32_t n_ours, int32_t n_theirs, double ball_speed_max,
                     pp_world* out) {
  return guarded(nullptr, 0, [&] {
    std::mt19937_64 rng(seed);
    from_world(oracles::random_world(rng, n_ours, n_theirs, ball_speed_max), out);
  });
}

int ref_lattice_world(uint64_t seed, int32_t n_ours, int32_t n_theirs, int32_t rolling,
                      pp_world* out) {
  return guarded(nullptr, 0, [&] {
    std::mt19937_64 rng(seed);
    from_world(oracles::lattice_world(rng, n_ours, n_theirs, rolling != 0), out);
  });
}

int ref_mirror_world(const pp_world* in, pp_world* out) {
  return guarded(nullptr, 0, [&] { from_world(mirror_world(to_world(*in)), out); });
}

int ref_load_snapshot(const char* path, pp_world* out, char* msg, size_t msg_len) {
  return guarded(msg, msg_len, [&] { from_world(load_world_snapshot(path), out); });
}

int ref_validate_world(const pp_world* world, char* msg, size_t msg_len) {
  return guarded(msg, msg_len, [&] { to_world(*world).validate(); });
}

int ref_validate_params(const pp_params* params, char* msg, size_t msg_len) {
  return guarded(msg, msg_len, [&] { to_config(*params).validate(); });
}

void ref_params_default(pp_params* p) {
  const PlannerConfig c;
  std::memset(p, 0, sizeof(*p));
  p->ball = {c.ball.slide_decel, c.ball.roll_decel, c.ball.transition_ratio, c.ball.power_min,
             c.ball.power_max, c.ball.chip_flight_fraction};
  p->motion_ours = {c.motion_ours.max_speed, c.motion_ours.max_accel, c.motion_ours.max_decel};
  p->motion_theirs = {c.motion_theirs.max_speed, c.motion_theirs.max_accel,
                      c.motion_theirs.max_decel};
  p->grid = {c.grid.n_directions, c.grid.n_powers, c.grid.power_min, c.grid.power_max,
             c.grid.flat ? 1 : 0, c.grid.chip ? 1 : 0};
  const PassWeights& pw = c.weights.pass;
  p->pass_weights = {pw.teammate_time, pw.shoot_angle, pw.dist_goal, pw.refraction, pw.margin};
  const RunWeights& rw = c.weights.run;
  p->run_weights = {rw.dist_goal, rw.dist_ball, rw.angle, rw.guard_time, rw.exposure};
  p->norm = {c.weights.norm.length_upper, c.weights.norm.angle_upper};
  p->angle_band = {c.angle_band.full_lo, c.angle_band.peak_lo, c.angle_band.peak_hi,
                   c.angle_band.full_hi};
  const PlannerThresholds& t = c.thresholds;
  p->thresholds = {t.sbip_dt,        t.robot_radius,    t.safety_margin, t.buffer_time,
                   t.possession_radius, t.angle_threshold, t.shot_power,  t.margin_cap,
                   t.possession_dt,  t.contest_epsilon, t.grid_step,     t.min_zone_width,
                   t.guard_time_cap, t.drag_v_min,      t.marking_radius};
}

void ref_direction_table(int32_t n, double* xy) {
  const auto d = direction_table(n);
  for (int32_t i = 0; i < n; ++i) {
    xy[2 * i] = d[i].x;
    xy[2 * i + 1] = d[i].y;
  }
}

int32_t ref_nearest_teammate(const pp_world* world) { return nearest_teammate(to_world(*world)); }

// One frame as the CLI `plan` path runs it: run_dpps(workers) + best_pass.
// Per-rep wall times (ms) of the search and of best_pass.
int ref_time_frame(const pp_world* world, const pp_params* params, const pp_search_grid* grid,
                   int32_t kicker_id, int32_t workers, int32_t reps, double* search_ms,
                   double* best_ms, char* msg, size_t msg_len) {
  return guarded(msg, msg_len, [&] {
    const WorldState w = to_world(*world);
    const PlannerConfig cfg = to_config(*params);
    const SearchGrid sg = to_grid(grid ? *grid : params->grid);
    for (int r = 0; r < reps; ++r) {
      auto t0 = Clock::now();
      const CandidateGrid g = workers <= 0 ? run_dpps_serial(w, kicker_id, sg, cfg)
                                           : run_dpps(w, kicker_id, sg, cfg, workers);
      auto t1 = Clock::now();
      const auto b = best_pass(g, w, cfg);
      auto t2 = Clock::now();
      (void)b;
      search_ms[r] = std::chrono::duration<double, std::milli>(t1 - t0).count();
      best_ms[r] = std::chrono::duration<double, std::milli>(t2 - t1).count();
    }
  });
}

// Frame-parallel throughput: `threads` host threads each take whole frames
// (run_dpps_serial + best_pass, the reference's best CPU throughput shape).
int ref_batch(const pp_world* frames, int64_t n_frames, const pp_params* params,
              const pp_search_grid* grid, const int32_t* kicker_ids, int32_t threads,
              int64_t* best_cell, double* best_score, int64_t* n_feasible, double* wall_ms,
              char* msg, size_t msg_len) {
  return guarded(msg, msg_len, [&] {
    const PlannerConfig cfg = to_config(*params);
    const SearchGrid sg = to_grid(grid ? *grid : params->grid);
    std::atomic<int64_t> next{0};
    std::atomic<int> failed{0};
    auto work = [&] {
      for (;;) {
        const int64_t i = next.fetch_add(1);
        if (i >= n_frames) break;
        try {
          const WorldState w = to_world(frames[i]);
          const int kicker = kicker_ids ? kicker_ids[i] : nearest_teammate(w);
          const CandidateGrid g = run_dpps_serial(w, kicker, sg, cfg);
          const auto b = best_pass(g, w, cfg);
          int64_t nf = 0;
          for (const auto& c : g.cells) nf += c.feasible ? 1 : 0;
          if (n_feasible) n_feasible[i] = nf;
          if (b) {
            int slot = 0;
            for (size_t t = 0; t < g.kick_types.size(); ++t)
              if (g.kick_types[t] == b->candidate.kick_type) slot = static_cast<int>(t);
            if (best_cell)
              best_cell[i] = g.cell_index(slot, b->candidate.dir_index, b->candidate.power_index);
            if (best_score) best_score[i] = b->score;
          } else {
            if (best_cell) best_cell[i] = -1;
            if (best_score) best_score[i] = 0.0;
          }
        } catch (...) {
          failed.store(1);
        }
      }
    };
    const int nt = threads < 1 ? 1 : threads;
    const auto t0 = Clock::now();
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    *wall_ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
    if (failed.load()) throw internal_error("a frame failed in ref_batch");
  });
}

}  // extern "C"

// ---- §8(f) rows: interception, possession, shot, free kick, CSV ---------
//   intercept_all    intercept.hpp:50-53      possession      pass_eval.hpp:104
//   decide_shot      pass_eval.hpp:76-77      plan_free_kick  pass_eval.hpp:90-91
//   grid_to_csv / heatmap_to_csv / run_heatmap_to_csv         csv.hpp:22-52
namespace {

BallTrajectory to_trajectory(const pp_kick& k, const BallModelParams& b) {
  const Vec2 o{k.origin_x, k.origin_y}, d{k.dir_x, k.dir_y};
  if (k.kind == 2) return BallTrajectory::free_roll(o, d, b);
  if (k.kind == 1) return BallTrajectory::chip_kick(o, d, k.speed, b);
  return BallTrajectory::flat_kick(o, d, k.speed, b);
}

PassCandidate to_candidate(const pp_candidate& c) {
  PassCandidate p;
  p.kick_type = c.kick_type == 1 ? KickType::chip : KickType::flat;
  p.dir_index = c.dir_index;
  p.power_index = c.power_index;
  p.our_id = c.our_id;
  p.opp_id = c.opp_id;
  p.feasible = c.feasible != 0;
  p.our_time = c.our_time;
  p.opp_time = c.opp_time;
  p.receive_point = {c.receive_x, c.receive_y};
  return p;
}

int64_t put_text(const std::string& s, char* buf, size_t len) {
  if (buf != nullptr && len > 0) {
    const size_t n = s.size() < len - 1 ? s.size() : len - 1;
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return static_cast<int64_t>(s.size());
}

}  // namespace

extern "C" {

int ref_intercept_all(const pp_world* world, const pp_params* params, const pp_kick* kick,
                      double dt, pp_intercept* out, char* msg, size_t msg_len) {
  return guarded(msg, msg_len, [&] {
    const WorldState w = to_world(*world);
    const PlannerConfig cfg = to_config(*params);
    const auto all = intercept_all(w, to_trajectory(*kick, cfg.ball), cfg.motion_ours,
                                   cfg.motion_theirs, dt, cfg.thresholds.robot_radius);
    for (size_t i = 0; i < all.size(); ++i) {
      pp_intercept& o = out[i];
      std::memset(&o, 0, sizeof(o));
      o.team = all[i].team == Team::ours ? 0 : 1;
      o.robot_id = all[i].robot_id;
      o.finite = all[i].finite() ? 1 : 0;
      if (all[i].finite()) {
        o.time = *all[i].intercept_time;
        o.point_x = all[i].intercept_point.x;
        o.point_y = all[i].intercept_point.y;
      }
    }
  });
}

int ref_possession(const pp_world* world, const pp_params* params, pp_possession_report* out,
                   char* msg, size_t msg_len) {
  return guarded(msg, msg_len, [&] {
    const PossessionReport r = possession(to_world(*world), to_config(*params));
    std::memset(out, 0, sizeof(*out));
    out->side = r.side == PossessionSide::ours ? 0 : (r.side == PossessionSide::theirs ? 1 : 2);
    out->has_our = r.our_time.has_value();
    out->has_their = r.their_time.has_value();
    out->our_time = r.our_time.value_or(0.0);
    out->their_time = r.their_time.value_or(0.0);
  });
}

int ref_decide_shot(const pp_world* world, const pp_params* params, int32_t shooter_id,
                    pp_shot_decision* out, char* msg, size_t msg_len) {
  return guarded(msg, msg_len, [&] {
    const WorldState w = to_world(*world);
    const RobotState* shooter = w.find(Team::ours, shooter_id);
    if (shooter == nullptr) throw validation_error("kicker id not on team ours");
    const ShotDecision d = decide_shot(*shooter, w, to_config(*params));
    std::memset(out, 0, sizeof(*out));
    out->shoot = d.shoot;
    out->blocked = d.blocked;
    out->reason = d.reason == ShotReason::angle_too_small ? 0
                  : d.reason == ShotReason::interceptable ? 1
                                                           : 2;
    out->shot_angle = d.shot_angle;
    out->target_x = d.shot_target.x;
    out->target_y = d.shot_target.y;
  });
}

int ref_plan_free_kick(const pp_world* world, const pp_params* params, int32_t kicker_id,
                       const pp_candidate* target, pp_free_kick_plan* out, char* msg,
                       size_t msg_len) {
  return guarded(msg, msg_len, [&] {
    const FreeKickPlan p =
        plan_free_kick(to_world(*world), kicker_id, to_candidate(*target), to_config(*params));
    std::memset(out, 0, sizeof(*out));
    out->t_ball = p.t_ball;
    out->t_robot = p.t_robot;
    out->order = p.order == KickOrder::kick_first ? 1 : 0;
    out->kick_delay = p.kick_delay;
  });
}

// guard_points + guard_time of the reference at n points (offball.cpp:125-174);
// ok[i] = 0 where either throws (point strictly inside the area).
int ref_guard_points(const pp_world* world, const pp_motion_limits* limits, double cap, int64_t n,
                     const double* px, const double* py, double* pq, double* t, uint8_t* ok,
                     char* msg, size_t msg_len) {
  return guarded(msg, msg_len, [&] {
    const WorldState w = to_world(*world);
    MotionLimits lim;
    lim.max_speed = limits->max_speed;
    lim.max_accel = limits->max_accel;
    lim.max_decel = limits->max_decel;
    for (int64_t i = 0; i < n; ++i) {
      try {
        const auto g = guard_points(w.field, {px[i], py[i]});
        pq[4 * i] = g.first.x;
        pq[4 * i + 1] = g.first.y;
        pq[4 * i + 2] = g.second.x;
        pq[4 * i + 3] = g.second.y;
        t[i] = guard_time({px[i], py[i]}, w, lim, cap);
        ok[i] = 1;
      } catch (const Error&) {
        ok[i] = 0;
      }
    }
  });
}

// JSON round trips of the reference: kind 0 = world snapshot (parse then
// serialize, snapshot.cpp), 1 = planner config (parse; a few values
// printed).  "ERROR <category>: <message>" when the reader throws.
int64_t ref_json_check(int32_t kind, const char* text, char* buf, size_t len) {
  std::string out;
  try {
    if (kind == 0) {
      out = serialize_world_snapshot(parse_world_snapshot(text));
    } else {
      const PlannerConfig c = PlannerConfig::from_json_text(text);
      char b[160];
      std::snprintf(b, sizeof b, "OK %.17g %.17g %d %d %.17g", c.ball.slide_decel,
                    c.thresholds.sbip_dt, c.grid.n_directions, c.grid.chip ? 1 : 0,
                    c.weights.pass.margin);
      out = b;
    }
  } catch (const Error& e) {
    out = std::string("ERROR ") + category_name(e.category()) + ": " + e.what();
  }
  return put_text(out, buf, len);
}

// CSV reader -> writer round trip of the reference (csv.cpp): kind 0 = grid,
// 1 = pass heat map, 2 = run heat map.  The output is the rewritten text, or
// "ERROR <category>: <message>" when the reader throws.
int64_t ref_csv_roundtrip(int32_t kind, const char* text, char* buf, size_t len) {
  std::string out;
  try {
    const std::string in(text);
    if (kind == 0) {
      out = grid_to_csv(grid_from_csv(in));
    } else if (kind == 1) {
      out = heatmap_to_csv(heatmap_from_csv(in));
    } else {
      out = run_heatmap_to_csv(run_heatmap_from_csv(in));
    }
  } catch (const Error& e) {
    out = std::string("ERROR ") + category_name(e.category()) + ": " + e.what();
  }
  return put_text(out, buf, len);
}

// kernels::scalar_kernel().scan_first of the reference for n (ray, robot)
// pairs (kernel.hpp:46-53); ts/ss per pair from the caller's arrays.
int ref_scan_first(int64_t n, const pp_scan_batch* batches, const pp_robot_kin* kins,
                   int32_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    kernels::ScanBatch b;
    b.ts = batches[i].ts;
    b.ss = batches[i].ss;
    b.k_begin = batches[i].k_begin;
    b.k_end = batches[i].k_end;
    b.ox = batches[i].ox;
    b.oy = batches[i].oy;
    b.ux = batches[i].ux;
    b.uy = batches[i].uy;
    kernels::RobotKin r;
    r.px = kins[i].px;
    r.py = kins[i].py;
    r.vx = kins[i].vx;
    r.vy = kins[i].vy;
    r.accel = kins[i].accel;
    r.decel = kins[i].decel;
    r.vmax = kins[i].vmax;
    r.radius = kins[i].radius;
    r.vbound = kins[i].vbound;
    out[i] = kernels::scalar_kernel().scan_first(b, r);
  }
  return 0;
}

// `passplan plan --out` CSV of one frame (passplan_main.cpp:89, csv.cpp:85-114).
// Returns the text length (buf gets a NUL-terminated copy, truncated to len).
int64_t ref_grid_csv(const pp_world* world, const pp_params* params, int32_t kicker_id,
                     char* buf, size_t len) {
  try {
    const PlannerConfig cfg = to_config(*params);
    const CandidateGrid g = run_dpps_serial(to_world(*world), kicker_id, cfg.grid, cfg);
    return put_text(grid_to_csv(g), buf, len);
  } catch (...) {
    return -1;
  }
}

// `passplan heatmap --mode pass` CSV (passplan_main.cpp:137-149).
int64_t ref_pass_heatmap_csv(const pp_world* world, const pp_params* params, int32_t kicker_id,
                             char* buf, size_t len) {
  try {
    const WorldState w = to_world(*world);
    const PlannerConfig cfg = to_config(*params);
    const CandidateGrid g = run_dpps_serial(w, kicker_id, cfg.grid, cfg);
    std::vector<HeatPoint> pts;
    for (const PassCandidate& c : g.cells) {
      if (!c.feasible) continue;
      pts.push_back({c.receive_point, score_pass(c, w, cfg).first});
    }
    return put_text(heatmap_to_csv(pts), buf, len);
  } catch (...) {
    return -1;
  }
}

// `passplan heatmap --mode run --zone <mask>` CSV (passplan_main.cpp:156-196);
// zone_mask bit z = ZoneLabel I..IV in that order.
int64_t ref_run_heatmap_csv(const pp_world* world, const pp_params* params, uint32_t zone_mask,
                            char* buf, size_t len) {
  try {
    const WorldState w = to_world(*world);
    const PlannerConfig cfg = to_config(*params);
    const ZonePartition part =
        partition_zones(w.field, w.ball.position, cfg.thresholds.min_zone_width);
    const ZoneLabel labels[4] = {ZoneLabel::I, ZoneLabel::II, ZoneLabel::III, ZoneLabel::IV};
    std::vector<RunHeatRow> rows;
    for (int z = 0; z < 4; ++z) {
      if (!(zone_mask & (1u << z))) continue;
      for (Vec2 v : zone_lattice(part.zone(labels[z]), cfg.thresholds.grid_step)) {
        try {
          const auto [score, ft] = score_running_point(v, w, cfg);
          rows.push_back({v, ft, score});
        } catch (const Error&) {
        }
      }
    }
    return put_text(run_heatmap_to_csv(rows), buf, len);
  } catch (...) {
    return -1;
  }
}

}  // extern "C"
