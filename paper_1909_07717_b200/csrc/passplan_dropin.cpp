// passplan_dropin.cpp -- the reference's C++ API (include/passplan/passplan.hpp)
// implemented on the C-ABI of passplan_b200.h.  Built into lib/libpassplan.so.
//
// Hot-path calls (run_dpps, score_pass, best_pass, goal_view,
// score_running_point, best_running_points) go to the GPU; the rest are the
// reference's small closed forms on the host.  Compiled with
// -ffp-contract=off so the host-side arithmetic rounds like the reference.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "passplan/detail/pp_math.hpp"
#include "passplan/passplan.hpp"
#include "passplan_b200.h"

namespace passplan {

namespace {

// One C-ABI context per host thread (the reference's functions are
// re-entrant; a pp_ctx is single-threaded).
struct ThreadCtx {
  pp_ctx* ctx = nullptr;
  void* block = nullptr;  // scratch result block (run maps)
  size_t block_bytes = 0;
  // The last run_dpps of this thread: its result block (summary with the
  // fused best_pass for all / flat / chip, per-cell outputs) and the inputs
  // it was computed from.  best_pass on a grid that still matches it is
  // served from the summary without re-scoring (run_dpps then
  // best_pass x3 is the reference's own plan sequence).
  void* dpps_block = nullptr;
  size_t dpps_bytes = 0;
  bool dpps_valid = false;
  int64_t dpps_cells = 0;
  pp_world dpps_world;
  pp_params dpps_params;
  pp_search_grid dpps_grid;
  // direction_table / power_table of the last grid shape
  int dir_n = -1;
  std::vector<Vec2> dirs;
  int pow_n = -1;
  double pow_lo = 0.0, pow_hi = 0.0;
  std::vector<double> pows;
  ~ThreadCtx() {
    if (block) pp_host_free(block);
    if (dpps_block) pp_host_free(dpps_block);
    if (ctx) pp_ctx_destroy(ctx);
  }
};

thread_local ThreadCtx tl;

pp_ctx* context() {
  if (!tl.ctx) {
    const char* dev = std::getenv("PASSPLAN_DEVICE");
    const int device = dev ? std::atoi(dev) : 0;
    if (pp_ctx_create(device, &tl.ctx) != PP_OK || !tl.ctx) {
      tl.ctx = nullptr;
      throw internal_error("passplan: no usable CUDA device " + std::to_string(device) +
                           " (the sm_100a path has no CPU fallback)");
    }
  }
  return tl.ctx;
}

void* grow_pinned(void** p, size_t* have, size_t bytes) {
  if (bytes > *have) {
    if (*p) pp_host_free(*p);
    *p = pp_host_alloc(bytes);
    if (!*p) {
      *have = 0;
      throw internal_error("passplan: pinned host allocation failed");
    }
    *have = bytes;
  }
  return *p;
}

void* host_block(size_t bytes) { return grow_pinned(&tl.block, &tl.block_bytes, bytes); }

ErrorCategory category_of(pp_status st) {
  switch (st) {
    case PP_SCHEMA: return ErrorCategory::schema;
    case PP_VALIDATION: return ErrorCategory::validation;
    case PP_CONFIG: return ErrorCategory::config;
    case PP_DOMAIN: return ErrorCategory::domain;
    default: return ErrorCategory::internal;
  }
}

void check(pp_status st, pp_ctx* ctx) {
  if (st != PP_OK) throw Error(category_of(st), ctx ? pp_last_error(ctx) : "passplan error");
}

pp_robot to_pp(const RobotState& r) {
  pp_robot o{};
  o.id = r.id;
  o.px = r.position.x;
  o.py = r.position.y;
  o.vx = r.velocity.x;
  o.vy = r.velocity.y;
  o.theta = r.theta;
  return o;
}

pp_world to_pp(const WorldState& w) {
  if (w.ours.size() > PP_MAX_TEAM || w.theirs.size() > PP_MAX_TEAM)
    throw validation_error("more than 16 robots on a team");
  pp_world o;
  std::memset(&o, 0, sizeof(o));
  o.field = {w.field.length, w.field.width, w.field.goal_width, w.field.defense_depth,
             w.field.defense_width};
  o.ball_px = w.ball.position.x;
  o.ball_py = w.ball.position.y;
  o.ball_vx = w.ball.velocity.x;
  o.ball_vy = w.ball.velocity.y;
  o.n_ours = static_cast<int32_t>(w.ours.size());
  o.n_theirs = static_cast<int32_t>(w.theirs.size());
  for (size_t i = 0; i < w.ours.size(); ++i) o.ours[i] = to_pp(w.ours[i]);
  for (size_t i = 0; i < w.theirs.size(); ++i) o.theirs[i] = to_pp(w.theirs[i]);
  return o;
}

pp_search_grid to_pp(const SearchGrid& g) {
  return {g.n_directions, g.n_powers, g.power_min, g.power_max, g.flat ? 1 : 0, g.chip ? 1 : 0};
}

pp_params to_pp(const PlannerConfig& c) {
  pp_params p;
  std::memset(&p, 0, sizeof(p));
  p.ball = {c.ball.slide_decel, c.ball.roll_decel, c.ball.transition_ratio, c.ball.power_min,
            c.ball.power_max, c.ball.chip_flight_fraction};
  p.motion_ours = {c.motion_ours.max_speed, c.motion_ours.max_accel, c.motion_ours.max_decel};
  p.motion_theirs = {c.motion_theirs.max_speed, c.motion_theirs.max_accel,
                     c.motion_theirs.max_decel};
  p.grid = to_pp(c.grid);
  const PassWeights& pw = c.weights.pass;
  p.pass_weights = {pw.teammate_time, pw.shoot_angle, pw.dist_goal, pw.refraction, pw.margin};
  const RunWeights& rw = c.weights.run;
  p.run_weights = {rw.dist_goal, rw.dist_ball, rw.angle, rw.guard_time, rw.exposure};
  p.norm = {c.weights.norm.length_upper, c.weights.norm.angle_upper};
  p.angle_band = {c.angle_band.full_lo, c.angle_band.peak_lo, c.angle_band.peak_hi,
                  c.angle_band.full_hi};
  const PlannerThresholds& t = c.thresholds;
  p.thresholds = {t.sbip_dt,         t.robot_radius,    t.safety_margin,  t.buffer_time,
                  t.possession_radius, t.angle_threshold, t.shot_power,   t.margin_cap,
                  t.possession_dt,   t.contest_epsilon, t.grid_step,      t.min_zone_width,
                  t.guard_time_cap,  t.drag_v_min,      t.marking_radius};
  return p;
}

PassFeatures from_pp(const pp_pass_features& f) {
  return {f.teammate_intercept_time, f.shoot_angle_at_receive, f.dist_receive_to_goal,
          f.refraction_angle, f.intercept_margin};
}

RunningPointFeatures from_pp(const pp_run_features& f) {
  return {f.dist_to_goal, f.dist_to_ball, f.angle_to_goal, f.guard_time, f.defense_exposure};
}

int axis_count(double span, double step) {  // offball.cpp:69-74
  const int n = static_cast<int>(std::floor(span / step + 1e-9)) + 1;
  return n > 0 ? n : 0;
}

std::vector<double> axis_lattice(double anchor, double span, double direction, double step) {
  const int n = axis_count(span, step);
  std::vector<double> v(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) v[static_cast<size_t>(i)] = anchor + direction * (i * step);
  return v;
}

}  // namespace

// ---- host closed forms -------------------------------------------------------

double segment_distance(Vec2 p, Vec2 a, Vec2 b) {
  const Vec2 ab = b - a;
  const double len2 = ab.norm2();
  if (len2 == 0.0) return distance(p, a);
  double t = (p - a).dot(ab) / len2;
  t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  return distance(p, a + ab * t);
}

const char* category_name(ErrorCategory c) {
  switch (c) {
    case ErrorCategory::schema: return "schema";
    case ErrorCategory::validation: return "validation";
    case ErrorCategory::config: return "config";
    case ErrorCategory::domain: return "domain";
    case ErrorCategory::internal: return "internal";
  }
  return "internal";
}

int exit_code_for(ErrorCategory c) {
  switch (c) {
    case ErrorCategory::schema:
    case ErrorCategory::validation: return 2;
    case ErrorCategory::config: return 3;
    default: return 4;
  }
}

void FieldGeometry::validate() const {
  if (!(length > 0.0) || !(width > 0.0)) throw config_error("field dimensions must be positive");
  if (!(goal_width > 0.0) || goal_width > width) throw config_error("goal_width out of range");
  if (!(defense_depth > 0.0) || defense_depth > length)
    throw config_error("defense_depth out of range");
  if (!(defense_width > 0.0) || defense_width > width)
    throw config_error("defense_width out of range");
}

const RobotState* WorldState::find(Team t, int id) const {
  for (const RobotState& r : team(t))
    if (r.id == id) return &r;
  return nullptr;
}

void WorldState::validate() const {
  field.validate();
  const double hx = 0.5 * field.length + 0.5, hy = 0.5 * field.width + 0.5;
  auto inside = [&](Vec2 p) { return p.x >= -hx && p.x <= hx && p.y >= -hy && p.y <= hy; };
  if (!inside(ball.position)) throw validation_error("ball outside field bounds");
  for (const auto* team : {&ours, &theirs}) {
    const char* name = team == &ours ? "ours" : "theirs";
    if (team->size() > 16)
      throw validation_error(std::string(name) + ": more than 16 robots (" +
                             std::to_string(team->size()) + ")");
    std::set<int> ids;
    for (const RobotState& r : *team) {
      if (!ids.insert(r.id).second)
        throw validation_error(std::string(name) + ": duplicate robot id " + std::to_string(r.id));
      if (!inside(r.position))
        throw validation_error(std::string(name) + ": robot " + std::to_string(r.id) +
                               " outside field bounds");
      if (!(r.velocity.norm() <= 5.0))
        throw validation_error(std::string(name) + ": robot " + std::to_string(r.id) +
                               " faster than 5 m/s");
    }
  }
}

WorldState mirror_world(const WorldState& w) {
  WorldState m = w;
  m.ball.position.y = -m.ball.position.y;
  m.ball.velocity.y = -m.ball.velocity.y;
  for (auto* team : {&m.ours, &m.theirs}) {
    for (RobotState& r : *team) {
      r.position.y = -r.position.y;
      r.velocity.y = -r.velocity.y;
      r.theta = -r.theta;
    }
  }
  return m;
}

void BallModelParams::validate() const {
  pp_params p;
  pp_params_default(&p);
  p.ball = {slide_decel, roll_decel, transition_ratio, power_min, power_max, chip_flight_fraction};
  char msg[256];
  if (pp_params_validate(&p, msg, sizeof(msg)) != PP_OK) throw config_error(msg);
}

void MotionLimits::validate() const {
  if (!(max_speed > 0.0) || !(max_accel > 0.0) || !(max_decel > 0.0))
    throw config_error("motion limits must all be positive");
}

std::vector<KickType> SearchGrid::kick_types() const {
  std::vector<KickType> out;
  if (flat) out.push_back(KickType::flat);
  if (chip) out.push_back(KickType::chip);
  return out;
}

void SearchGrid::validate() const {
  if (n_directions < 1) throw config_error("grid.n_directions must be >= 1");
  if (n_powers < 1) throw config_error("grid.n_powers must be >= 1");
  if (!(power_min > 0.0) || !(power_min <= power_max))
    throw config_error("grid requires 0 < power_min <= power_max");
}

void PlannerConfig::validate() const {
  const pp_params p = to_pp(*this);
  char msg[256];
  if (pp_params_validate(&p, msg, sizeof(msg)) != PP_OK) throw config_error(msg);
}

std::vector<Vec2> direction_table(int n) {  // dpps.cpp:30-48 via pp_math.hpp
  std::vector<double> xy(2 * static_cast<size_t>(n));
  pp::direction_table_xy(n, xy.data());
  std::vector<Vec2> dirs(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) dirs[static_cast<size_t>(k)] = {xy[2 * k], xy[2 * k + 1]};
  return dirs;
}

std::vector<double> power_table(int n, double power_min, double power_max) {  // dpps.cpp:50-62
  std::vector<double> p(static_cast<size_t>(n));
  for (int j = 0; j < n; ++j) p[static_cast<size_t>(j)] = pp::power_at(j, n, power_min, power_max).v;
  return p;
}

std::vector<PassCandidate> feasible_candidates(const CandidateGrid& g) {
  std::vector<PassCandidate> out;
  for (const PassCandidate& c : g.cells)
    if (c.feasible) out.push_back(c);
  return out;
}

bool grids_identical(const CandidateGrid& a, const CandidateGrid& b) {
  if (a.cells.size() != b.cells.size()) return false;
  for (size_t i = 0; i < a.cells.size(); ++i) {
    const PassCandidate& x = a.cells[i];
    const PassCandidate& y = b.cells[i];
    if (x.kick_type != y.kick_type || x.dir_index != y.dir_index ||
        x.power_index != y.power_index || x.our_id != y.our_id || x.opp_id != y.opp_id ||
        x.feasible != y.feasible || x.our_time != y.our_time || x.opp_time != y.opp_time ||
        x.receive_point.x != y.receive_point.x || x.receive_point.y != y.receive_point.y)
      return false;
  }
  return true;
}

// ---- GPU path ------------------------------------------------------------------

CandidateGrid run_dpps(const WorldState& world, int kicker_id, const SearchGrid& grid,
                       const PlannerConfig& cfg, int workers) {
  grid.validate();
  cfg.validate();
  if (world.find(Team::ours, kicker_id) == nullptr)
    throw validation_error("kicker id " + std::to_string(kicker_id) + " is not on team ours");
  pp_ctx* ctx = context();
  const pp_world w = to_pp(world);
  const pp_params p = to_pp(cfg);
  const pp_search_grid g = to_pp(grid);
  const int64_t n = pp_grid_cells(&g);
  tl.dpps_valid = false;
  void* block = grow_pinned(&tl.dpps_block, &tl.dpps_bytes, pp_grid_bytes(n));
  const auto t0 = std::chrono::steady_clock::now();
  check(pp_dpps(ctx, &w, &p, &g, kicker_id, PP_COPY_ALL, block), ctx);
  const auto t1 = std::chrono::steady_clock::now();
  tl.dpps_valid = true;
  tl.dpps_cells = n;
  tl.dpps_world = w;
  tl.dpps_params = p;
  tl.dpps_grid = g;
  pp_grid_view v;
  pp_grid_view_of(block, n, &v);
  const pp_dpps_summary& s = *v.summary;

  CandidateGrid out;
  out.grid = grid;
  out.kicker_id = kicker_id;
  out.ball_origin = world.ball.position;
  out.kick_types = grid.kick_types();
  if (tl.dir_n != grid.n_directions) {
    tl.dirs = direction_table(grid.n_directions);
    tl.dir_n = grid.n_directions;
  }
  out.directions = tl.dirs;
  if (tl.pow_n != grid.n_powers || tl.pow_lo != grid.power_min || tl.pow_hi != grid.power_max) {
    tl.pows = power_table(grid.n_powers, grid.power_min, grid.power_max);
    tl.pow_n = grid.n_powers;
    tl.pow_lo = grid.power_min;
    tl.pow_hi = grid.power_max;
  }
  out.powers = tl.pows;
  // (cell order: kick slot, direction, power -- nested loops, no per-cell
  // index arithmetic; each cell written once)
  out.cells.reserve(static_cast<size_t>(n));
  const int nd = grid.n_directions, np = grid.n_powers;
  int ours_ids[PP_MAX_TEAM + 1], theirs_ids[PP_MAX_TEAM + 1];  // slot + 1 -> id (-1 = none)
  ours_ids[0] = theirs_ids[0] = -1;
  for (int k = 0; k < PP_MAX_TEAM; ++k) {
    ours_ids[k + 1] = s.ours_ids[k];
    theirs_ids[k + 1] = s.theirs_ids[k];
  }
  int64_t i = 0;
  for (const KickType kt : out.kick_types) {
    for (int d = 0; d < nd; ++d) {
      for (int pw = 0; pw < np; ++pw, ++i) {
        PassCandidate& c = out.cells.emplace_back();
        c.kick_type = kt;
        c.dir_index = d;
        c.power_index = pw;
        c.our_id = ours_ids[v.our_slot[i] + 1];
        c.opp_id = theirs_ids[v.opp_slot[i] + 1];
        c.our_time = v.our_time[i];
        c.opp_time = v.opp_time[i];
        if (c.our_time < kNever) c.receive_point = {v.rx[i], v.ry[i]};
        c.feasible = v.feasible[i] != 0;
      }
    }
  }
  out.telemetry.sbip_calls = s.sbip_calls;
  out.telemetry.wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  out.telemetry.workers = workers < 1 ? 1 : workers;
  out.telemetry.kernel = kernels::active_kernel().name;
  out.telemetry.kicker_in_possession = s.kicker_in_possession != 0;
  return out;
}

CandidateGrid run_dpps_serial(const WorldState& world, int kicker_id, const SearchGrid& grid,
                              const PlannerConfig& cfg) {
  return run_dpps(world, kicker_id, grid, cfg, 1);
}

GoalView goal_view(Vec2 point, const WorldState& world, double robot_radius) {
  pp_ctx* ctx = context();
  const pp_world w = to_pp(world);
  double a, lo, hi, ty;
  check(pp_goal_views(ctx, &w, robot_radius, 1, &point.x, &point.y, &a, &lo, &hi, &ty), ctx);
  GoalView v;
  v.angle = a;
  v.window_lo = lo;
  v.window_hi = hi;
  v.target = {0.5 * world.field.length, ty};
  return v;
}

double shoot_angle(Vec2 point, const WorldState& world, double robot_radius) {
  return goal_view(point, world, robot_radius).angle;
}

std::pair<double, PassFeatures> score_pass(const PassCandidate& candidate, const WorldState& world,
                                           const PlannerConfig& cfg) {
  if (!candidate.feasible) throw domain_error("score_pass: candidate is not feasible");
  pp_ctx* ctx = context();
  const pp_world w = to_pp(world);
  const pp_params p = to_pp(cfg);
  const uint8_t feas = 1;
  double score;
  pp_pass_features f;
  check(pp_score_cells(ctx, &w, &p, 1, &candidate.receive_point.x, &candidate.receive_point.y,
                       &candidate.our_time, &candidate.opp_time, &feas, &score, &f),
        ctx);
  return {score, from_pp(f)};
}

namespace {

// best_pass served from this thread's last run_dpps summary when `g` is still
// that run's grid (same shape, every cell's feasibility and, for feasible
// cells, the receive point and both times as computed) and world/cfg are the
// inputs it ran on; false otherwise.  One pass over the cells, no GPU work.
bool cached_best_pass(const CandidateGrid& g, const WorldState& world, const PlannerConfig& cfg,
                      std::optional<KickType> only, std::optional<ScoredPass>* out) {
  if (!tl.dpps_valid || static_cast<int64_t>(g.cells.size()) != tl.dpps_cells) return false;
  const pp_search_grid gg = to_pp(g.grid);
  if (std::memcmp(&gg, &tl.dpps_grid, sizeof(gg)) != 0) return false;
  if (g.kick_types != g.grid.kick_types()) return false;
  if (world.ours.size() > PP_MAX_TEAM || world.theirs.size() > PP_MAX_TEAM) return false;
  const pp_world w = to_pp(world);
  if (std::memcmp(&w, &tl.dpps_world, sizeof(w)) != 0) return false;
  const pp_params p = to_pp(cfg);
  if (std::memcmp(&p, &tl.dpps_params, sizeof(p)) != 0) return false;
  pp_grid_view v;
  pp_grid_view_of(tl.dpps_block, tl.dpps_cells, &v);
  const int nd = g.grid.n_directions, np = g.grid.n_powers;
  int64_t i = 0;
  for (const KickType kt : g.kick_types) {
    for (int d = 0; d < nd; ++d) {
      for (int pw = 0; pw < np; ++pw, ++i) {
        const PassCandidate& c = g.cells[static_cast<size_t>(i)];
        if (c.feasible != (v.feasible[i] != 0)) return false;
        if (c.feasible &&
            (c.kick_type != kt || c.dir_index != d || c.power_index != pw ||
             c.our_time != v.our_time[i] || c.opp_time != v.opp_time[i] ||
             c.receive_point.x != v.rx[i] || c.receive_point.y != v.ry[i]))
          return false;
      }
    }
  }
  const pp_dpps_summary& s = *v.summary;
  const int which = !only ? 0 : (*only == KickType::flat ? 1 : 2);
  const int64_t b = s.best_cell[which];
  if (b < 0) {
    out->reset();
  } else {
    *out = ScoredPass{g.cells[static_cast<size_t>(b)], s.best_score[which],
                      from_pp(s.best_features[which])};
  }
  return true;
}

}  // namespace

std::optional<ScoredPass> best_pass(const CandidateGrid& g, const WorldState& world,
                                    const PlannerConfig& cfg, std::optional<KickType> only) {
  std::optional<ScoredPass> cached;
  if (cached_best_pass(g, world, cfg, only, &cached)) return cached;
  std::vector<size_t> idx;
  for (size_t i = 0; i < g.cells.size(); ++i) {
    const PassCandidate& c = g.cells[i];
    if (c.feasible && (!only || c.kick_type == *only)) idx.push_back(i);
  }
  if (idx.empty()) return std::nullopt;
  const size_t n = idx.size();
  std::vector<double> rx(n), ry(n), ot(n), pt(n), score(n);
  std::vector<uint8_t> feas(n, 1);
  std::vector<pp_pass_features> feat(n);
  for (size_t k = 0; k < n; ++k) {
    const PassCandidate& c = g.cells[idx[k]];
    rx[k] = c.receive_point.x;
    ry[k] = c.receive_point.y;
    ot[k] = c.our_time;
    pt[k] = c.opp_time;
  }
  pp_ctx* ctx = context();
  const pp_world w = to_pp(world);
  const pp_params p = to_pp(cfg);
  check(pp_score_cells(ctx, &w, &p, static_cast<int64_t>(n), rx.data(), ry.data(), ot.data(),
                       pt.data(), feas.data(), score.data(), feat.data()),
        ctx);
  size_t best = 0;  // first strict max in cell order (pass_eval.cpp:178-185)
  for (size_t k = 1; k < n; ++k)
    if (score[k] > score[best]) best = k;
  return ScoredPass{g.cells[idx[best]], score[best], from_pp(feat[best])};
}

std::optional<ScoredPass> best_pass(const CandidateGrid& g, const WorldState& world,
                                    const PlannerConfig& cfg) {
  return best_pass(g, world, cfg, std::nullopt);
}

// ---- running points ----------------------------------------------------------

const char* zone_name(ZoneLabel z) {
  switch (z) {
    case ZoneLabel::I: return "I";
    case ZoneLabel::II: return "II";
    case ZoneLabel::III: return "III";
    default: return "IV";
  }
}

std::optional<ZoneLabel> ZonePartition::label_at(Vec2 p) const {
  if (p.x < zones[0].x0 || p.x > zones[2].x1 || p.y < zones[1].y0 || p.y > zones[0].y1)
    return std::nullopt;
  if (p.x >= cut_x) return p.y >= cut_y ? ZoneLabel::III : ZoneLabel::IV;
  return p.y >= cut_y ? ZoneLabel::I : ZoneLabel::II;
}

ZonePartition partition_zones(const FieldGeometry& field, Vec2 ball, double min_zone_width) {
  if (!(min_zone_width > 0.0) || 2.0 * min_zone_width > field.width)
    throw config_error("min_zone_width must be positive and at most half the field width");
  ZonePartition part;
  part.cut_x = 0.25 * field.length;
  part.cut_y = std::clamp(ball.y, -0.5 * field.width + min_zone_width,
                          0.5 * field.width - min_zone_width);
  const double x_mid = 0.5 * field.length, y_top = 0.5 * field.width;
  part.zones[0] = {ZoneLabel::I, 0.0, part.cut_x, part.cut_y, y_top};
  part.zones[1] = {ZoneLabel::II, 0.0, part.cut_x, -y_top, part.cut_y};
  part.zones[2] = {ZoneLabel::III, part.cut_x, x_mid, part.cut_y, y_top};
  part.zones[3] = {ZoneLabel::IV, part.cut_x, x_mid, -y_top, part.cut_y};
  return part;
}

std::vector<Vec2> zone_lattice(const Zone& zone, double step) {
  if (!(step > 0.0)) throw config_error("lattice step must be positive");
  const bool upper = zone.label == ZoneLabel::I || zone.label == ZoneLabel::III;
  const auto xs = axis_lattice(zone.x0, zone.x1 - zone.x0, 1.0, step);
  const auto ys = upper ? axis_lattice(zone.y0, zone.y1 - zone.y0, 1.0, step)
                        : axis_lattice(zone.y1, zone.y1 - zone.y0, -1.0, step);
  std::vector<Vec2> out;
  out.reserve(xs.size() * ys.size());
  for (double x : xs)
    for (double y : ys) out.push_back({x, y});
  return out;
}

std::pair<double, RunningPointFeatures> score_running_point(Vec2 pt, const WorldState& world,
                                                            const PlannerConfig& cfg) {
  const FieldGeometry& f = world.field;
  if (!(pt.x >= 0.0 && pt.x <= 0.5 * f.length && std::fabs(pt.y) <= 0.5 * f.width))
    throw domain_error("running point outside the front-field region");
  if (f.strictly_in_their_defense_area(pt))
    throw domain_error("guard points undefined: point inside the defense area");
  pp_ctx* ctx = context();
  const pp_world w = to_pp(world);
  const pp_params p = to_pp(cfg);
  double score;
  pp_run_features feat;
  uint8_t ok = 0;
  check(pp_score_running_points(ctx, &w, &p, 1, &pt.x, &pt.y, &score, &feat, &ok), ctx);
  if (!ok) throw domain_error("running point not scorable");
  return {score, from_pp(feat)};
}

namespace {

// guard_points_kernel on one point: {P, Q} and the guard time.
std::pair<std::pair<Vec2, Vec2>, double> guard_query(Vec2 p, const WorldState& world,
                                                     const MotionLimits& limits, double cap) {
  pp_ctx* ctx = context();
  const pp_world w = to_pp(world);
  const pp_motion_limits lim{limits.max_speed, limits.max_accel, limits.max_decel};
  double pq[4];
  double t = 0.0;
  uint8_t ok = 0;
  check(pp_guard_points(ctx, &w, &lim, cap, 1, &p.x, &p.y, pq, &t, &ok), ctx);
  if (!ok) throw domain_error("guard points undefined: point inside the defense area");
  return {{{pq[0], pq[1]}, {pq[2], pq[3]}}, t};
}

}  // namespace

double guard_time(Vec2 p, const WorldState& world, const MotionLimits& limits, double cap) {
  if (!(cap > 0.0) || !std::isfinite(cap)) throw domain_error("guard time cap must be positive");
  return guard_query(p, world, limits, cap).second;
}

std::pair<Vec2, Vec2> guard_points(const FieldGeometry& field, Vec2 p) {
  WorldState w;  // no opponents: only the geometry is computed
  w.field = field;
  return guard_query(p, w, MotionLimits{}, 10.0).first;
}

std::vector<RunningPoint> best_running_points(const WorldState& world,
                                              const std::set<ZoneLabel>& occupied,
                                              const PlannerConfig& cfg, int n_runners,
                                              std::optional<Vec2> best_pass_point) {
  (void)partition_zones(world.field, world.ball.position, cfg.thresholds.min_zone_width);
  pp_ctx* ctx = context();
  const pp_world w = to_pp(world);
  const pp_params p = to_pp(cfg);
  pp_runmap_request req{};
  req.zone_mask = 0;
  for (ZoneLabel z : occupied) req.occupied_mask |= 1u << static_cast<int>(z);
  req.n_runners = n_runners;
  req.has_best_pass_point = best_pass_point ? 1 : 0;
  if (best_pass_point) {
    req.best_pass_px = best_pass_point->x;
    req.best_pass_py = best_pass_point->y;
  }
  req.want_map = 0;
  void* block = host_block(pp_runmap_bytes(0));
  check(pp_runmap(ctx, &w, &p, &req, block, 0), ctx);
  pp_runmap_view v;
  pp_runmap_view_of(block, 0, &v);
  std::vector<RunningPoint> out;
  for (int i = 0; i < v.summary->n_best; ++i) {
    const pp_running_point& rp = v.summary->best[v.summary->best_order[i]];
    out.push_back({static_cast<ZoneLabel>(rp.zone), {rp.px, rp.py}, rp.score, from_pp(rp.features)});
  }
  return out;
}

std::vector<FrameBest> best_pass_batch(const std::vector<WorldState>& frames,
                                       const std::vector<int>& kicker_ids, const SearchGrid& grid,
                                       const PlannerConfig& cfg) {
  grid.validate();
  cfg.validate();
  pp_ctx* ctx = context();
  std::vector<pp_world> w(frames.size());
  for (size_t i = 0; i < frames.size(); ++i) w[i] = to_pp(frames[i]);
  const pp_params p = to_pp(cfg);
  const pp_search_grid g = to_pp(grid);
  std::vector<pp_dpps_summary> sums(frames.size());
  check(pp_dpps_batch(ctx, w.data(), static_cast<int64_t>(w.size()), &p, &g,
                      kicker_ids.empty() ? nullptr : kicker_ids.data(), sums.data()),
        ctx);
  const int nd = grid.n_directions, np = grid.n_powers;
  const auto kts = grid.kick_types();
  std::vector<FrameBest> out(frames.size());
  for (size_t i = 0; i < frames.size(); ++i) {
    const pp_dpps_summary& s = sums[i];
    out[i].n_feasible = s.n_feasible[0];
    if (s.best_cell[0] < 0) continue;
    const int64_t c = s.best_cell[0];
    ScoredPass sp;
    sp.candidate.kick_type = kts[static_cast<size_t>(c / (int64_t(nd) * np))];
    sp.candidate.dir_index = static_cast<int>((c / np) % nd);
    sp.candidate.power_index = static_cast<int>(c % np);
    sp.candidate.our_time = s.best_features[0].teammate_intercept_time;
    sp.candidate.feasible = true;
    sp.score = s.best_score[0];
    sp.features = from_pp(s.best_features[0]);
    out[i].best = sp;
  }
  return out;
}

// ---- ball trajectory (ball_model.cpp:12-146), host -------------------------------
// The closed forms come from the one shared restatement, pp_math.hpp (the same
// functions the kernels use); only argument checks and type mapping live here.
namespace {

BallTrajectory resolve_trajectory(Vec2 origin, Vec2 dir, double speed, KickType type,
                                  const BallModelParams& params, bool slide_phase) {
  params.validate();
  if (!(speed >= 0.0) || !std::isfinite(speed))
    throw domain_error("kick speed must be finite and non-negative");
  if (dir.norm() == 0.0 && speed > 0.0) throw domain_error("kick direction must be non-zero");
  const pp::BallPath b =
      pp::make_path(origin.x, origin.y, dir.x, dir.y, speed, type == KickType::chip, slide_phase,
                    params.slide_decel, params.roll_decel, params.transition_ratio,
                    params.chip_flight_fraction);
  BallTrajectory t;
  t.origin = origin;
  t.direction = {b.ux, b.uy};
  t.kick_speed = speed;
  t.kick_type = type;
  t.v1 = b.tr.v1.v;
  t.slide_decel = b.slide;
  t.roll_decel = b.roll;
  t.slide_end_time = b.tr.t_se.v;
  t.slide_end_distance = b.tr.d_se.v;
  t.stop_time = b.tr.t_stop.v;
  t.stop_distance = b.tr.d_stop.v;
  t.interceptable_from = b.tr.from.v;
  return t;
}

pp::Traj profile_of(const BallTrajectory& t) {
  pp::Traj p;
  p.speed = t.kick_speed;
  p.v1 = t.v1;
  p.t_se = t.slide_end_time;
  p.d_se = t.slide_end_distance;
  p.t_stop = t.stop_time;
  p.d_stop = t.stop_distance;
  p.from = t.interceptable_from;
  return p;
}

pp_trajectory to_pp(const BallTrajectory& t) {
  pp_trajectory o;
  std::memset(&o, 0, sizeof(o));
  o.origin_x = t.origin.x;
  o.origin_y = t.origin.y;
  o.dir_x = t.direction.x;
  o.dir_y = t.direction.y;
  o.kick_speed = t.kick_speed;
  o.v1 = t.v1;
  o.slide_decel = t.slide_decel;
  o.roll_decel = t.roll_decel;
  o.slide_end_time = t.slide_end_time;
  o.slide_end_distance = t.slide_end_distance;
  o.stop_time = t.stop_time;
  o.stop_distance = t.stop_distance;
  o.interceptable_from = t.interceptable_from;
  o.kick_type = t.kick_type == KickType::chip ? 1 : 0;
  return o;
}

InterceptResult from_pp(const pp_intercept& r) {
  InterceptResult o;
  o.team = r.team == 0 ? Team::ours : Team::theirs;
  o.robot_id = r.robot_id;
  if (r.finite) {
    o.intercept_time = r.time;
    o.intercept_point = {r.point_x, r.point_y};
  }
  return o;
}

void check_nonneg(double v, const char* what) {
  if (std::isnan(v) || v < 0.0) throw domain_error(what);
}

}  // namespace

BallTrajectory BallTrajectory::flat_kick(Vec2 origin, Vec2 dir, double speed,
                                         const BallModelParams& params) {
  return resolve_trajectory(origin, dir, speed, KickType::flat, params, true);
}

BallTrajectory BallTrajectory::chip_kick(Vec2 origin, Vec2 dir, double speed,
                                         const BallModelParams& params) {
  return resolve_trajectory(origin, dir, speed, KickType::chip, params, true);
}

BallTrajectory BallTrajectory::free_roll(Vec2 origin, Vec2 velocity,
                                         const BallModelParams& params) {
  return resolve_trajectory(origin, velocity, velocity.norm(), KickType::flat, params, false);
}

double BallTrajectory::speed_at(double t) const {
  return pp::speed_at(profile_of(*this), slide_decel, roll_decel, t).v;
}

double BallTrajectory::distance_at(double t) const {
  return pp::distance_at(profile_of(*this), slide_decel, roll_decel, t).v;
}

bool BallTrajectory::airborne_at(double t) const {
  return kick_type == KickType::chip && distance_at(t) < interceptable_from;
}

std::optional<double> BallTrajectory::travel_time_to_distance(double d) const {
  const double t = pp::travel_time_to_distance(profile_of(*this), slide_decel, roll_decel, d).v;
  if (std::isnan(t)) return std::nullopt;  // beyond the rollout
  return t;
}

std::optional<double> BallTrajectory::time_of_first_interceptable_point(double d) const {
  if (kick_type == KickType::chip && d < interceptable_from) return std::nullopt;
  return travel_time_to_distance(d);
}

BallSample ball_state_at(const BallTrajectory& traj, double t) {
  check_nonneg(t, "ball_state_at: t must be >= 0");
  return {traj.position_at(t), traj.speed_at(t), traj.airborne_at(t)};
}

std::optional<double> travel_time_to_distance(const BallTrajectory& traj, double d) {
  check_nonneg(d, "travel_time_to_distance: d must be >= 0");
  return traj.travel_time_to_distance(d);
}

std::optional<double> time_of_first_interceptable_point(const BallTrajectory& traj, double d) {
  check_nonneg(d, "time_of_first_interceptable_point: d must be >= 0");
  return traj.time_of_first_interceptable_point(d);
}

PassPower pass_power_for(double d, double t, const BallModelParams& params) {
  params.validate();  // ball_model.cpp:129-146
  if (!(d > 0.0) || !std::isfinite(d)) throw domain_error("pass_power_for: d must be > 0");
  if (!(t > 0.0) || !std::isfinite(t)) throw domain_error("pass_power_for: t must be > 0");
  PassPower p;
  p.v1 = pp::pass_power_v1(d, t, params.roll_decel).v;
  const double raw = p.v1 / params.transition_ratio;
  p.kick_speed = std::clamp(raw, params.power_min, params.power_max);
  p.clamped = p.kick_speed != raw;
  return p;
}

double arrival_time(const RobotState& robot, Vec2 target, const MotionLimits& limits) {
  return pp::arrival_time(robot.position.x, robot.position.y, robot.velocity.x, robot.velocity.y,
                          target.x, target.y, limits.max_accel, limits.max_decel,
                          limits.max_speed)
      .v;
}

double arrival_time_with_buffer(const RobotState& robot, Vec2 target, const MotionLimits& limits,
                                double buffer) {
  check_nonneg(buffer, "arrival_time_with_buffer: buffer must be >= 0");
  return arrival_time(robot, target, limits) + buffer;
}

TrajectorySamples TrajectorySamples::build(const BallTrajectory& traj, double dt) {
  if (!(dt > 0.0)) throw domain_error("trajectory sampling requires dt > 0");
  TrajectorySamples s;
  s.dt = dt;
  const int n = static_cast<int>(std::floor(traj.stop_time / dt + 1e-9)) + 1;  // samples 0..k_last
  s.ts.reserve(static_cast<size_t>(n));
  s.ss.reserve(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) {
    s.ts.push_back(k * dt);
    s.ss.push_back(traj.distance_at(s.ts.back()));
  }
  return s;
}

std::optional<double> ray_exit_distance(const FieldGeometry& field, Vec2 origin, Vec2 u) {
  const double s = pp::ray_exit_distance(field.length, field.width, origin.x, origin.y, u.x, u.y).v;
  if (std::isnan(s)) return std::nullopt;  // origin outside the field
  return s;
}

// ---- the per-pair plug-in point (kernels/kernel.hpp) and the scan internals --------

namespace kernels {
namespace {

int scan_first_sm100a(const ScanBatch& b, const RobotKin& r) {
  pp_ctx* ctx = context();
  const pp_scan_batch pb{b.ts, b.ss, b.k_begin, b.k_end, b.ox, b.oy, b.ux, b.uy};
  const pp_robot_kin pk{r.px, r.py, r.vx, r.vy, r.accel, r.decel, r.vmax, r.radius, r.vbound};
  int32_t k = -1;
  check(pp_scan_first(ctx, 1, &pb, &pk, &k), ctx);
  return k;
}

}  // namespace

const KernelBackend& sm100a_kernel() {
  static const KernelBackend backend{pp_kernel_name(), &scan_first_sm100a};
  return backend;
}

const KernelBackend& active_kernel() { return sm100a_kernel(); }

std::vector<const KernelBackend*> available_kernels() { return {&sm100a_kernel()}; }

}  // namespace kernels

namespace detail_intercept {

// intercept.cpp:45-69: the in-field, landed part of the sampled trajectory.
ScanWindow scan_window(const BallTrajectory& traj, const TrajectorySamples& samples,
                       std::optional<double> d_exit) {
  ScanWindow w;
  if (!d_exit) return w;  // origin outside the field: nothing to scan
  w.k_end = samples.count();
  w.rest_in_field = !(*d_exit < traj.stop_distance);
  if (!w.rest_in_field) {
    const auto t_exit = traj.travel_time_to_distance(*d_exit);
    const int k_last = t_exit ? static_cast<int>(std::floor(*t_exit / samples.dt + 1e-9))
                              : samples.count() - 1;
    w.k_end = std::min(w.k_end, k_last + 1);
  }
  if (traj.interceptable_from > 0.0) {
    if (const auto t_air = traj.travel_time_to_distance(traj.interceptable_from))
      w.k_begin = static_cast<int>(std::ceil(*t_air / samples.dt - 1e-9));
  }
  return w;
}

// intercept.cpp:72-85
kernels::RobotKin make_kin(const RobotState& robot, const MotionLimits& limits,
                           double robot_radius) {
  kernels::RobotKin k;
  k.px = robot.position.x;
  k.py = robot.position.y;
  k.vx = robot.velocity.x;
  k.vy = robot.velocity.y;
  k.accel = limits.max_accel;
  k.decel = limits.max_decel;
  k.vmax = limits.max_speed;
  k.radius = robot_radius;
  k.vbound = std::max(robot.velocity.norm(), limits.max_speed);
  return k;
}

// intercept.cpp:87-115: the whole-window prune (closest point of the scanned
// segment out of reach at the last sample time), the start skip (samples
// before (dmin - radius - 1e-9) / vbound fail the quick reject), then the
// backend's scan.
int scan_robot(const kernels::ScanBatch& batch, const kernels::RobotKin& kin,
               const kernels::KernelBackend& backend) {
  if (batch.k_begin >= batch.k_end) return -1;
  const double t_hi = batch.ts[batch.k_end - 1];
  const double s_lo = batch.ss[batch.k_begin], s_hi = batch.ss[batch.k_end - 1];
  const Vec2 a{batch.ox + batch.ux * s_lo, batch.oy + batch.uy * s_lo};
  const Vec2 b{batch.ox + batch.ux * s_hi, batch.oy + batch.uy * s_hi};
  const double dmin = segment_distance({kin.px, kin.py}, a, b);
  if (dmin - kin.radius > kin.vbound * t_hi) return -1;
  kernels::ScanBatch clipped = batch;
  if (kin.vbound > 0.0) {
    const double t_lo = (dmin - kin.radius - 1e-9) / kin.vbound;
    if (t_lo > 0.0) {
      clipped.k_begin = static_cast<int>(
          std::lower_bound(batch.ts + batch.k_begin, batch.ts + batch.k_end, t_lo) - batch.ts);
      if (clipped.k_begin >= clipped.k_end) return -1;
    }
  }
  return backend.scan_first(clipped, kin);
}

}  // namespace detail_intercept

// ---- interception, possession, shot, free kick (GPU via the C-ABI) ---------------

std::vector<InterceptResult> intercept_all(const WorldState& world, const BallTrajectory& traj,
                                           const MotionLimits& ours_limits,
                                           const MotionLimits& theirs_limits, double dt,
                                           double robot_radius) {
  if (!(dt > 0.0)) throw domain_error("intercept_all: dt must be > 0");
  pp_ctx* ctx = context();
  const pp_world w = to_pp(world);
  PlannerConfig cfg;
  cfg.motion_ours = ours_limits;
  cfg.motion_theirs = theirs_limits;
  cfg.thresholds.robot_radius = robot_radius;
  const pp_params p = to_pp(cfg);
  const pp_trajectory t = to_pp(traj);
  pp_intercept res[2 * PP_MAX_TEAM];
  check(pp_intercept_all(ctx, &w, &p, &t, dt, res), ctx);
  std::vector<InterceptResult> out;
  for (int i = 0; i < w.n_ours + w.n_theirs; ++i) out.push_back(from_pp(res[i]));
  return out;
}

InterceptResult intercept_time(const RobotState& robot, const BallTrajectory& traj,
                               const MotionLimits& limits, const FieldGeometry& field, double dt,
                               double robot_radius) {
  if (!(dt > 0.0)) throw domain_error("intercept_time: dt must be > 0");
  WorldState one;
  one.field = field;
  one.ours = {robot};
  const std::vector<InterceptResult> r =
      intercept_all(one, traj, limits, limits, dt, robot_radius);
  InterceptResult o = r.front();
  o.team = Team::ours;  // the reference leaves team at its default here
  return o;
}

PossessionReport possession(const WorldState& world, const PlannerConfig& cfg) {
  pp_ctx* ctx = context();
  const pp_world w = to_pp(world);
  const pp_params p = to_pp(cfg);
  pp_possession_report r;
  check(pp_possession(ctx, &w, &p, &r), ctx);
  PossessionReport o;
  o.side = r.side == 0 ? PossessionSide::ours
                       : (r.side == 1 ? PossessionSide::theirs : PossessionSide::contested);
  if (r.has_our) o.our_time = r.our_time;
  if (r.has_their) o.their_time = r.their_time;
  return o;
}

ShotDecision decide_shot(const RobotState& shooter, const WorldState& world,
                         const PlannerConfig& cfg) {
  // Only the shooter's position and the opponents enter (pass_eval.cpp:194-233):
  // hand the C-ABI a world whose one teammate is the shooter.
  WorldState w2 = world;
  w2.ours = {shooter};
  pp_ctx* ctx = context();
  const pp_world w = to_pp(w2);
  const pp_params p = to_pp(cfg);
  pp_shot_decision d;
  check(pp_decide_shot(ctx, &w, &p, shooter.id, &d), ctx);
  ShotDecision o;
  o.shoot = d.shoot != 0;
  o.blocked = d.blocked != 0;
  o.shot_angle = d.shot_angle;
  o.shot_target = {d.target_x, d.target_y};
  o.reason = d.reason == 0 ? ShotReason::angle_too_small
                           : (d.reason == 1 ? ShotReason::interceptable : ShotReason::clear);
  return o;
}

FreeKickPlan plan_free_kick(const WorldState& world, int kicker_id, const PassCandidate& target,
                            const PlannerConfig& cfg) {
  pp_ctx* ctx = context();
  const pp_world w = to_pp(world);
  const pp_params p = to_pp(cfg);
  pp_candidate c;
  std::memset(&c, 0, sizeof(c));
  c.kick_type = target.kick_type == KickType::chip ? 1 : 0;
  c.dir_index = target.dir_index;
  c.power_index = target.power_index;
  c.our_id = target.our_id;
  c.opp_id = target.opp_id;
  c.feasible = target.feasible ? 1 : 0;
  c.our_time = target.our_time;
  c.opp_time = target.opp_time;
  c.receive_x = target.receive_point.x;
  c.receive_y = target.receive_point.y;
  pp_free_kick_plan fk;
  check(pp_plan_free_kick(ctx, &w, &p, kicker_id, &c, &fk), ctx);
  FreeKickPlan o;
  o.t_ball = fk.t_ball;
  o.t_robot = fk.t_robot;
  o.order = fk.order == 1 ? KickOrder::kick_first : KickOrder::robot_first;
  o.kick_delay = fk.kick_delay;
  return o;
}

}  // namespace passplan
