// test_dropin.cpp -- GPU parity tests of the C++ drop-in (libpassplan.so),
// written against the reference's API the way its own tests are
// (proj/tests/test_dpps.cpp, test_pass_eval.cpp, test_offball.cpp), with the
// plain-C oracle (oracle/pp_oracle.c, linked in under `or_` names) as the
// independent check.  Prints one line per check; exit code = failures.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <optional>
#include <random>
#include <string>
#include <vector>

#include "../../oracle/pp_oracle.h"
#include "passplan/dpps.hpp"
#include "passplan/errors.hpp"
#include "passplan/offball.hpp"
#include "passplan/pass_eval.hpp"
#include "passplan_b200_layout.h"

using namespace passplan;

namespace {

int g_fail = 0, g_pass = 0;

void check(bool ok, const std::string& what) {
  if (ok) {
    ++g_pass;
  } else {
    ++g_fail;
    std::printf("FAIL %s\n", what.c_str());
  }
}

template <typename F>
ErrorCategory category_of(F&& f, bool* threw) {
  *threw = false;
  try {
    f();
  } catch (const Error& e) {
    *threw = true;
    return e.category();
  }
  return ErrorCategory::internal;
}

// oracles::random_world's distribution (proj/tests/oracles.hpp:228-258)
WorldState random_world(std::mt19937_64& rng, int n_ours, int n_theirs, double ball_speed = 0.0) {
  WorldState w;
  std::uniform_real_distribution<double> ux(-6.0, 6.0), uy(-4.5, 4.5), uv(-2.0, 2.0);
  std::uniform_real_distribution<double> us(0.0, ball_speed > 0 ? ball_speed : 1.0), ua(-3.14, 3.14);
  for (int t = 0; t < 2; ++t) {
    auto& team = t == 0 ? w.ours : w.theirs;
    for (int i = 0; i < (t == 0 ? n_ours : n_theirs); ++i) {
      RobotState r;
      r.id = i;
      r.position = {ux(rng), uy(rng)};
      r.velocity = {uv(rng), uv(rng)};
      team.push_back(r);
    }
  }
  w.ball.position = {ux(rng), uy(rng)};
  if (ball_speed > 0.0) {
    const double s = us(rng), a = ua(rng);
    w.ball.velocity = {s * std::cos(a), s * std::sin(a)};
  }
  return w;
}

pp_world to_c(const WorldState& w) {
  pp_world o;
  std::memset(&o, 0, sizeof(o));
  o.field = {w.field.length, w.field.width, w.field.goal_width, w.field.defense_depth,
             w.field.defense_width};
  o.ball_px = w.ball.position.x;
  o.ball_py = w.ball.position.y;
  o.n_ours = static_cast<int>(w.ours.size());
  o.n_theirs = static_cast<int>(w.theirs.size());
  for (size_t i = 0; i < w.ours.size(); ++i)
    o.ours[i] = {w.ours[i].id, 0, w.ours[i].position.x, w.ours[i].position.y,
                 w.ours[i].velocity.x, w.ours[i].velocity.y, 0.0};
  for (size_t i = 0; i < w.theirs.size(); ++i)
    o.theirs[i] = {w.theirs[i].id, 0, w.theirs[i].position.x, w.theirs[i].position.y,
                   w.theirs[i].velocity.x, w.theirs[i].velocity.y, 0.0};
  return o;
}

// Oracle grid for the same inputs (default PlannerConfig).
std::vector<unsigned char> oracle_grid(const WorldState& w, int kicker, const SearchGrid& g) {
  pp_params p;
  or_params_default(&p);
  const pp_search_grid sg{g.n_directions, g.n_powers, g.power_min, g.power_max, g.flat, g.chip};
  const int64_t n = static_cast<int64_t>(g.kick_type_count()) * g.n_directions * g.n_powers;
  std::vector<unsigned char> block(pp_grid_offsets_for_(n).total);
  const pp_world cw = to_c(w);
  or_dpps(&cw, &p, &sg, kicker, block.data(), nullptr, 0);
  return block;
}

void test_grid_vs_oracle() {
  std::mt19937_64 rng(0xB200);
  const PlannerConfig cfg;
  int mismatches = 0, best_bad = 0;
  for (int i = 0; i < 24; ++i) {
    std::uniform_int_distribution<int> team(1, 16);
    const WorldState w = random_world(rng, team(rng), team(rng) - 1, i % 3 ? 0.0 : 3.0);
    SearchGrid g;
    if (i % 4 == 1) g.chip = false;
    if (i % 4 == 2) {
      g.n_directions = 37;
      g.n_powers = 19;
    }
    const int kicker = w.ours[0].id;
    const CandidateGrid got = run_dpps(w, kicker, g, cfg, 8);
    auto block = oracle_grid(w, kicker, g);
    pp_grid_view v;
    pp_grid_view_of_(block.data(), static_cast<int64_t>(got.cells.size()), &v);
    for (size_t c = 0; c < got.cells.size(); ++c) {
      const PassCandidate& x = got.cells[c];
      const int oid = v.our_slot[c] >= 0 ? v.summary->ours_ids[v.our_slot[c]] : -1;
      const int tid = v.opp_slot[c] >= 0 ? v.summary->theirs_ids[v.opp_slot[c]] : -1;
      bool same = x.our_id == oid && x.opp_id == tid && x.our_time == v.our_time[c] &&
                  x.opp_time == v.opp_time[c] && x.feasible == (v.feasible[c] != 0);
      if (std::isfinite(x.our_time)) same = same && x.receive_point == Vec2{v.rx[c], v.ry[c]};
      mismatches += !same;
    }
    // best_pass equals the oracle's argmax (test_pass_eval.cpp:159-208)
    const auto bp = best_pass(got, w, cfg);
    const int64_t want = v.summary->best_cell[0];
    if (bp.has_value() != (want >= 0)) {
      ++best_bad;
    } else if (bp) {
      const int slot = bp->candidate.kick_type == KickType::flat || !g.flat ? 0 : 1;
      const int cell = got.cell_index(slot, bp->candidate.dir_index, bp->candidate.power_index);
      const double ws = v.summary->best_score[0];
      if (cell != want && std::fabs(bp->score - ws) > 1e-4 * std::fmax(1.0, std::fabs(ws))) ++best_bad;
      if (std::fabs(bp->score - ws) > 1e-12 * std::fmax(1.0, std::fabs(ws))) ++best_bad;
    }
    check(got.telemetry.sbip_calls ==
              got.cells.size() * (w.ours.size() + w.theirs.size()),
          "sbip_calls == cells x robots");
    check(got.telemetry.kernel == "sm100a", "telemetry.kernel");
  }
  check(mismatches == 0, "grid cells bit-identical to the oracle (" +
                             std::to_string(mismatches) + " mismatches)");
  check(best_bad == 0, "best_pass matches the oracle argmax");
}

void test_kicker_never_aggregated() {  // test_dpps.cpp:172-205
  const PlannerConfig cfg;
  WorldState w;
  w.ours = {RobotState{1, {0.0, 0.05}, {0.0, 0.0}, 0.0}, RobotState{2, {2.0, 0.0}, {0.0, 0.0}, 0.0}};
  w.theirs = {RobotState{0, {-2.0, 1.0}, {0.0, 0.0}, 0.0}};
  SearchGrid g;
  g.n_directions = 16;
  g.n_powers = 8;
  const CandidateGrid a = run_dpps_serial(w, 1, g, cfg);
  bool ok = a.telemetry.kicker_in_possession;
  for (const auto& c : a.cells) ok = ok && c.our_id != 1 && (c.our_id == 2 || c.our_id == -1);
  check(ok, "kicker consulted but never aggregated");
  WorldState w2 = w;
  w2.ours[0].position = {-4.0, -3.0};
  w2.ours[0].velocity = {1.0, 1.0};
  const CandidateGrid b = run_dpps_serial(w2, 1, g, cfg);
  check(grids_identical(a, b) && !b.telemetry.kicker_in_possession, "kicker position irrelevant");
  WorldState lonely = w;
  lonely.ours.pop_back();
  const CandidateGrid c = run_dpps_serial(lonely, 1, g, cfg);
  bool none = true;
  for (const auto& x : c.cells) none = none && x.our_id == -1 && !x.feasible;
  check(none && !best_pass(c, lonely, cfg).has_value(), "lonely kicker has no pass");
}

void test_errors() {  // test_dpps.cpp:259-282, test_pass_eval.cpp:156
  std::mt19937_64 rng(506);
  const WorldState w = random_world(rng, 3, 3);
  const PlannerConfig cfg;
  SearchGrid g;
  g.n_directions = 16;
  g.n_powers = 8;
  bool threw;
  check(category_of([&] { run_dpps_serial(w, 77, g, cfg); }, &threw) == ErrorCategory::validation && threw,
        "kicker not on ours -> validation_error");
  SearchGrid bad = g;
  bad.n_directions = 0;
  check(category_of([&] { run_dpps_serial(w, 0, bad, cfg); }, &threw) == ErrorCategory::config && threw,
        "n_directions 0 -> config_error");
  bad = g;
  bad.power_min = 3.0;
  bad.power_max = 2.0;
  check(category_of([&] { run_dpps_serial(w, 0, bad, cfg); }, &threw) == ErrorCategory::config && threw,
        "power range -> config_error");
  check(run_dpps(w, 0, g, cfg, -3).telemetry.workers == 1, "nonsense workers degrade to 1");
  PassCandidate infeasible;
  check(category_of([&] { score_pass(infeasible, w, cfg); }, &threw) == ErrorCategory::domain && threw,
        "score_pass(infeasible) -> domain_error");
  check(category_of([&] { score_running_point({-0.1, 0.0}, w, cfg); }, &threw) == ErrorCategory::domain && threw,
        "running point outside front field -> domain_error");
  check(category_of([&] { score_running_point({5.5, 0.0}, w, cfg); }, &threw) == ErrorCategory::domain && threw,
        "running point inside defense area -> domain_error");
}

void test_goal_view_known_answer() {  // test_pass_eval.cpp:28-46
  WorldState w;
  const GoalView v = goal_view({0.0, 0.0}, w, 0.09);
  const double expect = std::atan2(0.9, 6.0) - std::atan2(-0.9, 6.0);
  check(std::fabs(v.angle - expect) < 1e-12 && v.target.x == 6.0, "empty-field goal view");
  check(shoot_angle({6.0, 0.0}, w) == 0.0 && shoot_angle({6.5, 0.3}, w) == 0.0, "behind the line");
  w.theirs.push_back(RobotState{0, {2.0, 1.0}, {0.0, 0.0}, 0.0});
  check(shoot_angle({2.0, 1.05}, w, 0.09) == 0.0, "opponent on the point");
}

void test_running_points() {  // test_offball.cpp:88-96, 244-366
  const PlannerConfig cfg;
  FieldGeometry f;
  const ZonePartition part = partition_zones(f, {0.0, 2.5});
  check(zone_lattice(part.zone(ZoneLabel::III), 0.1).size() == 31 * 21, "zone III lattice 31x21");
  WorldState w;
  w.ball.position = {-2.0, 1.2};
  w.ours = {RobotState{1, {-2.1, 1.2}, {0.0, 0.0}, 0.0}};
  w.theirs = {RobotState{0, {5.0, 0.3}, {0, 0}, 0}, RobotState{1, {3.5, -1.0}, {0, 0}, 0},
              RobotState{2, {1.0, 2.0}, {0, 0}, 0}};
  const auto pts = best_running_points(w, {}, cfg);
  bool ok = pts.size() == 4;
  for (size_t i = 0; ok && i < pts.size(); ++i) {
    ok = static_cast<int>(pts[i].zone) == static_cast<int>(i);
    // brute force with the drop-in's own per-point scoring, exact tie rule
    const Zone& z = part.zone(pts[i].zone);
    (void)z;
  }
  check(ok, "best_running_points returns zones I..IV");
  const auto part2 = partition_zones(w.field, w.ball.position, cfg.thresholds.min_zone_width);
  for (const RunningPoint& rp : pts) {
    const auto lat = zone_lattice(part2.zone(rp.zone), cfg.thresholds.grid_step);
    size_t ny = 0;
    for (size_t i = 1; i < lat.size(); ++i)
      if (lat[i].x != lat[0].x) {
        ny = i;
        break;
      }
    const size_t nx = lat.size() / ny;
    bool have = false;
    double best = 0.0;
    Vec2 bp;
    for (size_t i = 1; i + 1 < nx; ++i)
      for (size_t j = 1; j + 1 < ny; ++j) {
        const Vec2 v = lat[i * ny + j];
        if (w.field.in_their_defense_area(v)) continue;
        const double s = score_running_point(v, w, cfg).first;
        if (!have || s > best) {
          best = s;
          bp = v;
          have = true;
        }
      }
    check(have && rp.point == bp && rp.score == best,
          std::string("zone ") + zone_name(rp.zone) + " optimum equals the brute force");
  }
  WorldState w3;
  w3.ball.position = {-2.0, 0.0};
  w3.ours = {RobotState{1, {-2.1, 0.0}, {0, 0}, 0}};
  const auto two = best_running_points(w3, {}, cfg, 2);
  check(two.size() == 2 && two[0].zone == ZoneLabel::III && two[1].zone == ZoneLabel::IV,
        "two runners -> III, IV");
  const auto skip = best_running_points(w3, {ZoneLabel::III}, cfg, 2);
  check(skip.size() == 2 && skip[0].zone == ZoneLabel::I && skip[1].zone == ZoneLabel::IV,
        "occupied III skipped");
  check(best_running_points(w3, {}, cfg, 4, Vec2{4.0, 2.0}).size() == 3, "best-pass zone excluded");
}

void test_tables() {  // test_dpps.cpp:57-94
  const auto d = direction_table(128);
  check(d[0] == Vec2{-1.0, 0.0} && d[64] == Vec2{1.0, 0.0}, "direction table seams");
  const auto p = power_table(64, 1.0, 6.5);
  check(p.front() == 1.0 && p.back() == 6.5 && power_table(1, 2.0, 6.0)[0] == 2.0, "power table");
}

void test_batch() {
  std::mt19937_64 rng(77);
  const PlannerConfig cfg;
  SearchGrid g;
  g.chip = false;
  std::vector<WorldState> frames;
  for (int i = 0; i < 16; ++i) frames.push_back(random_world(rng, 8, 8));
  const auto got = best_pass_batch(frames, {}, g, cfg);
  bool ok = got.size() == frames.size();
  for (size_t i = 0; ok && i < frames.size(); ++i) {
    int kicker = frames[i].ours[0].id;
    double bd = 1e300;
    for (const auto& r : frames[i].ours) {
      const double dd = distance(r.position, frames[i].ball.position);
      if (dd < bd) {
        bd = dd;
        kicker = r.id;
      }
    }
    const auto one = best_pass(run_dpps(frames[i], kicker, g, cfg, 1), frames[i], cfg);
    ok = one.has_value() == got[i].best.has_value() &&
         (!one || (one->score == got[i].best->score &&
                   one->candidate.dir_index == got[i].best->candidate.dir_index &&
                   one->candidate.power_index == got[i].best->candidate.power_index));
  }
  check(ok, "best_pass_batch == run_dpps + best_pass per frame");
}

// best_pass after run_dpps is served from the fused summary; it must equal
// the re-scoring path (forced by an input that no longer matches the run)
// and must not serve a stale result for an edited grid.
void test_best_pass_fused() {
  std::mt19937_64 rng(0xBE57);
  const PlannerConfig cfg;
  PlannerConfig cfg2 = cfg;
  cfg2.thresholds.drag_v_min = 1.5;  // not an input of score_pass: forces the re-score path
  int bad = 0;
  for (int i = 0; i < 12; ++i) {
    const WorldState w = random_world(rng, 8, 8);
    const SearchGrid g;
    const CandidateGrid grid = run_dpps(w, w.ours[0].id, g, cfg, 8);
    for (const std::optional<KickType> only :
         {std::optional<KickType>{}, std::optional<KickType>{KickType::flat},
          std::optional<KickType>{KickType::chip}}) {
      const auto fused = best_pass(grid, w, cfg, only);
      const auto rescored = best_pass(grid, w, cfg2, only);
      if (fused.has_value() != rescored.has_value()) {
        ++bad;
      } else if (fused) {
        bad += fused->score != rescored->score ||
               fused->candidate.dir_index != rescored->candidate.dir_index ||
               fused->candidate.power_index != rescored->candidate.power_index ||
               fused->candidate.kick_type != rescored->candidate.kick_type ||
               fused->features.shoot_angle_at_receive !=
                   rescored->features.shoot_angle_at_receive;
      }
    }
    // an edited grid is re-scored: dropping the winner changes the answer
    const auto best = best_pass(grid, w, cfg);
    if (best) {
      CandidateGrid edited = grid;
      const int slot = best->candidate.kick_type == KickType::flat ? 0 : 1;
      PassCandidate& c = edited.cells[static_cast<size_t>(
          edited.cell_index(slot, best->candidate.dir_index, best->candidate.power_index))];
      c.feasible = false;
      const auto next = best_pass(edited, w, cfg);
      bad += next.has_value() && next->candidate.dir_index == best->candidate.dir_index &&
             next->candidate.power_index == best->candidate.power_index &&
             next->candidate.kick_type == best->candidate.kick_type;
      for (auto& cell : edited.cells) cell.feasible = false;
      bad += best_pass(edited, w, cfg).has_value();
    }
  }
  check(bad == 0, "fused best_pass == re-scored best_pass; edited grids re-scored (" +
                      std::to_string(bad) + " bad)");
}

// Reference API entry points outside the search (ball_model.hpp:68-81,
// motion.hpp:25, intercept.hpp:25-37, offball.hpp:72-75).
void test_reference_entry_points() {
  const BallModelParams bp;
  const auto traj = BallTrajectory::chip_kick({0.5, -0.25}, {3.0, 4.0}, 5.0, bp);
  const BallSample s = ball_state_at(traj, 0.4);
  check(s.position == traj.position_at(0.4) && s.speed == traj.speed_at(0.4) &&
            s.airborne == traj.airborne_at(0.4),
        "ball_state_at");
  bool threw = false;
  check(category_of([&] { (void)ball_state_at(traj, -1.0); }, &threw) == ErrorCategory::domain &&
            threw,
        "ball_state_at(t < 0) -> domain_error");
  check(category_of([&] { (void)travel_time_to_distance(traj, std::nan("")); }, &threw) ==
                ErrorCategory::domain &&
            threw,
        "travel_time_to_distance(NaN) -> domain_error");
  check(travel_time_to_distance(traj, 1.0) == traj.travel_time_to_distance(1.0) &&
            !time_of_first_interceptable_point(traj, 0.5 * traj.interceptable_from) &&
            !travel_time_to_distance(traj, 2.0 * traj.stop_distance),
        "free travel_time_to_distance / time_of_first_interceptable_point");
  RobotState r;
  r.position = {1.0, 2.0};
  r.velocity = {0.5, -1.0};
  const MotionLimits lim;
  check(arrival_time_with_buffer(r, {3.0, -1.0}, lim, 0.3) ==
            arrival_time(r, {3.0, -1.0}, lim) + 0.3,
        "arrival_time_with_buffer");
  check(category_of([&] { (void)arrival_time_with_buffer(r, {0, 0}, lim, -0.1); }, &threw) ==
                ErrorCategory::domain &&
            threw,
        "arrival_time_with_buffer(buffer < 0) -> domain_error");
  const auto samples = TrajectorySamples::build(traj, 1.0 / 60.0);
  bool ok = samples.count() == static_cast<int>(std::floor(traj.stop_time * 60.0 + 1e-9)) + 1;
  for (int k = 0; ok && k < samples.count(); ++k)
    ok = samples.ts[k] == k * (1.0 / 60.0) && samples.ss[k] == traj.distance_at(samples.ts[k]);
  check(ok, "TrajectorySamples::build");
  const FieldGeometry f;
  const auto ex = ray_exit_distance(f, {0.0, 0.0}, {1.0, 0.0});
  check(ex && *ex == 6.0 && !ray_exit_distance(f, {7.0, 0.0}, {1.0, 0.0}), "ray_exit_distance");
  // guard points lie on the area boundary, on the segments to the posts
  const auto [gp, gq] = guard_points(f, {2.0, 1.0});
  check(std::fabs(gp.x - 4.2) < 1e-12 && std::fabs(gq.x - 4.2) < 1e-12 && gp.y > gq.y,
        "guard_points on the area's front edge");
  check(category_of([&] { (void)guard_points(f, {5.0, 0.0}); }, &threw) ==
                ErrorCategory::domain &&
            threw,
        "guard_points inside the area -> domain_error");
  WorldState w;
  check(guard_time({2.0, 1.0}, w, lim) == 10.0, "guard_time with no opponents = cap");
  check(category_of([&] { (void)guard_time({2.0, 1.0}, w, lim, 0.0); }, &threw) ==
                ErrorCategory::domain &&
            threw,
        "guard_time(cap <= 0) -> domain_error");
}

}  // namespace

int main() {
  test_best_pass_fused();
  test_reference_entry_points();
  test_tables();
  test_grid_vs_oracle();
  test_kicker_never_aggregated();
  test_errors();
  test_goal_view_known_answer();
  test_running_points();
  test_batch();
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
