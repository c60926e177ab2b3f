// passplan_cli.cpp -- `passplan_b200`, a drop-in for the reference CLI's
// planning commands (proj/tools/passplan_main.cpp:82-279) on the B200 path:
//
//   passplan_b200 plan       --snapshot S [--config C] [--kicker K] [--freekick] [--out F]
//   passplan_b200 heatmap    --snapshot S --mode pass|run [--zone I|II|III|IV|all]
//                            [--kicker K] [--out F]
//   passplan_b200 bench      --snapshot S [--workers-list 1 2 4 8] [--reps N] [--kicker K]
//   passplan_b200 possession --snapshot S [--config C]
//   passplan_b200 freekick   --snapshot S [--config C] [--kicker K]
//
// Same options, stdout lines and CSV files as the reference (CSV byte for
// byte; `kernel=` reports sm100a and `wall_ms` this GPU's time).  `--svg`
// and `drag-eval` are not part of the drop-in (no SVG renderer): --svg is
// rejected with a config error.  Errors print "error (<category>): ..." and
// exit with the reference's codes (exit_code_for).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "passplan/passplan.hpp"

using namespace passplan;

namespace {

struct Args {
  std::string cmd;
  std::string snapshot, config, out, svg, mode, zone;
  int kicker = -1, workers = 0, reps = 5;
  bool freekick = false;
  std::vector<int> workers_list;
};

[[noreturn]] void usage_error(const std::string& what) {
  std::fprintf(stderr, "%s\nRun with --help for more information.\n", what.c_str());
  std::exit(1);
}

int to_int(const std::string& opt, const std::string& v) {
  char* end = nullptr;
  const long x = std::strtol(v.c_str(), &end, 10);
  if (v.empty() || *end != '\0') usage_error(opt + ": Value " + v + " could not be converted");
  return static_cast<int>(x);
}

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 2) usage_error("A subcommand is required");
  a.cmd = argv[1];
  if (a.cmd == "--help" || a.cmd == "-h") {
    std::puts(
        "passplan_b200: deterministic pass/shoot planning for SSL-style robot soccer (B200)\n"
        "subcommands: plan, heatmap, bench, possession, freekick");
    std::exit(0);
  }
  const std::vector<std::string> known = {"plan", "heatmap", "bench", "possession", "freekick"};
  if (std::find(known.begin(), known.end(), a.cmd) == known.end())
    usage_error("The following argument was not expected: " + a.cmd);
  for (int i = 2; i < argc; ++i) {
    const std::string o = argv[i];
    auto value = [&]() -> std::string {
      if (i + 1 >= argc) usage_error(o + ": 1 required argument missing");
      return argv[++i];
    };
    if (o == "--snapshot") a.snapshot = value();
    else if (o == "--config") a.config = value();
    else if (o == "--out") a.out = value();
    else if (o == "--svg") a.svg = value();
    else if (o == "--workers") a.workers = to_int(o, value());
    else if (o == "--kicker" && a.cmd != "possession") a.kicker = to_int(o, value());
    else if (o == "--freekick" && a.cmd == "plan") a.freekick = true;
    else if (o == "--mode" && a.cmd == "heatmap") a.mode = value();
    else if (o == "--zone" && a.cmd == "heatmap") a.zone = value();
    else if (o == "--reps" && a.cmd == "bench") a.reps = to_int(o, value());
    else if (o == "--workers-list" && a.cmd == "bench") {
      while (i + 1 < argc && argv[i + 1][0] != '-') a.workers_list.push_back(to_int(o, argv[++i]));
    } else {
      usage_error("The following argument was not expected: " + o);
    }
  }
  if (a.snapshot.empty()) usage_error("--snapshot is required");
  if (a.cmd == "heatmap" && a.mode.empty()) usage_error("--mode is required");
  return a;
}

PlannerConfig config_of(const Args& a) {
  if (a.config.empty()) {
    PlannerConfig c;
    c.validate();
    return c;
  }
  return PlannerConfig::load(a.config);
}

int workers_of(const Args& a) {
  if (a.workers > 0) return a.workers;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}

// The teammate nearest the ball (first on ties) when --kicker is omitted.
int nearest_kicker(const WorldState& w) {
  if (w.ours.empty()) throw validation_error("snapshot has no robots on team ours");
  const RobotState* best = &w.ours.front();
  for (const RobotState& r : w.ours)
    if (distance(r.position, w.ball.position) < distance(best->position, w.ball.position))
      best = &r;
  return best->id;
}

const char* kick_name(KickType k) { return k == KickType::flat ? "flat" : "chip"; }

void print_pass(const char* tag, const ScoredPass& s) {
  const PassCandidate& c = s.candidate;
  char opp[64] = "never";
  if (!std::isinf(c.opp_time)) std::snprintf(opp, sizeof(opp), "#%d@%.3fs", c.opp_id, c.opp_time);
  std::printf("%s: %s dir=%d power=%d receive=(%.3f, %.3f) our=#%d@%.3fs opp=%s score=%.6f\n",
              tag, kick_name(c.kick_type), c.dir_index, c.power_index, c.receive_point.x,
              c.receive_point.y, c.our_id, c.our_time, opp, s.score);
}

void print_freekick(const FreeKickPlan& fk) {
  std::printf("freekick: t_ball=%.4f t_robot=%.4f order=%s delay=%.4f\n", fk.t_ball, fk.t_robot,
              fk.order == KickOrder::kick_first ? "kick_first" : "robot_first", fk.kick_delay);
}

void no_svg(const Args& a) {
  if (!a.svg.empty())
    throw config_error("--svg: the B200 drop-in has no SVG renderer (use the reference's)");
}

int cmd_plan(const Args& a) {
  no_svg(a);
  const WorldState world = load_world_snapshot(a.snapshot);
  const PlannerConfig cfg = config_of(a);
  const int kicker = a.kicker >= 0 ? a.kicker : nearest_kicker(world);
  const CandidateGrid grid = run_dpps(world, kicker, cfg.grid, cfg, workers_of(a));
  std::printf("kernel=%s workers=%d sbip_calls=%llu wall_ms=%.3f\n", grid.telemetry.kernel.c_str(),
              grid.telemetry.workers, static_cast<unsigned long long>(grid.telemetry.sbip_calls),
              grid.telemetry.wall_ms);
  if (!grid.telemetry.kicker_in_possession)
    std::printf("warning: kicker %d is not in possession of the ball\n", kicker);
  size_t n_flat = 0, n_chip = 0;
  for (const PassCandidate& c : grid.cells)
    if (c.feasible) ++(c.kick_type == KickType::flat ? n_flat : n_chip);
  std::printf("feasible: flat=%zu chip=%zu\n", n_flat, n_chip);
  const std::optional<ScoredPass> best = best_pass(grid, world, cfg);
  if (best) {
    print_pass("best_pass", *best);
  } else {
    std::printf("NO_FEASIBLE_PASS\n");
  }
  const RobotState* shooter = world.find(Team::ours, kicker);
  if (!shooter) throw validation_error("kicker id not on team ours");
  const ShotDecision shot = decide_shot(*shooter, world, cfg);
  const char* why = shot.reason == ShotReason::clear             ? "clear"
                    : shot.reason == ShotReason::angle_too_small ? "angle_too_small"
                                                                 : "interceptable";
  std::printf("shot: %s angle=%.4f target=(%.3f, %.3f) reason=%s\n", shot.shoot ? "shoot" : "hold",
              shot.shot_angle, shot.shot_target.x, shot.shot_target.y, why);
  const std::optional<Vec2> bp =
      best ? std::optional<Vec2>(best->candidate.receive_point) : std::nullopt;
  for (const RunningPoint& rp : best_running_points(world, {}, cfg, 4, bp))
    std::printf("run zone %s: (%.3f, %.3f) score=%.6f guard=%.3fs\n", zone_name(rp.zone),
                rp.point.x, rp.point.y, rp.score, rp.features.guard_time);
  if (a.freekick && best) print_freekick(plan_free_kick(world, kicker, best->candidate, cfg));
  if (!a.out.empty()) write_text_file(a.out, grid_to_csv(grid));
  return 0;
}

void emit(const Args& a, const std::string& csv) {
  if (!a.out.empty()) {
    write_text_file(a.out, csv);
  } else {
    std::fputs(csv.c_str(), stdout);
  }
}

int cmd_heatmap(const Args& a) {
  no_svg(a);
  const WorldState world = load_world_snapshot(a.snapshot);
  const PlannerConfig cfg = config_of(a);
  if (a.mode == "pass") {
    const int kicker = a.kicker >= 0 ? a.kicker : nearest_kicker(world);
    const CandidateGrid grid = run_dpps(world, kicker, cfg.grid, cfg, workers_of(a));
    std::vector<HeatPoint> pts;
    for (const PassCandidate& c : grid.cells)
      if (c.feasible) pts.push_back({c.receive_point, score_pass(c, world, cfg).first});
    emit(a, heatmap_to_csv(pts));
    return 0;
  }
  if (a.mode != "run") throw config_error("heatmap mode must be 'pass' or 'run'");
  std::vector<ZoneLabel> zones;
  if (a.zone.empty() || a.zone == "all") zones = {ZoneLabel::I, ZoneLabel::II, ZoneLabel::III, ZoneLabel::IV};
  else if (a.zone == "I") zones = {ZoneLabel::I};
  else if (a.zone == "II") zones = {ZoneLabel::II};
  else if (a.zone == "III") zones = {ZoneLabel::III};
  else if (a.zone == "IV") zones = {ZoneLabel::IV};
  else throw config_error("zone must be one of I, II, III, IV, all");
  const ZonePartition part =
      partition_zones(world.field, world.ball.position, cfg.thresholds.min_zone_width);
  std::vector<RunHeatRow> rows;
  for (ZoneLabel z : zones) {
    for (Vec2 v : zone_lattice(part.zone(z), cfg.thresholds.grid_step)) {
      try {
        const auto [score, ft] = score_running_point(v, world, cfg);
        rows.push_back({v, ft, score});
      } catch (const Error&) {
        // not scorable (in the defense area): skipped, as the reference does
      }
    }
  }
  emit(a, run_heatmap_to_csv(rows));
  return 0;
}

int cmd_bench(const Args& a) {
  const WorldState world = load_world_snapshot(a.snapshot);
  const PlannerConfig cfg = config_of(a);
  const int kicker = a.kicker >= 0 ? a.kicker : nearest_kicker(world);
  if (a.reps < 1) throw config_error("--reps must be at least 1");
  std::vector<int> counts = a.workers_list.empty() ? std::vector<int>{1, 2, 4, 8} : a.workers_list;
  auto med_min = [](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return std::pair<double, double>{v[v.size() / 2], v.front()};
  };
  const CandidateGrid first = run_dpps_serial(world, kicker, cfg.grid, cfg);
  std::vector<double> ms;
  for (int r = 0; r < a.reps; ++r) {
    const CandidateGrid g = run_dpps_serial(world, kicker, cfg.grid, cfg);
    if (!grids_identical(first, g)) throw internal_error("bench: serial run not reproducible");
    ms.push_back(g.telemetry.wall_ms);
  }
  const auto [s_med, s_min] = med_min(ms);
  std::printf("kernel=%s cells=%zu sbip_calls=%llu\n", first.telemetry.kernel.c_str(),
              first.cells.size(), static_cast<unsigned long long>(first.telemetry.sbip_calls));
  std::printf("serial: median=%.3fms min=%.3fms\n", s_med, s_min);
  for (int w : counts) {
    if (w < 1) throw config_error("worker counts must be positive");
    std::vector<double> t;
    for (int r = 0; r < a.reps; ++r) {
      const CandidateGrid g = run_dpps(world, kicker, cfg.grid, cfg, w);
      if (!grids_identical(first, g))
        throw internal_error("bench: grid mismatch against serial oracle at workers=" +
                             std::to_string(w));
      t.push_back(g.telemetry.wall_ms);
    }
    const auto [med, mn] = med_min(t);
    std::printf("workers=%d: median=%.3fms min=%.3fms speedup=%.2fx\n", w, med, mn,
                med > 0.0 ? s_med / med : 0.0);
  }
  return 0;
}

int cmd_possession(const Args& a) {
  const WorldState world = load_world_snapshot(a.snapshot);
  const PossessionReport r = possession(world, config_of(a));
  const char* side = r.side == PossessionSide::ours     ? "ours"
                     : r.side == PossessionSide::theirs ? "theirs"
                                                        : "contested";
  auto fmt = [](const std::optional<double>& t) {
    return t ? std::to_string(*t) + "s" : std::string("never");
  };
  std::printf("possession: %s our_time=%s their_time=%s\n", side, fmt(r.our_time).c_str(),
              fmt(r.their_time).c_str());
  return 0;
}

int cmd_freekick(const Args& a) {
  const WorldState world = load_world_snapshot(a.snapshot);
  const PlannerConfig cfg = config_of(a);
  const int kicker = a.kicker >= 0 ? a.kicker : nearest_kicker(world);
  const CandidateGrid grid = run_dpps(world, kicker, cfg.grid, cfg, workers_of(a));
  const std::optional<ScoredPass> best = best_pass(grid, world, cfg);
  if (!best) {
    std::printf("NO_FEASIBLE_PASS\n");
    return 0;
  }
  print_pass("best_pass", *best);
  print_freekick(plan_free_kick(world, kicker, best->candidate, cfg));
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const Args a = parse(argc, argv);
  try {
    if (a.cmd == "plan") return cmd_plan(a);
    if (a.cmd == "heatmap") return cmd_heatmap(a);
    if (a.cmd == "bench") return cmd_bench(a);
    if (a.cmd == "possession") return cmd_possession(a);
    return cmd_freekick(a);
  } catch (const Error& e) {
    std::fprintf(stderr, "error (%s): %s\n", category_name(e.category()), e.what());
    return exit_code_for(e.category());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error (internal): %s\n", e.what());
    return exit_code_for(ErrorCategory::internal);
  }
}
