// plan_sequence.cpp -- times the reference's own plan sequence through the
// C++ drop-in (lib/libpassplan.so): run_dpps then best_pass for all / flat /
// chip (proj/tools/passplan_main.cpp:87,102-104), on frame F8 (bench_16v16
// truncated to the first 8 robots per team: 128 x 64, flat +
// chip).  Host timing around the whole sequence: the world conversion, the
// GPU search + value function + argmax, and the 16,384-cell CandidateGrid the
// API returns.  Prints one JSON line.  usage: plan_sequence SNAPSHOT [REPS]
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "passplan/passplan.hpp"

using namespace passplan;
using Clock = std::chrono::steady_clock;

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: plan_sequence SNAPSHOT [REPS]\n");
    return 2;
  }
  const int reps = argc > 2 ? std::atoi(argv[2]) : 200;
  WorldState w = load_world_snapshot(argv[1]);
  if (w.ours.size() > 8) w.ours.resize(8);
  if (w.theirs.size() > 8) w.theirs.resize(8);
  int kicker = w.ours.front().id;
  double best_d = 1e300;
  for (const RobotState& r : w.ours) {
    const double d = distance(r.position, w.ball.position);
    if (d < best_d) {
      best_d = d;
      kicker = r.id;
    }
  }
  const PlannerConfig cfg;
  const SearchGrid grid;  // 128 x 64, flat + chip
  std::vector<double> seq, search, value;
  double score = 0.0;
  for (int r = 0; r < reps + 5; ++r) {
    const auto t0 = Clock::now();
    const CandidateGrid g = run_dpps(w, kicker, grid, cfg, 16);
    const auto t1 = Clock::now();
    const auto all = best_pass(g, w, cfg);
    const auto flat = best_pass(g, w, cfg, KickType::flat);
    const auto chip = best_pass(g, w, cfg, KickType::chip);
    const auto t2 = Clock::now();
    if (!all || !flat || !chip) {
      std::fprintf(stderr, "no feasible pass\n");
      return 1;
    }
    score = all->score;
    if (r < 5) continue;  // warm-up
    search.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
    value.push_back(std::chrono::duration<double, std::milli>(t2 - t1).count());
    seq.push_back(std::chrono::duration<double, std::milli>(t2 - t0).count());
  }
  auto p50 = [](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  std::printf(
      "{\"sequence_p50_ms\": %.4f, \"run_dpps_p50_ms\": %.4f, \"best_pass_x3_p50_ms\": %.4f, "
      "\"reps\": %d, \"best_score\": %.9f, \"path\": \"C++ drop-in: run_dpps(F8, 128x64 "
      "flat+chip) + best_pass all/flat/chip (passplan_main.cpp:87,102-104)\"}\n",
      p50(seq), p50(search), p50(value), reps, score);
  return 0;
}
