// passplan/passplan.hpp -- C++ drop-in for the reference's hot-path API.
//
// Source-compatible with the declarations a caller of the reference uses on
// this path (reference headers proj/include/passplan/{vec2,world,errors,
// weights,ball_model,motion,dpps,pass_eval,offball,intercept,config,csv,
// snapshot}.hpp and detail/arrival_math.hpp): same namespace, type and field
// names, defaults, signatures and error categories.  The per-header names
// (passplan/dpps.hpp, ...) are provided as one-line forwarders to this file;
// detail/arrival_math.hpp forwards to the shared restatement pp_math.hpp.
// Every computation on the hot path runs on the GPU through the C-ABI of
// passplan_b200.h; the small host-side helpers here (geometry, tables,
// lattices, validation, the closed-form ball model) are the same closed forms.
//
// The per-pair plug-in point kernels::KernelBackend (passplan/kernels/
// kernel.hpp) has one backend, "sm100a", whose scan_first runs on the GPU;
// run_dpps does not call through it (one call is a single (trajectory,
// robot) pair) but reports its name in telemetry.kernel.
//
// Not provided (outside the accelerated path, SURVEY.md 2 out of scope): the
// SVG renderer (svg.hpp, SvgStyle), drag_decision / DragDecision, the JSON
// serialisation of PlannerConfig (to_json_text) and the reference's CPU scan
// backends (scalar_kernel / avx2_kernel).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numbers>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "passplan/kernels/kernel.hpp"

namespace passplan {

// ---- geometry (vec2.hpp) ---------------------------------------------------
struct Vec2 {
  double x = 0.0;
  double y = 0.0;
  constexpr Vec2() = default;
  constexpr Vec2(double x_, double y_) : x(x_), y(y_) {}
  constexpr Vec2 operator+(Vec2 o) const { return {x + o.x, y + o.y}; }
  constexpr Vec2 operator-(Vec2 o) const { return {x - o.x, y - o.y}; }
  constexpr Vec2 operator*(double s) const { return {x * s, y * s}; }
  constexpr Vec2 operator-() const { return {-x, -y}; }
  constexpr bool operator==(const Vec2&) const = default;
  constexpr double dot(Vec2 o) const { return x * o.x + y * o.y; }
  constexpr double cross(Vec2 o) const { return x * o.y - y * o.x; }
  double norm() const { return std::sqrt(x * x + y * y); }
  constexpr double norm2() const { return x * x + y * y; }
  Vec2 normalized() const {
    const double n = norm();
    return n == 0.0 ? *this : Vec2{x / n, y / n};
  }
  constexpr Vec2 perp_left() const { return {-y, x}; }
  constexpr Vec2 perp_right() const { return {y, -x}; }
  double angle() const { return std::atan2(y, x); }
};
inline constexpr Vec2 operator*(double s, Vec2 v) { return {s * v.x, s * v.y}; }
inline double distance(Vec2 a, Vec2 b) { return (a - b).norm(); }
double segment_distance(Vec2 p, Vec2 a, Vec2 b);

// ---- errors (errors.hpp) ---------------------------------------------------
enum class ErrorCategory { schema, validation, config, domain, internal };

class Error : public std::runtime_error {
 public:
  Error(ErrorCategory category, const std::string& message)
      : std::runtime_error(message), category_(category) {}
  ErrorCategory category() const { return category_; }

 private:
  ErrorCategory category_;
};

inline Error schema_error(const std::string& m) { return Error(ErrorCategory::schema, m); }
inline Error validation_error(const std::string& m) { return Error(ErrorCategory::validation, m); }
inline Error config_error(const std::string& m) { return Error(ErrorCategory::config, m); }
inline Error domain_error(const std::string& m) { return Error(ErrorCategory::domain, m); }
inline Error internal_error(const std::string& m) { return Error(ErrorCategory::internal, m); }
const char* category_name(ErrorCategory c);
int exit_code_for(ErrorCategory c);

// ---- world (world.hpp) -----------------------------------------------------
struct FieldGeometry {
  double length = 12.0;
  double width = 9.0;
  double goal_width = 1.8;
  double defense_depth = 1.8;
  double defense_width = 3.6;

  bool contains(Vec2 p) const {
    return p.x >= -0.5 * length && p.x <= 0.5 * length && p.y >= -0.5 * width &&
           p.y <= 0.5 * width;
  }
  Vec2 their_goal_center() const { return {0.5 * length, 0.0}; }
  Vec2 our_goal_center() const { return {-0.5 * length, 0.0}; }
  Vec2 their_left_post() const { return {0.5 * length, 0.5 * goal_width}; }
  Vec2 their_right_post() const { return {0.5 * length, -0.5 * goal_width}; }
  bool in_their_defense_area(Vec2 p) const {
    return p.x >= 0.5 * length - defense_depth && p.x <= 0.5 * length &&
           p.y >= -0.5 * defense_width && p.y <= 0.5 * defense_width;
  }
  bool strictly_in_their_defense_area(Vec2 p) const {
    return p.x > 0.5 * length - defense_depth && p.x < 0.5 * length &&
           p.y > -0.5 * defense_width && p.y < 0.5 * defense_width;
  }
  void validate() const;
};

struct RobotState {
  int id = 0;
  Vec2 position;
  Vec2 velocity;
  double theta = 0.0;
};

struct BallState {
  Vec2 position;
  Vec2 velocity;
};

enum class Team { ours, theirs };

struct WorldState {
  FieldGeometry field;
  BallState ball;
  std::vector<RobotState> ours;
  std::vector<RobotState> theirs;
  const std::vector<RobotState>& team(Team t) const { return t == Team::ours ? ours : theirs; }
  const RobotState* find(Team t, int id) const;
  void validate() const;
};

WorldState mirror_world(const WorldState& w);

// ---- parameters (weights.hpp, ball_model.hpp, motion.hpp, config.hpp) -------
struct PassWeights {
  double teammate_time = 1.0;
  double shoot_angle = 2.0;
  double dist_goal = 1.0;
  double refraction = 0.5;
  double margin = 1.0;
};

struct RunWeights {
  double dist_goal = 1.0;
  double dist_ball = 0.3;
  double angle = 1.0;
  double guard_time = 0.3;
  double exposure = 0.5;
};

struct NormBounds {
  double length_upper = 0.0;
  double angle_upper = std::numbers::pi;
};

struct AngleBand {
  double full_lo = 0.0;
  double peak_lo = 15.0 * std::numbers::pi / 180.0;
  double peak_hi = 45.0 * std::numbers::pi / 180.0;
  double full_hi = 90.0 * std::numbers::pi / 180.0;
};

struct WeightConfig {
  PassWeights pass;
  RunWeights run;
  NormBounds norm;
};

struct BallModelParams {
  double slide_decel = 3.4;
  double roll_decel = 0.5;
  double transition_ratio = 5.0 / 7.0;
  double power_min = 1.0;
  double power_max = 6.5;
  double chip_flight_fraction = 0.5;
  void validate() const;
};

enum class KickType { flat, chip };

struct MotionLimits {
  double max_speed = 3.25;
  double max_accel = 3.0;
  double max_decel = 3.0;
  void validate() const;
};

struct SearchGrid {
  int n_directions = 128;
  int n_powers = 64;
  double power_min = 1.0;
  double power_max = 6.5;
  bool flat = true;
  bool chip = true;
  int kick_type_count() const { return (flat ? 1 : 0) + (chip ? 1 : 0); }
  std::vector<KickType> kick_types() const;
  void validate() const;
};

struct PlannerThresholds {
  double sbip_dt = 1.0 / 60.0;
  double robot_radius = 0.09;
  double safety_margin = 0.3;
  double buffer_time = 0.3;
  double possession_radius = 0.15;
  double angle_threshold = 0.1;
  double shot_power = 0.0;
  double margin_cap = 10.0;
  double possession_dt = 1e-3;
  double contest_epsilon = 1e-3;
  double grid_step = 0.1;
  double min_zone_width = 1.0;
  double guard_time_cap = 10.0;
  double drag_v_min = 1.0;
  double marking_radius = 0.6;
};

struct PlannerConfig {
  BallModelParams ball;
  MotionLimits motion_ours;
  MotionLimits motion_theirs;
  SearchGrid grid;
  WeightConfig weights;
  AngleBand angle_band;
  PlannerThresholds thresholds;

  double shot_power() const {
    return thresholds.shot_power > 0.0 ? thresholds.shot_power : ball.power_max;
  }
  double length_upper(const FieldGeometry& f) const {
    return weights.norm.length_upper > 0.0 ? weights.norm.length_upper : f.length;
  }
  void validate() const;  // config_error on the first bad value (SvgStyle excluded)
  // JSON config (config.cpp:203-241): unknown keys and wrong types are
  // config_error; an "svg" section is accepted (pixels_per_meter > 0
  // checked) but not stored -- the SVG renderer is not part of the drop-in.
  static PlannerConfig from_json_text(const std::string& text);
  static PlannerConfig load(const std::string& path);
};

// ---- search (dpps.hpp) -------------------------------------------------------
inline double direction_angle(int k, int n_directions) {
  return -std::numbers::pi + k * (2.0 * std::numbers::pi / n_directions);
}
std::vector<Vec2> direction_table(int n_directions);
std::vector<double> power_table(int n_powers, double power_min, double power_max);

constexpr double kNever = std::numeric_limits<double>::infinity();

struct PassCandidate {
  KickType kick_type = KickType::flat;
  int dir_index = 0;
  int power_index = 0;
  int our_id = -1;
  double our_time = kNever;
  int opp_id = -1;
  double opp_time = kNever;
  Vec2 receive_point;
  bool feasible = false;
};

struct DppsTelemetry {
  std::uint64_t sbip_calls = 0;
  double wall_ms = 0.0;
  int workers = 1;
  std::string kernel;
  bool kicker_in_possession = true;
};

struct CandidateGrid {
  SearchGrid grid;
  int kicker_id = -1;
  Vec2 ball_origin;
  std::vector<KickType> kick_types;
  std::vector<Vec2> directions;
  std::vector<double> powers;
  std::vector<PassCandidate> cells;
  DppsTelemetry telemetry;
  int cell_index(int kick_type_slot, int dir, int power) const {
    return (kick_type_slot * grid.n_directions + dir) * grid.n_powers + power;
  }
  const PassCandidate& at(int kick_type_slot, int dir, int power) const {
    return cells[cell_index(kick_type_slot, dir, power)];
  }
};

// `workers` is accepted for source compatibility; the search always runs on
// the GPU (telemetry.kernel == "sm100a").
CandidateGrid run_dpps(const WorldState& world, int kicker_id, const SearchGrid& grid,
                       const PlannerConfig& cfg, int workers);
CandidateGrid run_dpps_serial(const WorldState& world, int kicker_id, const SearchGrid& grid,
                              const PlannerConfig& cfg);
std::vector<PassCandidate> feasible_candidates(const CandidateGrid& g);
bool grids_identical(const CandidateGrid& a, const CandidateGrid& b);

// ---- value function (pass_eval.hpp) ----------------------------------------
struct PassFeatures {
  double teammate_intercept_time = 0.0;
  double shoot_angle_at_receive = 0.0;
  double dist_receive_to_goal = 0.0;
  double refraction_angle = 0.0;
  double intercept_margin = 0.0;
};

struct GoalView {
  double angle = 0.0;
  double window_lo = 0.0;
  double window_hi = 0.0;
  Vec2 target;
};

GoalView goal_view(Vec2 point, const WorldState& world, double robot_radius);
double shoot_angle(Vec2 point, const WorldState& world, double robot_radius = 0.09);
std::pair<double, PassFeatures> score_pass(const PassCandidate& candidate, const WorldState& world,
                                           const PlannerConfig& cfg);

struct ScoredPass {
  PassCandidate candidate;
  double score = 0.0;
  PassFeatures features;
};

std::optional<ScoredPass> best_pass(const CandidateGrid& g, const WorldState& world,
                                    const PlannerConfig& cfg);
std::optional<ScoredPass> best_pass(const CandidateGrid& g, const WorldState& world,
                                    const PlannerConfig& cfg, std::optional<KickType> only);

// ---- off-the-ball running points (offball.hpp) -------------------------------
enum class ZoneLabel { I, II, III, IV };
const char* zone_name(ZoneLabel z);

struct Zone {
  ZoneLabel label = ZoneLabel::I;
  double x0 = 0.0, x1 = 0.0;
  double y0 = 0.0, y1 = 0.0;
  bool contains(Vec2 p) const { return p.x >= x0 && p.x <= x1 && p.y >= y0 && p.y <= y1; }
};

struct ZonePartition {
  std::array<Zone, 4> zones;
  double cut_x = 0.0;
  double cut_y = 0.0;
  const Zone& zone(ZoneLabel z) const { return zones[static_cast<int>(z)]; }
  std::optional<ZoneLabel> label_at(Vec2 p) const;
};

ZonePartition partition_zones(const FieldGeometry& field, Vec2 ball, double min_zone_width = 1.0);

struct RunningPointFeatures {
  double dist_to_goal = 0.0;
  double dist_to_ball = 0.0;
  double angle_to_goal = 0.0;
  double guard_time = 0.0;
  double defense_exposure = 0.0;
};

std::pair<double, RunningPointFeatures> score_running_point(Vec2 p, const WorldState& world,
                                                            const PlannerConfig& cfg);

struct RunningPoint {
  ZoneLabel zone = ZoneLabel::I;
  Vec2 point;
  double score = 0.0;
  RunningPointFeatures features;
};

// guard_time (offball.hpp:72): the two opponents nearest their defense area
// race to the guard points; capped at `cap`.  guard_points (offball.hpp:75):
// where the segments from p to the two posts enter the defense area.  Both
// throw domain_error for p strictly inside the area (and guard_time for a
// cap that is not positive and finite).  Computed on the GPU.
double guard_time(Vec2 p, const WorldState& world, const MotionLimits& limits, double cap = 10.0);
std::pair<Vec2, Vec2> guard_points(const FieldGeometry& field, Vec2 p);

std::vector<Vec2> zone_lattice(const Zone& zone, double step);
std::vector<RunningPoint> best_running_points(const WorldState& world,
                                              const std::set<ZoneLabel>& occupied,
                                              const PlannerConfig& cfg, int n_runners = 4,
                                              std::optional<Vec2> best_pass_point = std::nullopt);

// ---- ball trajectory (ball_model.hpp) ------------------------------------------
struct BallTrajectory {
  Vec2 origin;
  Vec2 direction;  // unit; arbitrary when kick_speed == 0
  double kick_speed = 0.0;
  KickType kick_type = KickType::flat;
  double v1 = 0.0;  // speed at the slide-to-roll transition
  double slide_decel = 0.0;
  double roll_decel = 0.0;
  double slide_end_time = 0.0;
  double slide_end_distance = 0.0;
  double stop_time = 0.0;
  double stop_distance = 0.0;
  double interceptable_from = 0.0;  // chip: airborne until this distance

  static BallTrajectory flat_kick(Vec2 origin, Vec2 dir, double speed,
                                  const BallModelParams& params);
  static BallTrajectory chip_kick(Vec2 origin, Vec2 dir, double speed,
                                  const BallModelParams& params);
  static BallTrajectory free_roll(Vec2 origin, Vec2 velocity, const BallModelParams& params);
  double speed_at(double t) const;
  double distance_at(double t) const;
  Vec2 position_at(double t) const { return origin + direction * distance_at(t); }
  bool airborne_at(double t) const;
  std::optional<double> travel_time_to_distance(double d) const;
  std::optional<double> time_of_first_interceptable_point(double d) const;
};

struct BallSample {
  Vec2 position;
  double speed = 0.0;
  bool airborne = false;
};

// Checked free forms (ball_model.hpp:68-81): domain_error on t < 0 / d < 0 / NaN.
BallSample ball_state_at(const BallTrajectory& traj, double t);
std::optional<double> travel_time_to_distance(const BallTrajectory& traj, double d);
std::optional<double> time_of_first_interceptable_point(const BallTrajectory& traj, double d);

struct PassPower {
  double kick_speed = 0.0;
  double v1 = 0.0;
  bool clamped = false;
};
PassPower pass_power_for(double d, double t, const BallModelParams& params);

// ---- interception (intercept.hpp) ----------------------------------------------
struct InterceptResult {
  Team team = Team::ours;
  int robot_id = -1;
  std::optional<double> intercept_time;  // nullopt = Never
  Vec2 intercept_point;
  bool finite() const { return intercept_time.has_value(); }
};
InterceptResult intercept_time(const RobotState& robot, const BallTrajectory& traj,
                               const MotionLimits& limits, const FieldGeometry& field, double dt,
                               double robot_radius = 0.09);
std::vector<InterceptResult> intercept_all(const WorldState& world, const BallTrajectory& traj,
                                           const MotionLimits& ours_limits,
                                           const MotionLimits& theirs_limits, double dt,
                                           double robot_radius = 0.09);
double arrival_time(const RobotState& robot, Vec2 target, const MotionLimits& limits);
// arrival_time + buffer (motion.hpp:25); domain_error on a negative or NaN buffer.
double arrival_time_with_buffer(const RobotState& robot, Vec2 target, const MotionLimits& limits,
                                double buffer);

// Sampled trajectory (intercept.hpp:25-33): ts[k] = k*dt, ss[k] = distance_at(ts[k]),
// k = 0 .. floor(stop_time/dt + 1e-9).  domain_error unless dt > 0.
struct TrajectorySamples {
  std::vector<double> ts;
  std::vector<double> ss;
  double dt = 0.0;
  int count() const { return static_cast<int>(ts.size()); }
  static TrajectorySamples build(const BallTrajectory& traj, double dt);
};

// Distance along unit u from origin to the field boundary (intercept.hpp:35-37);
// nullopt when the origin is outside the field.
std::optional<double> ray_exit_distance(const FieldGeometry& field, Vec2 origin, Vec2 u);

// The scan's internals (intercept.hpp:52-72), for callers of the plug-in point.
namespace detail_intercept {
struct ScanWindow {
  int k_begin = 0;  // first sample past a chip's airborne prefix
  int k_end = 0;    // one past the last in-field sample
  bool rest_in_field = false;
};
ScanWindow scan_window(const BallTrajectory& traj, const TrajectorySamples& samples,
                       std::optional<double> d_exit);
kernels::RobotKin make_kin(const RobotState& robot, const MotionLimits& limits,
                           double robot_radius);
// scan_robot's window prune and start skip, then backend.scan_first.
int scan_robot(const kernels::ScanBatch& batch, const kernels::RobotKin& kin,
               const kernels::KernelBackend& backend);
}  // namespace detail_intercept

// ---- shot, free kick, possession (pass_eval.hpp) --------------------------------
enum class ShotReason { angle_too_small, interceptable, clear };
struct ShotDecision {
  bool shoot = false;
  double shot_angle = 0.0;
  Vec2 shot_target;
  bool blocked = false;
  ShotReason reason = ShotReason::clear;
};
ShotDecision decide_shot(const RobotState& shooter, const WorldState& world,
                         const PlannerConfig& cfg);

enum class KickOrder { robot_first, kick_first };
struct FreeKickPlan {
  double t_ball = 0.0;
  double t_robot = 0.0;
  KickOrder order = KickOrder::kick_first;
  double kick_delay = 0.0;
};
FreeKickPlan plan_free_kick(const WorldState& world, int kicker_id, const PassCandidate& target,
                            const PlannerConfig& cfg);

enum class PossessionSide { ours, theirs, contested };
struct PossessionReport {
  PossessionSide side = PossessionSide::contested;
  std::optional<double> our_time;
  std::optional<double> their_time;
};
PossessionReport possession(const WorldState& world, const PlannerConfig& cfg);

// ---- CSV (csv.hpp) and JSON snapshot / config I/O (snapshot.hpp, config.hpp) ------
std::string format_double(double v);  // %.17g, +inf -> "never"
double parse_double_field(const std::string& field);
std::string grid_to_csv(const CandidateGrid& g);
CandidateGrid grid_from_csv(const std::string& text);
struct HeatPoint {
  Vec2 point;
  double value = 0.0;
};
std::string heatmap_to_csv(const std::vector<HeatPoint>& points);
std::vector<HeatPoint> heatmap_from_csv(const std::string& text);
struct RunHeatRow {
  Vec2 point;
  RunningPointFeatures features;
  double score = 0.0;
};
std::string run_heatmap_to_csv(const std::vector<RunHeatRow>& rows);
std::vector<RunHeatRow> run_heatmap_from_csv(const std::string& text);
std::string read_text_file(const std::string& path);
void write_text_file(const std::string& path, const std::string& text);  // atomic (tmp+rename)

WorldState parse_world_snapshot(const std::string& bytes);
WorldState load_world_snapshot(const std::string& path);
std::string serialize_world_snapshot(const WorldState& w);

// ---- batched frames (GPU extension, no reference counterpart) ---------------
struct FrameBest {
  std::optional<ScoredPass> best;  // best_pass over all kick types
  std::int64_t n_feasible = 0;
};
// run_dpps + best_pass for many independent frames (one GPU).  kicker_ids may
// be empty: then the teammate nearest the ball kicks.
std::vector<FrameBest> best_pass_batch(const std::vector<WorldState>& frames,
                                       const std::vector<int>& kicker_ids, const SearchGrid& grid,
                                       const PlannerConfig& cfg);

}  // namespace passplan
