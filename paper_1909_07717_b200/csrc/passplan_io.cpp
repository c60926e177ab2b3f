// passplan_io.cpp -- the drop-in's JSON formats: world snapshots and planner
// configs (reference snapshot.cpp, config.cpp:14-241), with the same keys,
// type checks, unknown-key errors and error categories, on the same
// header-only nlohmann/json the reference builds against.  The CSV formats
// are in passplan_csv.cpp.  Host code, part of lib/libpassplan.so.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "passplan/passplan.hpp"

namespace passplan {

// ---- JSON world snapshots (snapshot.cpp) ----------------------------------------
namespace {

using nlohmann::json;

// Checks an object's keys: all of `need` present, nothing outside need+opt.
void check_keys(const json& o, const std::string& at, std::initializer_list<const char*> need,
                std::initializer_list<const char*> opt = {}) {
  for (const char* k : need)
    if (!o.contains(k)) throw schema_error(at + ": missing key '" + k + "'");
  for (const auto& it : o.items()) {
    bool known = false;
    for (const char* k : need) known = known || it.key() == k;
    for (const char* k : opt) known = known || it.key() == k;
    if (!known) throw schema_error(at + ": unknown key '" + it.key() + "'");
  }
}

double json_number(const json& o, const std::string& at, const char* key) {
  const json& v = o.at(key);
  if (!v.is_number()) throw schema_error(at + ": '" + key + "' must be a number");
  return v.get<double>();
}

std::vector<RobotState> json_team(const json& arr, const std::string& at) {
  if (!arr.is_array()) throw schema_error(at + ": must be an array");
  std::vector<RobotState> team;
  for (size_t i = 0; i < arr.size(); ++i) {
    const json& r = arr[i];
    const std::string where = at + "[" + std::to_string(i) + "]";
    if (!r.is_object()) throw schema_error(where + ": must be an object");
    check_keys(r, where, {"id", "x", "y", "vx", "vy", "theta"});
    if (!r.at("id").is_number_integer())
      throw schema_error(where + ": 'id' must be an integer");
    RobotState s;
    s.id = r.at("id").get<int>();
    s.position = {json_number(r, where, "x"), json_number(r, where, "y")};
    s.velocity = {json_number(r, where, "vx"), json_number(r, where, "vy")};
    s.theta = json_number(r, where, "theta");
    team.push_back(s);
  }
  return team;
}

}  // namespace

WorldState parse_world_snapshot(const std::string& bytes) {
  json root;
  try {
    root = json::parse(bytes);
  } catch (const json::parse_error& e) {
    throw schema_error(std::string("snapshot is not valid JSON: ") + e.what());
  }
  if (!root.is_object()) throw schema_error("snapshot: top level must be an object");
  check_keys(root, "snapshot", {"field", "ball", "ours", "theirs"});
  WorldState w;
  const json& f = root.at("field");
  if (!f.is_object()) throw schema_error("field: must be an object");
  check_keys(f, "field", {}, {"length", "width", "goal_width", "defense_depth", "defense_width"});
  struct {
    const char* key;
    double* dst;
  } const fields[] = {{"length", &w.field.length},
                      {"width", &w.field.width},
                      {"goal_width", &w.field.goal_width},
                      {"defense_depth", &w.field.defense_depth},
                      {"defense_width", &w.field.defense_width}};
  for (const auto& fd : fields)
    if (f.contains(fd.key)) *fd.dst = json_number(f, "field", fd.key);
  const json& b = root.at("ball");
  if (!b.is_object()) throw schema_error("ball: must be an object");
  check_keys(b, "ball", {"x", "y", "vx", "vy"});
  w.ball.position = {json_number(b, "ball", "x"), json_number(b, "ball", "y")};
  w.ball.velocity = {json_number(b, "ball", "vx"), json_number(b, "ball", "vy")};
  w.ours = json_team(root.at("ours"), "ours");
  w.theirs = json_team(root.at("theirs"), "theirs");
  w.validate();
  return w;
}

WorldState load_world_snapshot(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw schema_error("cannot open snapshot file: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return parse_world_snapshot(ss.str());
}

std::string serialize_world_snapshot(const WorldState& w) {
  auto robot = [](const RobotState& r) {
    return json{{"id", r.id},         {"x", r.position.x},  {"y", r.position.y},
                {"vx", r.velocity.x}, {"vy", r.velocity.y}, {"theta", r.theta}};
  };
  json root;
  root["field"] = {{"length", w.field.length},
                   {"width", w.field.width},
                   {"goal_width", w.field.goal_width},
                   {"defense_depth", w.field.defense_depth},
                   {"defense_width", w.field.defense_width}};
  root["ball"] = {{"x", w.ball.position.x},
                  {"y", w.ball.position.y},
                  {"vx", w.ball.velocity.x},
                  {"vy", w.ball.velocity.y}};
  root["ours"] = json::array();
  for (const RobotState& r : w.ours) root["ours"].push_back(robot(r));
  root["theirs"] = json::array();
  for (const RobotState& r : w.theirs) root["theirs"].push_back(robot(r));
  return root.dump(2) + "\n";
}

// ---- JSON planner config (config.cpp:14-241) ------------------------------------
namespace {

// Reads the known keys of one config object; unknown keys -> config_error.
class ConfigSection {
 public:
  ConfigSection(const json& obj, std::string path) : obj_(obj), path_(std::move(path)) {
    if (!obj.is_object()) throw config_error(path_ + ": must be an object");
  }
  void num(const char* key, double* out) {
    known_.push_back(key);
    if (!obj_.contains(key)) return;
    if (!obj_.at(key).is_number()) throw config_error(path_ + "." + key + ": must be a number");
    *out = obj_.at(key).get<double>();
  }
  void integer(const char* key, int* out) {
    known_.push_back(key);
    if (!obj_.contains(key)) return;
    if (!obj_.at(key).is_number_integer())
      throw config_error(path_ + "." + key + ": must be an integer");
    *out = obj_.at(key).get<int>();
  }
  void flag(const char* key, bool* out) {
    known_.push_back(key);
    if (!obj_.contains(key)) return;
    if (!obj_.at(key).is_boolean()) throw config_error(path_ + "." + key + ": must be a boolean");
    *out = obj_.at(key).get<bool>();
  }
  void text(const char* key) {
    known_.push_back(key);
    if (obj_.contains(key) && !obj_.at(key).is_string())
      throw config_error(path_ + "." + key + ": must be a string");
  }
  void sub(const char* key, const std::function<void(const json&, const std::string&)>& f) {
    known_.push_back(key);
    if (obj_.contains(key)) f(obj_.at(key), path_ + "." + key);
  }
  void done() const {
    for (const auto& it : obj_.items()) {
      if (std::find(known_.begin(), known_.end(), it.key()) == known_.end())
        throw config_error(path_ + ": unknown key '" + it.key() + "'");
    }
  }

 private:
  const json& obj_;
  std::string path_;
  std::vector<std::string> known_;
};

}  // namespace

PlannerConfig PlannerConfig::from_json_text(const std::string& text) {
  json root;
  try {
    root = json::parse(text);
  } catch (const json::parse_error& e) {
    throw config_error(std::string("config is not valid JSON: ") + e.what());
  }
  PlannerConfig c;
  double px_per_m = 100.0;
  ConfigSection s(root, "config");
  s.sub("ball", [&](const json& j, const std::string& p) {
    ConfigSection b(j, p);
    b.num("slide_decel", &c.ball.slide_decel);
    b.num("roll_decel", &c.ball.roll_decel);
    b.num("transition_ratio", &c.ball.transition_ratio);
    b.num("power_min", &c.ball.power_min);
    b.num("power_max", &c.ball.power_max);
    b.num("chip_flight_fraction", &c.ball.chip_flight_fraction);
    b.done();
  });
  for (const char* team : {"motion_ours", "motion_theirs"}) {
    MotionLimits* m = std::string(team) == "motion_ours" ? &c.motion_ours : &c.motion_theirs;
    s.sub(team, [&](const json& j, const std::string& p) {
      ConfigSection ms(j, p);
      ms.num("max_speed", &m->max_speed);
      ms.num("max_accel", &m->max_accel);
      ms.num("max_decel", &m->max_decel);
      ms.done();
    });
  }
  s.sub("grid", [&](const json& j, const std::string& p) {
    ConfigSection g(j, p);
    g.integer("n_directions", &c.grid.n_directions);
    g.integer("n_powers", &c.grid.n_powers);
    g.num("power_min", &c.grid.power_min);
    g.num("power_max", &c.grid.power_max);
    g.flag("flat", &c.grid.flat);
    g.flag("chip", &c.grid.chip);
    g.done();
  });
  s.sub("pass_weights", [&](const json& j, const std::string& p) {
    ConfigSection w(j, p);
    PassWeights& pw = c.weights.pass;
    w.num("teammate_time", &pw.teammate_time);
    w.num("shoot_angle", &pw.shoot_angle);
    w.num("dist_goal", &pw.dist_goal);
    w.num("refraction", &pw.refraction);
    w.num("margin", &pw.margin);
    w.done();
  });
  s.sub("run_weights", [&](const json& j, const std::string& p) {
    ConfigSection w(j, p);
    RunWeights& rw = c.weights.run;
    w.num("dist_goal", &rw.dist_goal);
    w.num("dist_ball", &rw.dist_ball);
    w.num("angle", &rw.angle);
    w.num("guard_time", &rw.guard_time);
    w.num("exposure", &rw.exposure);
    w.done();
  });
  s.sub("norm", [&](const json& j, const std::string& p) {
    ConfigSection n(j, p);
    n.num("length_upper", &c.weights.norm.length_upper);
    n.num("angle_upper", &c.weights.norm.angle_upper);
    n.done();
  });
  s.sub("angle_band", [&](const json& j, const std::string& p) {
    ConfigSection a(j, p);
    a.num("full_lo", &c.angle_band.full_lo);
    a.num("peak_lo", &c.angle_band.peak_lo);
    a.num("peak_hi", &c.angle_band.peak_hi);
    a.num("full_hi", &c.angle_band.full_hi);
    a.done();
  });
  s.sub("thresholds", [&](const json& j, const std::string& p) {
    ConfigSection t(j, p);
    PlannerThresholds& th = c.thresholds;
    t.num("sbip_dt", &th.sbip_dt);
    t.num("robot_radius", &th.robot_radius);
    t.num("safety_margin", &th.safety_margin);
    t.num("buffer_time", &th.buffer_time);
    t.num("possession_radius", &th.possession_radius);
    t.num("angle_threshold", &th.angle_threshold);
    t.num("shot_power", &th.shot_power);
    t.num("margin_cap", &th.margin_cap);
    t.num("possession_dt", &th.possession_dt);
    t.num("contest_epsilon", &th.contest_epsilon);
    t.num("grid_step", &th.grid_step);
    t.num("min_zone_width", &th.min_zone_width);
    t.num("guard_time_cap", &th.guard_time_cap);
    t.num("drag_v_min", &th.drag_v_min);
    t.num("marking_radius", &th.marking_radius);
    t.done();
  });
  s.sub("svg", [&](const json& j, const std::string& p) {  // accepted, not stored
    ConfigSection v(j, p);
    v.num("pixels_per_meter", &px_per_m);
    for (const char* k : {"field_color", "line_color", "our_color", "their_color", "ball_color",
                          "flat_feasible_color", "chip_feasible_color", "best_flat_color",
                          "best_chip_color"})
      v.text(k);
    v.done();
  });
  s.done();
  c.validate();
  if (!(px_per_m > 0.0)) throw config_error("svg.pixels_per_meter must be > 0");
  return c;
}

PlannerConfig PlannerConfig::load(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw config_error("cannot open config file: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return from_json_text(ss.str());
}

}  // namespace passplan
