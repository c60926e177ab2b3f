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
#include <iterator>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "passplan/passplan.hpp"

namespace passplan {

// ---- JSON world snapshots (snapshot.hpp) -----------------------------------------
// Schema-driven: every object is described by its keys (required or optional,
// each with a reader), and one routine enforces the reference's rules in its
// order -- object type, missing required keys (schema order), unknown keys,
// then the values (schema order) -- so malformed input gets the same
// schema_error text as from the reference (snapshot.cpp:17-95).
namespace {

using nlohmann::json;
using Reader = std::function<void(const json&, const std::string&)>;

struct SchemaKey {
  const char* name;
  bool required;
  Reader read;
};

void read_object(const json& v, const std::string& where, const std::vector<SchemaKey>& keys,
                 const char* not_object = nullptr) {
  if (!v.is_object())
    throw schema_error(not_object ? std::string(not_object) : where + ": must be an object");
  for (const SchemaKey& k : keys)
    if (k.required && !v.contains(k.name))
      throw schema_error(where + ": missing key '" + k.name + "'");
  for (const auto& item : v.items()) {
    const bool known = std::any_of(keys.begin(), keys.end(),
                                   [&](const SchemaKey& k) { return item.key() == k.name; });
    if (!known) throw schema_error(where + ": unknown key '" + item.key() + "'");
  }
  for (const SchemaKey& k : keys)
    if (v.contains(k.name)) k.read(v.at(k.name), where);
}

Reader number_into(double* dst, const char* key) {
  return [dst, key](const json& x, const std::string& where) {
    if (!x.is_number()) throw schema_error(where + ": '" + key + "' must be a number");
    *dst = x.get<double>();
  };
}

Reader integer_into(int* dst, const char* key) {
  return [dst, key](const json& x, const std::string& where) {
    if (!x.is_number_integer()) throw schema_error(where + ": '" + key + "' must be an integer");
    *dst = x.get<int>();
  };
}

std::vector<SchemaKey> robot_schema(RobotState* r) {
  return {{"id", true, integer_into(&r->id, "id")},
          {"x", true, number_into(&r->position.x, "x")},
          {"y", true, number_into(&r->position.y, "y")},
          {"vx", true, number_into(&r->velocity.x, "vx")},
          {"vy", true, number_into(&r->velocity.y, "vy")},
          {"theta", true, number_into(&r->theta, "theta")}};
}

Reader team_into(std::vector<RobotState>* team, const char* key) {
  return [team, key](const json& x, const std::string&) {
    if (!x.is_array()) throw schema_error(std::string(key) + ": must be an array");
    team->assign(x.size(), RobotState{});
    for (size_t i = 0; i < x.size(); ++i)
      read_object(x[i], std::string(key) + "[" + std::to_string(i) + "]",
                  robot_schema(&(*team)[i]));
  };
}

std::string file_text(const std::string& path, ErrorCategory cat, const char* what) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(cat, std::string("cannot open ") + what + " file: " + path);
  return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

}  // namespace

WorldState parse_world_snapshot(const std::string& bytes) {
  json root;
  try {
    root = json::parse(bytes);
  } catch (const json::parse_error& e) {
    throw schema_error(std::string("snapshot is not valid JSON: ") + e.what());
  }
  WorldState w;
  FieldGeometry& f = w.field;
  const std::vector<SchemaKey> field_keys = {
      {"length", false, number_into(&f.length, "length")},
      {"width", false, number_into(&f.width, "width")},
      {"goal_width", false, number_into(&f.goal_width, "goal_width")},
      {"defense_depth", false, number_into(&f.defense_depth, "defense_depth")},
      {"defense_width", false, number_into(&f.defense_width, "defense_width")}};
  const std::vector<SchemaKey> ball_keys = {
      {"x", true, number_into(&w.ball.position.x, "x")},
      {"y", true, number_into(&w.ball.position.y, "y")},
      {"vx", true, number_into(&w.ball.velocity.x, "vx")},
      {"vy", true, number_into(&w.ball.velocity.y, "vy")}};
  read_object(root, "snapshot",
              {{"field", true, [&](const json& x, const std::string&) {
                  read_object(x, "field", field_keys);
                }},
               {"ball", true, [&](const json& x, const std::string&) {
                  read_object(x, "ball", ball_keys);
                }},
               {"ours", true, team_into(&w.ours, "ours")},
               {"theirs", true, team_into(&w.theirs, "theirs")}},
              "snapshot: top level must be an object");
  w.validate();
  return w;
}

WorldState load_world_snapshot(const std::string& path) {
  return parse_world_snapshot(file_text(path, ErrorCategory::schema, "snapshot"));
}

// (nlohmann::json objects keep their keys sorted, so the text does not depend
// on the order they are set in)
std::string serialize_world_snapshot(const WorldState& w) {
  json root = json::object();
  const FieldGeometry& f = w.field;
  for (const auto& [k, v] : {std::pair<const char*, double>{"length", f.length},
                             {"width", f.width},
                             {"goal_width", f.goal_width},
                             {"defense_depth", f.defense_depth},
                             {"defense_width", f.defense_width}})
    root["field"][k] = v;
  root["ball"]["x"] = w.ball.position.x;
  root["ball"]["y"] = w.ball.position.y;
  root["ball"]["vx"] = w.ball.velocity.x;
  root["ball"]["vy"] = w.ball.velocity.y;
  for (const auto& [key, team] : {std::pair<const char*, const std::vector<RobotState>*>{
                                      "ours", &w.ours},
                                  {"theirs", &w.theirs}}) {
    json arr = json::array();
    for (const RobotState& r : *team) {
      json o = json::object();
      o["id"] = r.id;
      o["x"] = r.position.x;
      o["y"] = r.position.y;
      o["vx"] = r.velocity.x;
      o["vy"] = r.velocity.y;
      o["theta"] = r.theta;
      arr.push_back(std::move(o));
    }
    root[key] = std::move(arr);
  }
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
  return from_json_text(file_text(path, ErrorCategory::config, "config"));
}

}  // namespace passplan
