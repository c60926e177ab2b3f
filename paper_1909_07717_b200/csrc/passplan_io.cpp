// passplan_io.cpp -- the drop-in's file formats: the reference's CSV outputs
// (csv.hpp / csv.cpp:70-295) and its JSON world snapshots and planner configs
// (snapshot.cpp, config.cpp:14-241).  Host code, part of lib/libpassplan.so.
//
// The CSV writers reproduce the reference byte for byte (%.17g, "never" for
// +inf, fixed headers, '\n' line ends); tests/test_gpu_cli.py compares the
// CLI's files with the reference's own.  JSON uses the same header-only
// nlohmann/json the reference builds against.
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

namespace {

using nlohmann::json;

constexpr const char* kGridHeader =
    "kick_type,dir_index,power_index,angle,power,our_id,our_time,opp_id,opp_time,"
    "receive_x,receive_y,feasible";
constexpr const char* kHeatHeader = "x,y,value";
constexpr const char* kRunHeader = "x,y,dist_goal,dist_ball,angle_goal,guard_time,exposure,score";

// Lines without their '\n' (and a trailing '\r'); empty lines are skipped.
std::vector<std::string> lines_of(const std::string& text) {
  std::vector<std::string> out;
  std::string cur;
  std::istringstream in(text);
  while (std::getline(in, cur)) {
    if (!cur.empty() && cur.back() == '\r') cur.pop_back();
    if (!cur.empty()) out.push_back(cur);
  }
  return out;
}

std::vector<std::string> fields_of(const std::string& line) {
  std::vector<std::string> out(1);
  for (char ch : line) {
    if (ch == ',') {
      out.emplace_back();
    } else {
      out.back().push_back(ch);
    }
  }
  return out;
}

[[noreturn]] void row_error(size_t line, const std::string& what) {
  throw schema_error("csv line " + std::to_string(line) + ": " + what);
}

int int_field(const std::string& f, size_t line) {
  if (f.empty()) row_error(line, "empty integer field");
  char* end = nullptr;
  const long v = std::strtol(f.c_str(), &end, 10);
  if (end != f.c_str() + f.size()) row_error(line, "bad integer '" + f + "'");
  return static_cast<int>(v);
}

double num_field(const std::string& f, size_t line) {
  try {
    return parse_double_field(f);
  } catch (const Error& e) {
    row_error(line, e.what());
  }
}

void append_num(std::string* out, double v) {
  *out += format_double(v);
}

}  // namespace

std::string format_double(double v) {
  if (std::isinf(v) && v > 0.0) return "never";
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

double parse_double_field(const std::string& field) {
  if (field == "never") return kNever;
  if (field.empty()) throw schema_error("empty number field");
  char* end = nullptr;
  const double v = std::strtod(field.c_str(), &end);
  if (end != field.c_str() + field.size()) throw schema_error("bad number '" + field + "'");
  return v;
}

std::string grid_to_csv(const CandidateGrid& g) {
  std::string out = kGridHeader;
  out += '\n';
  out.reserve(out.size() + g.cells.size() * 140);
  for (const PassCandidate& c : g.cells) {
    out += c.kick_type == KickType::flat ? "flat," : "chip,";
    out += std::to_string(c.dir_index) + ',' + std::to_string(c.power_index) + ',';
    append_num(&out, direction_angle(c.dir_index, g.grid.n_directions));
    out += ',';
    append_num(&out, g.powers[static_cast<size_t>(c.power_index)]);
    out += ',' + std::to_string(c.our_id) + ',';
    append_num(&out, c.our_time);
    out += ',' + std::to_string(c.opp_id) + ',';
    append_num(&out, c.opp_time);
    out += ',';
    append_num(&out, c.receive_point.x);
    out += ',';
    append_num(&out, c.receive_point.y);
    out += c.feasible ? ",1\n" : ",0\n";
  }
  return out;
}

CandidateGrid grid_from_csv(const std::string& text) {
  const std::vector<std::string> lines = lines_of(text);
  if (lines.empty()) throw schema_error("csv: empty input");
  if (lines[0] != kGridHeader) throw schema_error("csv line 1: unexpected header");
  struct Row {
    PassCandidate cell;
    double power;
  };
  std::vector<Row> rows;
  int n_dirs = 0, n_powers = 0;
  bool has_flat = false, has_chip = false;
  for (size_t i = 1; i < lines.size(); ++i) {
    const size_t ln = i + 1;
    const std::vector<std::string> f = fields_of(lines[i]);
    if (f.size() != 12) row_error(ln, "expected 12 fields");
    Row r{};
    if (f[0] == "flat") {
      r.cell.kick_type = KickType::flat;
      has_flat = true;
    } else if (f[0] == "chip") {
      r.cell.kick_type = KickType::chip;
      has_chip = true;
    } else {
      row_error(ln, "unknown kick type '" + f[0] + "'");
    }
    r.cell.dir_index = int_field(f[1], ln);
    r.cell.power_index = int_field(f[2], ln);
    num_field(f[3], ln);  // the angle follows from dir_index: checked only
    r.power = num_field(f[4], ln);
    r.cell.our_id = int_field(f[5], ln);
    r.cell.our_time = num_field(f[6], ln);
    r.cell.opp_id = int_field(f[7], ln);
    r.cell.opp_time = num_field(f[8], ln);
    r.cell.receive_point = {num_field(f[9], ln), num_field(f[10], ln)};
    if (f[11] != "0" && f[11] != "1") row_error(ln, "feasible must be 0 or 1");
    r.cell.feasible = f[11] == "1";
    if (r.cell.dir_index < 0 || r.cell.power_index < 0) row_error(ln, "negative index");
    n_dirs = std::max(n_dirs, r.cell.dir_index + 1);
    n_powers = std::max(n_powers, r.cell.power_index + 1);
    rows.push_back(r);
  }
  if (rows.empty()) throw schema_error("csv: no data rows");
  CandidateGrid g;
  g.grid.n_directions = n_dirs;
  g.grid.n_powers = n_powers;
  g.grid.flat = has_flat;
  g.grid.chip = has_chip;
  g.kick_types = g.grid.kick_types();
  g.directions = direction_table(n_dirs);
  g.powers.assign(static_cast<size_t>(n_powers), 0.0);
  const size_t expected = g.kick_types.size() * size_t(n_dirs) * size_t(n_powers);
  if (rows.size() != expected)
    throw schema_error("csv: " + std::to_string(rows.size()) + " rows, expected " +
                       std::to_string(expected));
  g.cells.assign(expected, PassCandidate{});
  for (const Row& r : rows) {
    const int slot = (r.cell.kick_type == KickType::chip && has_flat) ? 1 : 0;
    g.cells[static_cast<size_t>(g.cell_index(slot, r.cell.dir_index, r.cell.power_index))] = r.cell;
    g.powers[static_cast<size_t>(r.cell.power_index)] = r.power;
  }
  g.grid.power_min = g.powers.front();
  g.grid.power_max = g.powers.back();
  return g;
}

std::string heatmap_to_csv(const std::vector<HeatPoint>& points) {
  std::string out = std::string(kHeatHeader) + '\n';
  for (const HeatPoint& p : points) {
    append_num(&out, p.point.x);
    out += ',';
    append_num(&out, p.point.y);
    out += ',';
    append_num(&out, p.value);
    out += '\n';
  }
  return out;
}

std::vector<HeatPoint> heatmap_from_csv(const std::string& text) {
  const std::vector<std::string> lines = lines_of(text);
  if (lines.empty() || lines[0] != kHeatHeader)
    throw schema_error("csv line 1: expected x,y,value");
  std::vector<HeatPoint> out;
  for (size_t i = 1; i < lines.size(); ++i) {
    const std::vector<std::string> f = fields_of(lines[i]);
    if (f.size() != 3) row_error(i + 1, "expected 3 fields");
    out.push_back({{num_field(f[0], i + 1), num_field(f[1], i + 1)}, num_field(f[2], i + 1)});
  }
  return out;
}

std::string run_heatmap_to_csv(const std::vector<RunHeatRow>& rows) {
  std::string out = std::string(kRunHeader) + '\n';
  for (const RunHeatRow& r : rows) {
    const double v[8] = {r.point.x,
                         r.point.y,
                         r.features.dist_to_goal,
                         r.features.dist_to_ball,
                         r.features.angle_to_goal,
                         r.features.guard_time,
                         r.features.defense_exposure,
                         r.score};
    for (int k = 0; k < 8; ++k) {
      if (k) out += ',';
      append_num(&out, v[k]);
    }
    out += '\n';
  }
  return out;
}

std::vector<RunHeatRow> run_heatmap_from_csv(const std::string& text) {
  const std::vector<std::string> lines = lines_of(text);
  if (lines.empty() || lines[0] != kRunHeader)
    throw schema_error("csv line 1: unexpected run-heatmap header");
  std::vector<RunHeatRow> out;
  for (size_t i = 1; i < lines.size(); ++i) {
    const std::vector<std::string> f = fields_of(lines[i]);
    if (f.size() != 8) row_error(i + 1, "expected 8 fields");
    double v[8];
    for (int k = 0; k < 8; ++k) v[k] = num_field(f[k], i + 1);
    RunHeatRow r;
    r.point = {v[0], v[1]};
    r.features = {v[2], v[3], v[4], v[5], v[6]};
    r.score = v[7];
    out.push_back(r);
  }
  return out;
}

std::string read_text_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw config_error("cannot open " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

void write_text_file(const std::string& path, const std::string& text) {
  const std::string tmp = path + ".tmp";
  {
    std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
    if (!out) throw config_error("cannot write " + tmp);
    out << text;
    if (!out.flush()) throw config_error("short write to " + tmp);
  }
  std::error_code ec;
  std::filesystem::rename(tmp, path, ec);
  if (ec) throw config_error("cannot rename " + tmp + " to " + path + ": " + ec.message());
}

// ---- JSON world snapshots (snapshot.cpp) ----------------------------------------
namespace {

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
