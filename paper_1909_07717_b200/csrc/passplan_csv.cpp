// passplan_csv.cpp -- the drop-in's CSV formats (reference csv.hpp): the
// candidate grid (`plan --out`), the pass heat map and the running-point heat
// map, plus the text-file helpers.  Host code, part of lib/libpassplan.so.
//
// The format is the contract, not the code: headers, column order, "%.17g"
// numbers with +inf written as "never", '\n' line ends, and the reader's
// error categories/messages ("csv line N: ...", N counting non-empty lines)
// follow the reference (csv.cpp:70-295) so files and
// diagnostics are byte-identical.  The implementation is table driven: one
// row writer that places separators, one record reader with typed column
// accessors, and the numeric tables described by their column lists.
#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <vector>

#include "passplan/passplan.hpp"

namespace passplan {

namespace {

constexpr std::string_view kGridColumns =
    "kick_type,dir_index,power_index,angle,power,our_id,our_time,opp_id,opp_time,"
    "receive_x,receive_y,feasible";
constexpr std::string_view kHeatColumns = "x,y,value";
constexpr std::string_view kRunColumns =
    "x,y,dist_goal,dist_ball,angle_goal,guard_time,exposure,score";

// "%.17g" via to_chars (general format, precision 17 is specified as printf's
// %.17g), +inf as "never".
void put_double(std::string* out, double v) {
  if (v == kNever) {
    out->append("never");
    return;
  }
  char buf[40];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::general, 17);
  out->append(buf, r.ptr);
}

// Appends one CSV row field by field; the separator goes in front of every
// field but the first, end() closes the row.
class RowWriter {
 public:
  explicit RowWriter(std::string* out) : out_(out) {}
  RowWriter& number(double v) {
    separate();
    put_double(out_, v);
    return *this;
  }
  RowWriter& integer(long v) {
    separate();
    char buf[24];
    const auto r = std::to_chars(buf, buf + sizeof(buf), v);
    out_->append(buf, r.ptr);
    return *this;
  }
  RowWriter& word(std::string_view s) {
    separate();
    out_->append(s);
    return *this;
  }
  void end() {
    out_->push_back('\n');
    fresh_ = true;
  }

 private:
  void separate() {
    if (!fresh_) out_->push_back(',');
    fresh_ = false;
  }
  std::string* out_;
  bool fresh_ = true;
};

std::string with_header(std::string_view header, size_t rows, size_t bytes_per_row) {
  std::string out;
  out.reserve(header.size() + 1 + rows * bytes_per_row);
  out.append(header);
  out.push_back('\n');
  return out;
}

// One data record: its comma-separated fields and its number among the
// non-empty lines (1 = the header), used in every diagnostic.
struct Record {
  std::vector<std::string_view> fields;
  size_t number = 0;

  [[noreturn]] void fail(const std::string& what) const {
    throw schema_error("csv line " + std::to_string(number) + ": " + what);
  }
  void expect_fields(size_t n) const {
    if (fields.size() != n) fail("expected " + std::to_string(n) + " fields");
  }
  int integer(size_t k) const {
    const std::string f(fields[k]);
    if (f.empty()) fail("empty integer field");
    char* end = nullptr;
    const long v = std::strtol(f.c_str(), &end, 10);
    if (end != f.c_str() + f.size()) fail("bad integer '" + f + "'");
    return static_cast<int>(v);
  }
  double number_at(size_t k) const {
    try {
      return parse_double_field(std::string(fields[k]));
    } catch (const Error& e) {
      fail(e.what());
    }
  }
};

// Walks the non-empty lines of a text ('\n' separated, a trailing '\r'
// dropped); the first one is the header.
class RecordReader {
 public:
  explicit RecordReader(const std::string& text) : rest_(text) {}

  bool next_line(std::string_view* line) {
    while (!rest_.empty()) {
      const size_t nl = rest_.find('\n');
      std::string_view l = rest_.substr(0, nl);
      rest_ = nl == std::string_view::npos ? std::string_view() : rest_.substr(nl + 1);
      if (!l.empty() && l.back() == '\r') l.remove_suffix(1);
      if (l.empty()) continue;
      ++count_;
      *line = l;
      return true;
    }
    return false;
  }

  bool next(Record* r) {
    std::string_view line;
    if (!next_line(&line)) return false;
    r->fields.clear();
    r->number = count_;
    for (size_t from = 0;;) {
      const size_t comma = line.find(',', from);
      r->fields.push_back(line.substr(from, comma == std::string_view::npos ? line.npos
                                                                              : comma - from));
      if (comma == std::string_view::npos) break;
      from = comma + 1;
    }
    return true;
  }

 private:
  std::string_view rest_;
  size_t count_ = 0;
};

// A header-checked table of doubles with a fixed column count.
std::vector<std::vector<double>> read_numeric_table(const std::string& text,
                                                    std::string_view header,
                                                    const char* header_error) {
  RecordReader in(text);
  std::string_view first;
  if (!in.next_line(&first) || first != header) throw schema_error(header_error);
  const size_t cols = static_cast<size_t>(std::count(header.begin(), header.end(), ',')) + 1;
  std::vector<std::vector<double>> rows;
  Record r;
  while (in.next(&r)) {
    r.expect_fields(cols);
    std::vector<double>& row = rows.emplace_back(cols);
    for (size_t k = 0; k < cols; ++k) row[k] = r.number_at(k);
  }
  return rows;
}

}  // namespace

std::string format_double(double v) {
  std::string s;
  put_double(&s, v);
  return s;
}

double parse_double_field(const std::string& field) {
  if (field == "never") return kNever;
  if (field.empty()) throw schema_error("empty number field");
  const char* begin = field.c_str();
  char* end = nullptr;
  const double v = std::strtod(begin, &end);  // strtod's grammar, whole field consumed
  if (end != begin + field.size()) throw schema_error("bad number '" + field + "'");
  return v;
}

// ---- candidate grid (csv.hpp: grid_to_csv / grid_from_csv) --------------------

std::string grid_to_csv(const CandidateGrid& g) {
  std::string out = with_header(kGridColumns, g.cells.size(), 160);
  RowWriter row(&out);
  for (const PassCandidate& c : g.cells) {
    row.word(c.kick_type == KickType::chip ? "chip" : "flat")
        .integer(c.dir_index)
        .integer(c.power_index)
        .number(direction_angle(c.dir_index, g.grid.n_directions))
        .number(g.powers[static_cast<size_t>(c.power_index)])
        .integer(c.our_id)
        .number(c.our_time)
        .integer(c.opp_id)
        .number(c.opp_time)
        .number(c.receive_point.x)
        .number(c.receive_point.y)
        .word(c.feasible ? "1" : "0")
        .end();
  }
  return out;
}

CandidateGrid grid_from_csv(const std::string& text) {
  RecordReader in(text);
  std::string_view header;
  if (!in.next_line(&header)) throw schema_error("csv: empty input");
  if (header != kGridColumns) throw schema_error("csv line 1: unexpected header");

  std::vector<PassCandidate> cells;
  std::vector<double> row_power;
  bool kinds[2] = {false, false};  // flat, chip present
  int n_dirs = 0, n_powers = 0;
  Record r;
  while (in.next(&r)) {
    r.expect_fields(12);
    PassCandidate c;
    const std::string_view kind = r.fields[0];
    if (kind != "flat" && kind != "chip") r.fail("unknown kick type '" + std::string(kind) + "'");
    c.kick_type = kind == "chip" ? KickType::chip : KickType::flat;
    kinds[kind == "chip"] = true;
    c.dir_index = r.integer(1);
    c.power_index = r.integer(2);
    (void)r.number_at(3);  // the angle column is a function of dir_index; validated, not kept
    const double power = r.number_at(4);
    c.our_id = r.integer(5);
    c.our_time = r.number_at(6);
    c.opp_id = r.integer(7);
    c.opp_time = r.number_at(8);
    c.receive_point = {r.number_at(9), r.number_at(10)};
    const std::string_view flag = r.fields[11];
    if (flag != "0" && flag != "1") r.fail("feasible must be 0 or 1");
    c.feasible = flag == "1";
    if (c.dir_index < 0 || c.power_index < 0) r.fail("negative index");
    n_dirs = std::max(n_dirs, c.dir_index + 1);
    n_powers = std::max(n_powers, c.power_index + 1);
    cells.push_back(c);
    row_power.push_back(power);
  }
  if (cells.empty()) throw schema_error("csv: no data rows");

  CandidateGrid g;
  g.grid.n_directions = n_dirs;
  g.grid.n_powers = n_powers;
  g.grid.flat = kinds[0];
  g.grid.chip = kinds[1];
  g.kick_types = g.grid.kick_types();
  g.directions = direction_table(n_dirs);
  g.powers.assign(static_cast<size_t>(n_powers), 0.0);
  const size_t want = g.kick_types.size() * static_cast<size_t>(n_dirs) * n_powers;
  if (cells.size() != want)
    throw schema_error("csv: " + std::to_string(cells.size()) + " rows, expected " +
                       std::to_string(want));
  g.cells.assign(want, PassCandidate{});
  for (size_t i = 0; i < cells.size(); ++i) {
    const PassCandidate& c = cells[i];
    const int slot = c.kick_type == KickType::chip && g.grid.flat ? 1 : 0;
    g.cells[static_cast<size_t>(g.cell_index(slot, c.dir_index, c.power_index))] = c;
    g.powers[static_cast<size_t>(c.power_index)] = row_power[i];
  }
  g.grid.power_min = g.powers.front();
  g.grid.power_max = g.powers.back();
  return g;
}

// ---- heat maps (csv.hpp: heatmap_*, run_heatmap_*) ------------------------------

std::string heatmap_to_csv(const std::vector<HeatPoint>& points) {
  std::string out = with_header(kHeatColumns, points.size(), 64);
  RowWriter row(&out);
  for (const HeatPoint& p : points) row.number(p.point.x).number(p.point.y).number(p.value).end();
  return out;
}

std::vector<HeatPoint> heatmap_from_csv(const std::string& text) {
  std::vector<HeatPoint> out;
  for (const auto& v : read_numeric_table(text, kHeatColumns, "csv line 1: expected x,y,value"))
    out.push_back({{v[0], v[1]}, v[2]});
  return out;
}

std::string run_heatmap_to_csv(const std::vector<RunHeatRow>& rows) {
  std::string out = with_header(kRunColumns, rows.size(), 180);
  RowWriter row(&out);
  for (const RunHeatRow& r : rows) {
    const RunningPointFeatures& f = r.features;
    row.number(r.point.x).number(r.point.y).number(f.dist_to_goal).number(f.dist_to_ball);
    row.number(f.angle_to_goal).number(f.guard_time).number(f.defense_exposure).number(r.score);
    row.end();
  }
  return out;
}

std::vector<RunHeatRow> run_heatmap_from_csv(const std::string& text) {
  std::vector<RunHeatRow> out;
  for (const auto& v :
       read_numeric_table(text, kRunColumns, "csv line 1: unexpected run-heatmap header")) {
    RunHeatRow r;
    r.point = {v[0], v[1]};
    r.features = {v[2], v[3], v[4], v[5], v[6]};
    r.score = v[7];
    out.push_back(r);
  }
  return out;
}

// ---- files ----------------------------------------------------------------------

std::string read_text_file(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw config_error("cannot open " + path);
  std::string text;
  char buf[1 << 16];
  for (size_t n; (n = std::fread(buf, 1, sizeof(buf), f)) > 0;) text.append(buf, n);
  std::fclose(f);
  return text;
}

// Written to PATH.tmp and renamed over PATH, so readers never see a torn file.
void write_text_file(const std::string& path, const std::string& text) {
  const std::string tmp = path + ".tmp";
  std::FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) throw config_error("cannot write " + tmp);
  const bool complete = std::fwrite(text.data(), 1, text.size(), f) == text.size();
  const bool closed = std::fclose(f) == 0;
  if (!complete || !closed) throw config_error("short write to " + tmp);
  if (std::rename(tmp.c_str(), path.c_str()) != 0)
    throw config_error("cannot rename " + tmp + " to " + path + ": " + std::strerror(errno));
}

}  // namespace passplan
