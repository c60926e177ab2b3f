// csv_roundtrip.cpp -- CPU test driver for the drop-in's CSV formats
// (passplan_csv.cpp): reads a CSV text on stdin, parses it with the reader
// named by argv[1] (grid | heat | run) and writes it back with the matching
// writer, or prints "ERROR <category>: <message>" when the reader throws --
// the same contract as oracle/ref_shim.cpp's ref_csv_roundtrip, so
// tests/test_csv_cpu.py can compare both byte for byte; "snapshot" and
// "config" do the same for the JSON readers.  No GPU is used.
#include <cstdio>
#include <iostream>
#include <iterator>
#include <string>

#include "passplan/passplan.hpp"

int main(int argc, char** argv) {
  const std::string kind = argc > 1 ? argv[1] : "grid";
  const std::string text((std::istreambuf_iterator<char>(std::cin)), std::istreambuf_iterator<char>());
  std::string out;
  try {
    if (kind == "grid") {
      out = passplan::grid_to_csv(passplan::grid_from_csv(text));
    } else if (kind == "snapshot") {
      out = passplan::serialize_world_snapshot(passplan::parse_world_snapshot(text));
    } else if (kind == "config") {
      const passplan::PlannerConfig c = passplan::PlannerConfig::from_json_text(text);
      char buf[160];
      std::snprintf(buf, sizeof buf, "OK %.17g %.17g %d %d %.17g", c.ball.slide_decel,
                    c.thresholds.sbip_dt, c.grid.n_directions, c.grid.chip ? 1 : 0,
                    c.weights.pass.margin);
      out = buf;
    } else if (kind == "heat") {
      out = passplan::heatmap_to_csv(passplan::heatmap_from_csv(text));
    } else {
      out = passplan::run_heatmap_to_csv(passplan::run_heatmap_from_csv(text));
    }
  } catch (const passplan::Error& e) {
    out = std::string("ERROR ") + passplan::category_name(e.category()) + ": " + e.what();
  }
  std::fwrite(out.data(), 1, out.size(), stdout);
  return 0;
}
