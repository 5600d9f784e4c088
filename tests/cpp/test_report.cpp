// RunReport JSON (include/actmap/report.hpp; SPEC.md:365-371 examples) without a device:
// round trip to an equal structure, 8 targets -> 8 path entries, byte-stable output,
// timing block last, unknown schema versions and malformed text rejected.
// Built and run by tests/test_report_cpu.py.
#include <cmath>
#include <cstdio>
#include <string>

#include "actmap/errors.hpp"
#include "actmap/report.hpp"

using namespace actmap;

static int failures = 0;
#define CHECK(cond)                                              \
  do {                                                           \
    if (!(cond)) {                                               \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                \
    }                                                            \
  } while (0)

static size_t count(const std::string& s, const std::string& what) {
  size_t n = 0;
  for (size_t p = s.find(what); p != std::string::npos; p = s.find(what, p + 1)) ++n;
  return n;
}

int main() {
  // minimal report -> parses back to an equal structure
  {
    RunReport r;
    r.command = "plan";
    const std::string j = serialize_run_report(r);
    CHECK(j.rfind("{\"schema_version\":1,", 0) == 0);
    CHECK(parse_run_report(j) == r);
  }
  // full report with 8 targets -> exactly 8 path entries, exact round trip
  RunReport r;
  r.command = "validate";
  r.scene = SceneSummary{767, 881, 123456, 9, 8};
  r.config.layers = 350;
  r.config.auto_cap = 4000;
  r.config.mode = Mode::kIterative;
  r.config.method = Method::kSimple;
  r.config.seed = 0xFFFFFFFFFFFFFFFFull;
  r.config.corner_rule = CornerRule::kPermissive;
  r.config.threads = 16;
  r.layers_used = 350;
  r.termination = "fixed";
  r.max_activity = 351;
  r.bounds = LayerBound{349174, 1322, 1762};
  for (uint32_t i = 0; i < 8; ++i) {
    TargetReport t;
    t.target = Coord{i, 2 * i};
    t.covered = i != 3;
    if (t.covered) {
      t.reached_source = Coord{100 + i, 7};
      t.steps = i + 1;
      t.euclidean_length = i + std::sqrt(2.0) * (i % 3);
      for (uint32_t k = 0; k <= i + 1; ++k) t.points.push_back(Coord{i + k, 4294967295u - k});
    }
    r.paths.push_back(t);
  }
  ValidationReport v;
  v.layers_used = 350;
  v.termination = AutoStop::kStalled;
  v.bounds = *r.bounds;
  v.activity.violations = 2;
  v.activity.samples = {Coord{1, 2}, Coord{3, 4}};
  v.kernels_checked = true;
  v.kernel_mismatch = Coord{5, 6};
  TargetValidation tv;
  tv.target = Coord{9, 9};
  tv.covered = true;
  tv.simple_steps = 12;
  tv.bfs_hops = 12;
  tv.euclidean_length = 13.656854249492381;
  tv.octile_distance = 1.0 / 3.0;
  tv.euclidean_excess = 1e-300;
  v.targets = {tv, tv};
  v.covered_targets = 7;
  v.max_excess = 0.1 + 0.2;
  v.findings = {"nearest source \"disagrees\"\n", "tab\there"};
  r.validation = v;
  BenchReport b;
  b.samples = {BenchSample{1024, 1024, Mode::kBatched, 8, 5, 1.25, 1.0, false},
               BenchSample{65535, 1, Mode::kIterative, 1, 3, 0.0, 0.0, true}};
  b.fit = ScalingFit{std::nullopt, 2.5e-9, 1.0e-12, 0.04};
  b.mode_compare = ModeComparison{6.4, 193.0, 193.0 / 6.4};
  r.bench = b;
  r.timing = Timings{1.5, 2.25, 3.125, 0.0, 7.0};
  const std::string j = serialize_run_report(r);
  CHECK(count(j, "\"reached_source\"") == 8);
  const RunReport back = parse_run_report(j);
  CHECK(back == r);
  CHECK(back.paths.size() == 8 && back.paths[3].reached_source == std::nullopt);
  CHECK(serialize_run_report(back) == j);  // byte-stable
  // two identical runs differ only in the timing block, which comes last
  RunReport r2 = r;
  r2.timing = Timings{9, 9, 9, 9, 36};
  const std::string j2 = serialize_run_report(r2);
  const size_t cut = j.find("\"timing\":");
  CHECK(cut != std::string::npos && j.compare(0, cut, j2, 0, cut) == 0 && j != j2);
  CHECK(j.find("\"timing\":") > j.find("\"bench\":"));
  // empty sample lists ("samples": [] reads like an empty coordinate array) round-trip exactly
  {
    RunReport e = r;
    e.bench = BenchReport{};
    e.validation->activity.samples.clear();
    const std::string je = serialize_run_report(e);
    CHECK(parse_run_report(je) == e);
    CHECK(serialize_run_report(parse_run_report(je)) == je);
  }
  // rejections
  {
    std::string bad = j;
    bad.replace(bad.find("\"schema_version\":1"), 18, "\"schema_version\":2");
    bool threw = false;
    try {
      parse_run_report(bad);
    } catch (const InvalidInputError&) {
      threw = true;
    }
    CHECK(threw);
  }
  {
    bool pos = false;
    try {
      parse_run_report("{\n  \"schema_version\": 1,\n  \"command\": plan\n}");
    } catch (const ParseError& e) {
      pos = e.line() == 3 && e.column() == 14;
    }
    CHECK(pos);
  }
  {
    bool threw = false;
    try {
      parse_run_report("{\"schema_version\":1,\"command\":\"plan\"}");  // missing fields
    } catch (const InvalidInputError&) {
      threw = true;
    }
    CHECK(threw);
  }
  // LayerRule::layers_for (bench.hpp)
  LayerRule fixed{512, 1.0}, ratio{std::nullopt, 1.5};
  CHECK(fixed.layers_for(100) == 512 && ratio.layers_for(1001) == 1502);
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
