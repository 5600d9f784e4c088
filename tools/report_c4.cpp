// C4 planner run through the C++ drop-in API with RunReport emission:
// random_maze(23170, 0.40, seed 4), 64 sources, 4096 targets, propagate_auto on the resident
// grid, every path traced on the device into TargetReport entries, the report serialised to
// JSON and parsed back.  Prints one JSON line of phase timings (wall clock).
//   g++ -std=c++20 -O2 -Iinclude tools/report_c4.cpp -Lpaper_2004_00540_b200 -lactmap_b200 \
//       -Wl,-rpath,$PWD/paper_2004_00540_b200 -o /tmp/report_c4 && /tmp/report_c4
#include <chrono>
#include <cstdio>
#include <vector>

#include "actmap/b200.hpp"
#include "actmap/report.hpp"

using namespace actmap;
using Clock = std::chrono::steady_clock;

static double ms(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double, std::milli>(b - a).count();
}

int main() {
  const uint32_t n = 23170;
  // process-wide CUDA / context start-up, measured apart from the C4 upload
  const auto tw0 = Clock::now();
  {
    const GridMap tiny = build_grid(8, 8, {});
    const std::vector<Coord> ts{{0, 0}};
    const SourceSet tsrc(tiny, ts);
    (void)propagate(tiny, tsrc, 1);
  }
  const auto tw1 = Clock::now();
  const auto t0 = Clock::now();
  const GridMap g = random_maze(n, n, 0.40, 4);
  std::vector<Coord> s, tg;  // free cells on two interleaved lattices
  for (uint32_t r = 181; r < n && s.size() < 64; r += 2897)
    for (uint32_t c = 181; c < n && s.size() < 64; c += 2897)
      for (uint32_t d = 0; d < 64; ++d)
        if (g.is_free({r, c + d})) {
          s.push_back({r, c + d});
          break;
        }
  for (uint32_t r = 97; r < n && tg.size() < 4096; r += 361)
    for (uint32_t c = 53; c < n && tg.size() < 4096; c += 361)
      for (uint32_t d = 0; d < 64; ++d)
        if (c + d < n && g.is_free({r, c + d})) {
          tg.push_back({r, c + d});
          break;
        }
  const SourceSet src(g, s);
  const auto t1 = Clock::now();
  b200::Planner planner(g, src);
  const auto t2 = Clock::now();
  const AutoResult a = planner.propagate_auto(4 * n);
  const auto t3 = Clock::now();
  RunReport rep;
  rep.command = "plan";
  rep.scene = SceneSummary{n, n, g.obstacle_count(), src.size(), tg.size()};
  rep.config.auto_cap = 4 * n;
  rep.layers_used = a.layers_used;
  rep.termination = a.cause == AutoStop::kFilled ? "filled" : a.cause == AutoStop::kStalled ? "stalled" : "cap";
  rep.max_activity = a.layers_used + 1;
  rep.bounds = layer_bound(g);
  rep.paths = planner.target_reports(tg, b200::Method::kEuclidean);  // first call: pool growth, page faults
  const auto t3b = Clock::now();
  rep.paths = planner.target_reports(tg, b200::Method::kEuclidean);
  const auto t4 = Clock::now();
  const std::string json = serialize_run_report(rep);
  const auto t5 = Clock::now();
  const RunReport back = parse_run_report(json);
  const auto t6 = Clock::now();
  size_t pts = 0, covered = 0;
  for (const auto& t : rep.paths) pts += t.points.size(), covered += t.covered;
  std::printf("{\"workload\": \"C4 through the C++ API: 23170^2 random_maze(0.40, seed 4), %zu sources, %zu targets\", "
              "\"layers_used\": %u, \"covered\": %zu, \"points\": %zu, \"json_bytes\": %zu, \"round_trip_equal\": %s, "
              "\"ms\": {\"context_init\": %.1f, \"generate\": %.1f, \"upload\": %.1f, \"propagate_auto\": %.1f, \"target_reports\": %.1f, "
              "\"target_reports_first\": %.1f, \"serialize\": %.1f, \"parse\": %.1f}}\n",
              src.size(), tg.size(), a.layers_used, covered, pts, json.size(), back == rep ? "true" : "false",
              ms(tw0, tw1), ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3b, t4), ms(t3, t3b), ms(t4, t5), ms(t5, t6));
  return back == rep ? 0 : 1;
}
