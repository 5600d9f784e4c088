// Test driver for tests/test_gpu_reports.py: runs the drop-in planner session
// (actmap::b200::Planner, include/actmap/b200.hpp) on a grid given as raw
// files and prints the RunReport (report.hpp:35-42,85-102) with every
// target's entry, so the Python test can compare each entry with the CPU
// oracle's reconstruct_* + path_metrics on the same grid.
//
//   planner_reports W H occ.u8 src.u32 tgt.u32 method(0 simple|1 euclidean) seed auto_cap
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "actmap/b200.hpp"
#include "actmap/propagate.hpp"
#include "actmap/report.hpp"

using namespace actmap;

template <class T>
static std::vector<T> slurp(const char* path) {
  std::ifstream f(path, std::ios::binary);
  std::vector<char> b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  std::vector<T> v(b.size() / sizeof(T));
  std::memcpy(v.data(), b.data(), v.size() * sizeof(T));
  return v;
}

static std::vector<Coord> coords(const std::vector<uint32_t>& rc) {
  std::vector<Coord> c(rc.size() / 2);
  for (size_t i = 0; i < c.size(); ++i) c[i] = Coord{rc[2 * i], rc[2 * i + 1]};
  return c;
}

int main(int argc, char** argv) {
  if (argc != 9) {
    std::fprintf(stderr, "usage: %s W H occ src tgt method seed auto_cap\n", argv[0]);
    return 2;
  }
  const uint32_t W = std::stoul(argv[1]), H = std::stoul(argv[2]);
  const GridMap g(W, H, slurp<uint8_t>(argv[3]));
  const auto src = coords(slurp<uint32_t>(argv[4]));
  const auto tgt = coords(slurp<uint32_t>(argv[5]));
  const auto method = std::stoi(argv[6]) ? b200::Method::kEuclidean : b200::Method::kSimple;
  const uint64_t seed = std::stoull(argv[7]);
  const uint32_t cap = std::stoul(argv[8]);
  const SourceSet ss(g, src);
  b200::Planner planner(g, ss);
  const AutoResult a = planner.propagate_auto(cap);
  RunReport rep;
  rep.command = "plan";
  rep.scene = SceneSummary{W, H, g.obstacle_count(), ss.size(), tgt.size()};
  rep.config.auto_cap = cap;
  rep.config.method = method == b200::Method::kEuclidean ? Method::kEuclidean : Method::kSimple;
  rep.config.seed = seed;
  rep.layers_used = a.layers_used;
  rep.termination = a.cause == AutoStop::kFilled ? "filled" : a.cause == AutoStop::kStalled ? "stalled" : "cap";
  rep.max_activity = a.layers_used + 1;
  rep.bounds = layer_bound(g);
  rep.paths = planner.target_reports(tgt, method, seed);
  const std::string j = serialize_run_report(rep);
  if (!(parse_run_report(j) == rep)) {
    std::fprintf(stderr, "report does not round-trip\n");
    return 1;
  }
  std::fwrite(j.data(), 1, j.size(), stdout);
  return 0;
}
