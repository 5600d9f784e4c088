// Drop-in check of the actmap:: C++ API (include/actmap/*.hpp, same
// signatures as the reference headers) on the device.  Built and run by
// tests/test_cpp_api.py; prints one line per check, exits nonzero on failure.
#include <cmath>
#include <cstdio>
#include <memory>
#include <string>
#include <vector>

#include "actmap/b200.hpp"
#include "actmap/errors.hpp"
#include "actmap/mapio.hpp"
#include "actmap/report.hpp"
#include "actmap/propagate.hpp"
#include "actmap/reconstruct.hpp"

using namespace actmap;

static int failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond);           \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

template <class E, class F>
static bool throws(F f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  // 9x9 empty grid, centre source, L=4 -> corner 1, centre 5, no zeros
  {
    const GridMap g = build_grid(9, 9, {});
    const std::vector<Coord> s{{4, 4}};
    const SourceSet src(g, s);
    const ActivityMap m = propagate(g, src, 4);
    CHECK(m.at(0, 0) == 1 && m.at(4, 4) == 5 && m.zero_free_cells(g) == 0 && m.layers_applied() == 4);
    for (uint32_t r = 0; r < 9; ++r)
      for (uint32_t c = 0; c < 9; ++c) CHECK(m.at(r, c) == 5 - chebyshev({r, c}, {4, 4}));
    const ActivityMap it = propagate(g, src, 4, Mode::kIterative);
    CHECK(it == m);
    CHECK(propagate_reference(g, src, 4) == m);
    // auto -> L_used 4, filled
    const AutoResult a = propagate_auto(g, src, 100);
    CHECK(a.layers_used == 4 && a.cause == AutoStop::kFilled && a.map == m);
    // simple path, any seed -> 4 steps
    for (uint64_t seed : {0ull, 1ull, 7ull}) CHECK(reconstruct_simple(m, g, src, {0, 0}, seed).steps() == 4);
    // propagate_layer from the initial map == propagate(L=1)
    CHECK(propagate_layer(ActivityMap::initial(g, src), g, src) == propagate(g, src, 1));
    CHECK(layer_bound(g).worst_case == 49);
  }
  // Euclidean path (2,2) -> (0,0) is two diagonal moves, length 2*sqrt(2)
  {
    const GridMap g = build_grid(5, 5, {});
    const std::vector<Coord> s{{0, 0}};
    const SourceSet src(g, s);
    const AutoResult a = propagate_auto(g, src, 20);
    const Path p = reconstruct_euclidean(a.map, g, src, {2, 2});
    CHECK(p.points.size() == 3 && p.points[1] == (Coord{1, 1}));
    CHECK(std::fabs(path_metrics(p).euclidean_length - 2 * std::sqrt(2.0)) < 1e-12);
    // reconstruct on a host-built map (uploaded, not device-backed)
    const ActivityMap host(a.map.width(), a.map.height(),
                           std::vector<uint32_t>(a.map.values().begin(), a.map.values().end()), a.layers_used);
    CHECK(reconstruct_euclidean(host, g, src, {2, 2}).points == p.points);
  }
  // errors (errors.hpp; grid.hpp:59-61,78)
  {
    const GridMap g = build_grid(9, 9, std::vector<Coord>{{2, 2}});
    const std::vector<Coord> s{{0, 0}};
    const SourceSet src(g, s);
    const ActivityMap m = propagate(g, src, 1);
    CHECK(throws<UncoveredTargetError>([&] { reconstruct_euclidean(m, g, src, {8, 8}); }));
    CHECK(throws<InvalidInputError>([&] { reconstruct_simple(m, g, src, {2, 2}, 0); }));
    CHECK(throws<InvalidInputError>([&] { reconstruct_simple(m, g, src, {9, 0}, 0); }));
    CHECK(throws<InvalidInputError>([&] { propagate(g, src, 0); }));
    CHECK(throws<InvalidInputError>([&] { propagate_auto(g, src, 0); }));
    CHECK(throws<InvalidInputError>([&] { build_grid(0, 3, {}); }));
    CHECK(throws<InvalidInputError>([&] { build_grid(3, 3, std::vector<Coord>{{3, 0}}); }));
    CHECK(throws<InvalidInputError>([&] { SourceSet(g, std::vector<Coord>{{2, 2}}); }));
    CHECK(throws<InvalidInputError>([&] { SourceSet(g, std::vector<Coord>{}); }));
  }
  // comb maze: auto L_used == BFS eccentricity of the corridor end
  {
    const GridMap g = comb_maze(9, 9);
    const std::vector<Coord> s{{0, 8}};
    const SourceSet src(g, s);
    const AutoResult a = propagate_auto(g, src, 1000);
    CHECK(a.cause == AutoStop::kFilled);
    CHECK(a.map.max_value() == a.layers_used + 1);
  }
  // batched planner on a random maze: every path step-optimal and ends at a source
  {
    const GridMap g = random_maze(600, 400, 0.3, 11);
    std::vector<Coord> s;
    for (uint32_t r = 0; r < 400 && s.size() < 4; r += 97)
      for (uint32_t c = 0; c < 600 && s.size() < 4; c += 131)
        if (g.is_free({r, c})) s.push_back({r, c});
    const SourceSet src(g, s);
    b200::Planner planner(g, src);
    const AutoResult a = planner.propagate_auto(2400);
    std::vector<Coord> targets;
    for (uint32_t r = 5; r < 400; r += 37)
      for (uint32_t c = 3; c < 600; c += 53)
        if (g.is_free({r, c})) targets.push_back({r, c});
    const auto paths = planner.reconstruct_all(targets, b200::Method::kEuclidean);
    int ok = 0;
    for (size_t i = 0; i < paths.size(); ++i) {
      const uint32_t at = a.map.at(targets[i]);
      if (at == 0) {
        CHECK(paths[i].status == b200::TargetStatus::kUncovered);
        continue;
      }
      CHECK(paths[i].status == b200::TargetStatus::kOk);
      CHECK(paths[i].path.steps() == a.layers_used + 1 - at);
      CHECK(src.contains(paths[i].path.source()));
      CHECK(paths[i].path.points == reconstruct_euclidean(a.map, g, src, targets[i]).points);
      ++ok;
    }
    CHECK(ok > 10);
    // RunReport path entries from the same device trace (report.hpp), serialised and read back
    RunReport rep;
    rep.command = "plan";
    rep.scene = SceneSummary{g.width(), g.height(), g.obstacle_count(), src.size(), targets.size()};
    rep.config.auto_cap = 2400;
    rep.layers_used = a.layers_used;
    rep.termination = a.cause == AutoStop::kFilled ? "filled" : a.cause == AutoStop::kStalled ? "stalled" : "cap";
    rep.max_activity = a.layers_used + 1;
    rep.bounds = layer_bound(g);
    rep.paths = planner.target_reports(targets, b200::Method::kEuclidean);
    CHECK(rep.paths.size() == targets.size());
    for (size_t i = 0; i < rep.paths.size(); ++i) {
      const TargetReport& t = rep.paths[i];
      CHECK(t.target == targets[i]);
      CHECK(t.covered == (paths[i].status == b200::TargetStatus::kOk));
      if (!t.covered) continue;
      CHECK(t.points == paths[i].path.points && t.steps + 1 == t.points.size());
      CHECK(t.reached_source && src.contains(*t.reached_source));
      CHECK(t.euclidean_length == path_metrics(paths[i].path).euclidean_length);
    }
    CHECK(parse_run_report(serialize_run_report(rep)) == rep);
    const auto no_pts = planner.target_reports(targets, b200::Method::kEuclidean, 0, false);
    CHECK(no_pts.size() == targets.size() && no_pts[0].points.empty() && no_pts[0].steps == rep.paths[0].steps);
  }
  // a planner's earlier maps keep their values across later propagations (value semantics)
  {
    const GridMap g = build_grid(9, 9, {});
    const std::vector<Coord> s{{4, 4}};
    const SourceSet src(g, s);
    b200::Planner planner(g, src);
    const ActivityMap a = planner.propagate(3);
    const ActivityMap b = planner.propagate(5);
    const AutoResult c = planner.propagate_auto(100);
    CHECK(a.at(4, 4) == 4 && a.layers_applied() == 3);
    CHECK(b.at(4, 4) == 6 && b.layers_applied() == 5);
    CHECK(c.layers_used == 4 && c.map.at(4, 4) == 5 && c.map.at(0, 0) == 1);
    CHECK(a == propagate(g, src, 3) && b == propagate(g, src, 5));
    // a device-backed (not yet downloaded) map fed to propagate_layer: the lazy download must not
    // re-enter the API lock
    const ActivityMap d3 = propagate(g, src, 3);
    CHECK(propagate_layer(d3, g, src) == propagate(g, src, 4));
    const ActivityMap p3 = planner.propagate(3);
    CHECK(propagate_layer(p3, g, src) == b200::Planner(g, src).propagate(4));
  }
  // the planner does not depend on the caller's GridMap after construction (it may die first)
  {
    auto g = std::make_unique<GridMap>(random_maze(64, 48, 0.3, 11));
    const std::vector<Coord> s{{0, 0}, {47, 63}};
    std::vector<Coord> free_s;
    for (Coord c : s)
      if (g->is_free(c)) free_s.push_back(c);
    if (free_s.empty()) free_s.push_back(Coord{1, 1});
    const GridMap copy = *g;
    const SourceSet src(*g, free_s);
    b200::Planner planner(*g, src);
    const SourceSet src_copy(copy, free_s);
    g.reset();  // the planner's grid is gone
    const ActivityMap a = planner.propagate(7);      // shares the planner's device map
    const AutoResult b = planner.propagate_auto(400);  // a is alive: the planner clones its grid on the device
    CHECK(a == propagate(copy, src_copy, 7));
    CHECK(b.map == propagate_auto(copy, src_copy, 400).map);
  }
  // map / scene text (mapio.hpp)
  {
    const GridMap g = parse_movingai("type octile\nheight 2\nwidth 2\nmap\n.@\n@.\n");
    CHECK(g.width() == 2 && g.height() == 2 && g.is_obstacle({0, 1}) && g.is_obstacle({1, 0}) && g.is_free({0, 0}));
    CHECK(emit_movingai(g) == "type octile\nheight 2\nwidth 2\nmap\n.@\n@.\n");
    bool pos = false;
    try {
      parse_movingai("type octile\nheight 3\nwidth 2\nmap\n..\n..\n");
    } catch (const ParseError& e) {
      pos = e.line() == 7 && e.column() == 1;
    }
    CHECK(pos);
    pos = false;
    try {
      parse_movingai("type octile\nheight 2\nwidth 2\nmap\n.@\n@x\n");
    } catch (const ParseError& e) {
      pos = e.line() == 6 && e.column() == 2;
    }
    CHECK(pos);
    const Scene sc = parse_ascii_scene("S.\n.T\n");
    CHECK(sc.grid.width() == 2 && sc.sources.size() == 1 && sc.sources.coords()[0] == (Coord{0, 0}));
    CHECK(sc.targets.size() == 1 && sc.targets[0] == (Coord{1, 1}));
    CHECK(emit_ascii_scene(sc) == "S.\n.T\n");
    const Scene dis = parse_ascii_scene("S#\n#T");
    CHECK(dis.grid.is_obstacle({0, 1}) && dis.grid.is_obstacle({1, 0}) && dis.targets.size() == 1);

    CHECK(throws<ParseError>([&] { parse_ascii_scene("S.\n.T.\n"); }));
    CHECK(throws<InvalidInputError>([&] { parse_ascii_scene("..\n.T\n"); }));
    const std::string p1 = export_pgm(ActivityMap(1, 1, std::vector<uint32_t>{2}, 1));
    CHECK(p1 == std::string("P5\n1 1\n255\n\xff", 12));
    const std::string p0 = export_pgm(ActivityMap(2, 1, std::vector<uint32_t>{0, 0}, 1));
    CHECK(p0 == std::string("P5\n2 1\n255\n\0\0", 13));
    // device-resident map: same bytes as the host-map path
    const GridMap e = build_grid(9, 9, {});
    const std::vector<Coord> cs{{4, 4}};
    const SourceSet src(e, cs);
    const ActivityMap m = propagate(e, src, 300);
    const ActivityMap host(9, 9, std::vector<uint32_t>(m.values().begin(), m.values().end()), 300);
    const std::string pd = export_pgm(m), ph = export_pgm(host);
    CHECK(pd == ph && pd.size() == std::string("P5\n9 9\n65535\n").size() + 162);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
