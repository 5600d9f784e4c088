// actmap/b200.hpp -- batched planner surface (new; SURVEY.md §8b notes the
// reference has no batched-target API).  A Planner keeps the grid, sources
// and activity map resident in HBM across calls, so a multi-target plan is
// one propagation plus one batched trace with no map round trip.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "actmap/propagate.hpp"
#include "actmap/reconstruct.hpp"
#include "actmap/report.hpp"

namespace actmap::b200 {

struct DeviceOptions {
  int device = 0;
  bool timing = false;  // CUDA-event time every stencil block launch
};

enum class Method { kSimple, kEuclidean };  // report.hpp:15

enum class TargetStatus { kOk = 0, kInvalid = 1, kUncovered = 2, kInternal = 6 };

struct PlannedPath {
  Coord target;
  TargetStatus status = TargetStatus::kOk;
  Path path;  // empty unless status == kOk
};

struct PropagationStats {
  std::uint32_t layers_computed = 0;  // device layers incl. exactly-rolled-back overshoot
  std::uint32_t cell_bits = 16;
  std::uint64_t block_launches = 0;
  std::uint64_t layer_launches = 0;
  double stencil_ms = 0.0;
};

class Planner {
 public:
  Planner(const GridMap& grid, const SourceSet& sources, DeviceOptions options = {});
  ~Planner();
  Planner(const Planner&) = delete;
  Planner& operator=(const Planner&) = delete;

  /// propagate_auto on the resident grid; the returned map downloads lazily.
  AutoResult propagate_auto(std::uint32_t auto_cap);
  /// propagate on the resident grid.
  ActivityMap propagate(std::uint32_t layers, Mode mode = Mode::kBatched);
  /// Batched path extraction over the last propagated map; uncovered or
  /// invalid targets are reported per target, not thrown.
  std::vector<PlannedPath> reconstruct_all(std::span<const Coord> targets, Method method, std::uint64_t seed = 0,
                                           CornerRule rule = CornerRule::kStrict);
  /// RunReport path entries (report.hpp TargetReport) for a target batch from one batched
  /// device trace: covered, reached source, steps, Euclidean length and (emit_points) the
  /// points; throws InvalidInputError for a target out of bounds or on an obstacle.
  std::vector<TargetReport> target_reports(std::span<const Coord> targets, Method method, std::uint64_t seed = 0,
                                           bool emit_points = true, CornerRule rule = CornerRule::kStrict);
  const PropagationStats& last_stats() const noexcept { return stats_; }

 private:
  std::shared_ptr<void> impl_;
  PropagationStats stats_;
};

}  // namespace actmap::b200
