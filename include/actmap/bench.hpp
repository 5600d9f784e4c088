// actmap/bench.hpp -- benchmark records carried by RunReport (reference bench.hpp:12-52).
//
// Same record types as the reference.  The reference's own benchmark driver
// (run_benchmark / fit_scaling, bench.hpp:36-52) is outside this tier's scope
// (DESIGN.md §9); this repository's measurement is bench.py.
#pragma once

#include <cstdint>
#include <optional>

#include "actmap/propagate.hpp"

namespace actmap {

struct BenchSample {
  std::uint32_t n = 0;       // linear grid size (n x n cells)
  std::uint32_t layers = 0;  // L
  Mode mode = Mode::kBatched;
  unsigned threads = 1;
  std::uint32_t repeats = 0;
  double median_ms = 0.0;
  double min_ms = 0.0;
  bool skipped = false;  // allocation failure at this size

  friend bool operator==(const BenchSample&, const BenchSample&) = default;
};

/// Layer count per grid size: a fixed L, or ratio * n.
struct LayerRule {
  std::optional<std::uint32_t> fixed;
  double ratio = 1.0;
  std::uint32_t layers_for(std::uint32_t n) const;
};

struct ScalingFit {
  std::optional<double> slope_vs_nodes;   // ms per cell at the common L
  std::optional<double> slope_vs_layers;  // ms per layer at the common n
  double coefficient = 0.0;               // c in t = c * L * n^2
  double max_rel_residual = 0.0;

  friend bool operator==(const ScalingFit&, const ScalingFit&) = default;
};

}  // namespace actmap
