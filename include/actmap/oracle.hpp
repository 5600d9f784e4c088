// actmap/oracle.hpp -- the oracle result type carried by reports (reference oracle.hpp:89-94).
//
// The reference's CPU oracles themselves (BFS, octile Dijkstra, check_activity,
// oracle.hpp:73-98) are test infrastructure here: they live in oracle/ and are
// used only by tests/ and bench.py's CPU baseline, never by the product path.
#pragma once

#include <cstdint>
#include <vector>

#include "actmap/coord.hpp"

namespace actmap {

/// Outcome of the activity-law check: violation count plus the
/// first few offending cells.
struct ActivityCheck {
  std::uint64_t violations = 0;
  std::vector<Coord> samples;

  bool ok() const noexcept { return violations == 0; }

  friend bool operator==(const ActivityCheck&, const ActivityCheck&) = default;
};

}  // namespace actmap
