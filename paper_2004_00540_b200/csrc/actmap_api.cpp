// actmap_api.cpp -- the reference's actmap:: planner API (include/actmap/*.hpp)
// implemented over the C ABI (include/actmap_b200.h).  Compute always runs
// on the device; this file only validates inputs, maps status codes to the
// reference exception types (errors.hpp) and does O(path) host
// post-processing (straighten, metrics).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "actmap/b200.hpp"
#include "actmap/errors.hpp"
#include "actmap/mapio.hpp"
#include "actmap/propagate.hpp"
#include "actmap/reconstruct.hpp"
#include "actmap_b200.h"

namespace actmap {

namespace {

std::mutex& api_mutex() {
  static std::mutex m;
  return m;
}

am_ctx* default_ctx() {
  static am_ctx* ctx = nullptr;
  static std::once_flag once;
  static am_status st = AM_OK;
  std::call_once(once, [] {
    am_ctx_opts o{};
    const char* env = std::getenv("ACTMAP_DEVICE");
    o.device = env ? std::atoi(env) : 0;
    st = am_ctx_create(&o, &ctx);
  });
  if (st != AM_OK || !ctx) throw Error("actmap: cannot create the B200 device context (status " + std::to_string(st) + ")");
  return ctx;
}

[[noreturn]] void throw_status(am_status st, am_ctx* ctx, const std::string& what) {
  const std::string msg = what + ": " + (ctx ? am_last_error(ctx) : "");
  if (st == AM_EINVAL) throw InvalidInputError(msg);
  if (st == AM_EUNCOVERED) throw UncoveredTargetError(msg);
  throw Error(msg);
}

void check(am_status st, am_ctx* ctx, const char* what) {
  if (st != AM_OK) throw_status(st, ctx, what);
}

uint64_t splitmix64(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t bounded(uint64_t u, uint64_t n) { return (uint64_t)(((unsigned __int128)u * n) >> 64); }

uint64_t chunk_hash(const uint8_t* p, size_t n, uint64_t seed) {
  // four independent multiply chains (32 bytes per round) so the multiplier latency overlaps
  uint64_t h[4] = {0x243F6A8885A308D3ull ^ seed, 0x13198A2E03707344ull ^ seed, 0xA4093822299F31D0ull ^ seed,
                   0x082EFA98EC4E6C89ull ^ seed};
  size_t i = 0;
  for (; i + 32 <= n; i += 32)
    for (int k = 0; k < 4; ++k) {
      uint64_t w;
      std::memcpy(&w, p + i + 8 * k, 8);
      h[k] = (h[k] ^ w) * 0x9E3779B97F4A7C15ull;
      h[k] ^= h[k] >> 29;
    }
  uint64_t r = h[0] ^ (h[1] * 0xBF58476D1CE4E5B9ull) ^ (h[2] * 0x94D049BB133111EBull) ^ (h[3] * 0x9E3779B97F4A7C15ull);
  for (; i < n; ++i) r = (r ^ p[i]) * 0x100000001B3ull;
  return r;
}

// identity of a GridMap's contents (DeviceMap::matches): 32 MiB chunks hashed on up to 16 threads, combined
// in chunk order
uint64_t occupancy_hash(std::span<const uint8_t> occ) {
  constexpr size_t kChunk = size_t(32) << 20;
  const size_t nchunks = (occ.size() + kChunk - 1) / kChunk;
  std::vector<uint64_t> part(nchunks);
  auto work = [&](size_t first, size_t step) {
    for (size_t c = first; c < nchunks; c += step)
      part[c] = chunk_hash(occ.data() + c * kChunk, std::min(kChunk, occ.size() - c * kChunk), c);
  };
  const unsigned hw = std::thread::hardware_concurrency();
  const size_t nt = std::min<size_t>(nchunks, std::min<unsigned>(hw ? hw : 1, 16));
  std::vector<std::thread> pool;
  for (size_t t = 1; t < nt; ++t) pool.emplace_back(work, t, nt);
  work(0, nt ? nt : 1);
  for (auto& th : pool) th.join();
  uint64_t h = 0x9E3779B97F4A7C15ull ^ occ.size();
  for (uint64_t v : part) h = (h ^ v) * 0xBF58476D1CE4E5B9ull, h ^= h >> 31;
  return h;
}

// f(i) for i in [0, n) on up to 16 host threads (grain: 16 consecutive indices per fetch); small n inline
template <class F>
void parallel_for(size_t n, F&& f) {
  const unsigned hw = std::thread::hardware_concurrency();
  const unsigned nt = std::min<unsigned>(hw ? hw : 1, 16);
  if (n < 256 || nt <= 1) {
    for (size_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (size_t i; (i = next.fetch_add(16)) < n;)
      for (size_t j = i; j < std::min(n, i + 16); ++j) f(j);
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
}

std::vector<uint32_t> flatten(const std::vector<Coord>& cs) {
  std::vector<uint32_t> rc(cs.size() * 2);
  for (size_t i = 0; i < cs.size(); ++i) {
    rc[2 * i] = cs[i].row;
    rc[2 * i + 1] = cs[i].col;
  }
  return rc;
}

}  // namespace

namespace detail {

// A grid + sources + activity map resident on the device.
struct DeviceMap {
  am_ctx* ctx = nullptr;
  am_grid* grid = nullptr;
  uint32_t width = 0, height = 0;
  const uint8_t* occ_ptr = nullptr;
  uint64_t obstacles = 0, occ_hash = 0;
  std::vector<Coord> sources;
  uint32_t layers = 0;

  DeviceMap(const GridMap& g, const SourceSet& s) {
    ctx = default_ctx();
    width = g.width();
    height = g.height();
    occ_ptr = g.occupancy().data();
    obstacles = g.obstacle_count();
    occ_hash = occupancy_hash(g.occupancy());
    sources = s.coords();
    const auto rc = flatten(sources);
    check(am_grid_create(ctx, width, height, g.occupancy().data(), rc.data(), sources.size(), &grid), ctx,
          "grid upload");
  }
  // same grid and sources, built on the device from `from`'s resident copies (no host GridMap needed)
  explicit DeviceMap(const DeviceMap& from)
      : ctx(from.ctx), width(from.width), height(from.height), occ_ptr(from.occ_ptr), obstacles(from.obstacles),
        occ_hash(from.occ_hash), sources(from.sources) {
    check(am_grid_clone(ctx, from.grid, &grid), ctx, "grid clone");
  }
  DeviceMap& operator=(const DeviceMap&) = delete;
  ~DeviceMap() {
    if (grid) am_grid_destroy(ctx, grid);
    if (pts) am_host_free(ctx, pts);
  }
  // pinned trace buffer (am_host_alloc): the walkers write the points into it directly
  uint32_t* pts = nullptr;
  size_t pts_words = 0;
  uint32_t* trace_buffer(size_t words) {
    if (words > pts_words) {
      if (pts) am_host_free(ctx, pts);
      pts = nullptr;
      pts_words = 0;
      void* p = nullptr;
      const size_t want = words + words / 4;
      check(am_host_alloc(ctx, want * 4, &p), ctx, "trace buffer");
      pts = static_cast<uint32_t*>(p);
      pts_words = want;
    }
    return pts;
  }
  bool matches(const GridMap& g, const SourceSet& s) const {
    if (g.width() != width || g.height() != height || g.obstacle_count() != obstacles) return false;
    if (s.coords() != sources) return false;
    return g.occupancy().data() == occ_ptr || occupancy_hash(g.occupancy()) == occ_hash;
  }
};

struct LazyValues {
  std::once_flag once;
  std::vector<uint32_t> v;
};

}  // namespace detail

// ------------------------------------------------------------------ grid

GridMap::GridMap(uint32_t width, uint32_t height, std::vector<uint8_t> occupancy)
    : width_(width), height_(height), obstacle_count_(0), occupancy_(std::move(occupancy)) {
  if (width == 0 || height == 0 || width > kMaxGridDim || height > kMaxGridDim)
    throw InvalidInputError("grid dimensions must be 1.." + std::to_string(kMaxGridDim));
  if (occupancy_.size() != static_cast<size_t>(width) * height)
    throw InvalidInputError("occupancy size does not match width*height");
  for (uint8_t o : occupancy_) obstacle_count_ += o != 0;
}

GridMap build_grid(uint32_t width, uint32_t height, std::span<const Coord> obstacles) {
  if (width == 0 || height == 0) throw InvalidInputError("build_grid: zero dimension");
  if (width > kMaxGridDim || height > kMaxGridDim) throw InvalidInputError("build_grid: dimension above kMaxGridDim");
  std::vector<uint8_t> occ(static_cast<size_t>(width) * height, 0);
  for (Coord c : obstacles) {
    if (c.row >= height || c.col >= width) throw InvalidInputError("build_grid: obstacle out of bounds " + to_string(c));
    occ[static_cast<size_t>(c.row) * width + c.col] = 1;
  }
  return GridMap(width, height, std::move(occ));
}

GridMap comb_maze(uint32_t width, uint32_t height) {
  if (width < 2 || height < 2) throw InvalidInputError("comb_maze: dimensions must be >= 2");
  if (width > kMaxGridDim || height > kMaxGridDim) throw InvalidInputError("comb_maze: dimension above kMaxGridDim");
  std::vector<uint8_t> occ(static_cast<size_t>(width) * height, 0);
  if (width >= height) {  // odd rows are walls; gaps alternate col 0 / col width-1
    for (uint32_t r = 1, k = 0; r < height; r += 2, ++k) {
      std::fill_n(occ.begin() + static_cast<size_t>(r) * width, width, 1);
      occ[static_cast<size_t>(r) * width + (k % 2 ? width - 1 : 0)] = 0;
    }
  } else {  // odd columns are walls; gaps alternate row 0 / row height-1
    for (uint32_t c = 1, k = 0; c < width; c += 2, ++k) {
      for (uint32_t r = 0; r < height; ++r) occ[static_cast<size_t>(r) * width + c] = 1;
      occ[static_cast<size_t>(k % 2 ? height - 1 : 0) * width + c] = 0;
    }
  }
  return GridMap(width, height, std::move(occ));
}

GridMap random_maze(uint32_t width, uint32_t height, double density, uint64_t seed) {
  if (width == 0 || height == 0 || width > kMaxGridDim || height > kMaxGridDim)
    throw InvalidInputError("random_maze: bad dimensions");
  if (!(density >= 0.0) || !(density < 1.0)) throw InvalidInputError("random_maze: density must be in [0,1)");
  const uint64_t n = static_cast<uint64_t>(width) * height;
  uint64_t m = static_cast<uint64_t>(std::llround(density * static_cast<double>(n)));
  if (m > n) m = n;
  std::vector<uint8_t> occ(n);
  uint64_t st = seed, chosen = 0;
  for (uint64_t i = 0; i < n; ++i) {  // selection sampling: uniform m-subset
    const uint64_t left = n - i, need = m - chosen;
    const uint8_t ob = need && (need == left || bounded(splitmix64(st), left) < need);
    occ[i] = ob;
    chosen += ob;
  }
  return GridMap(width, height, std::move(occ));
}

// Workload generators of the benchmark configurations.  C2:
// perfect maze on the odd lattice (corridor cells at odd (r, c), 1-cell
// walls) by randomised Kruskal: the lattice edges (right / down of each
// corridor cell) in a splitmix64 Fisher-Yates order, a wall cell opened when
// its edge joins two components.
GridMap kruskal_maze(uint32_t width, uint32_t height, uint64_t seed) {
  if (width < 3 || height < 3 || width > kMaxGridDim || height > kMaxGridDim)
    throw InvalidInputError("kruskal_maze: bad dimensions");
  std::vector<uint8_t> occ(static_cast<size_t>(width) * height, 1);
  const uint32_t cw = (width - 1) / 2, ch = (height - 1) / 2;
  const uint64_t cells = static_cast<uint64_t>(cw) * ch;
  for (uint32_t i = 0; i < ch; ++i)
    for (uint32_t j = 0; j < cw; ++j) occ[static_cast<size_t>(2 * i + 1) * width + 2 * j + 1] = 0;
  std::vector<uint64_t> edges;  // 2 * cell + (0 right, 1 down)
  edges.reserve(2 * cells);
  for (uint64_t c = 0; c < cells; ++c) {
    if (c % cw + 1 < cw) edges.push_back(2 * c);
    if (c / cw + 1 < ch) edges.push_back(2 * c + 1);
  }
  uint64_t st = seed;
  for (uint64_t i = edges.size(); i > 1; --i) std::swap(edges[i - 1], edges[bounded(splitmix64(st), i)]);
  std::vector<uint32_t> parent(cells);
  for (uint64_t c = 0; c < cells; ++c) parent[c] = static_cast<uint32_t>(c);
  auto root = [&](uint32_t x) {
    while (parent[x] != x) x = parent[x] = parent[parent[x]];
    return x;
  };
  for (uint64_t e : edges) {
    const uint64_t c = e >> 1;
    const bool down = e & 1;
    const uint32_t a = root(static_cast<uint32_t>(c)), b = root(static_cast<uint32_t>(down ? c + cw : c + 1));
    if (a == b) continue;
    parent[a] = b;
    const uint32_t i = static_cast<uint32_t>(c / cw), j = static_cast<uint32_t>(c % cw);
    occ[static_cast<size_t>(2 * i + 1 + (down ? 1 : 0)) * width + 2 * j + 1 + (down ? 0 : 1)] = 0;
  }
  return GridMap(width, height, std::move(occ));
}

// C3: city blocks of side U[32,96] separated by streets of width U[3,8]
// along both axes; 10% of the blocks are left free as plazas (per-block
// hash), and 1% single-cell clutter (per-cell hash) everywhere else.
GridMap city_grid(uint32_t width, uint32_t height, uint64_t seed) {
  if (width == 0 || height == 0 || width > kMaxGridDim || height > kMaxGridDim)
    throw InvalidInputError("city_grid: bad dimensions");
  uint64_t st = seed;
  auto bands = [&](uint32_t n, std::vector<int64_t>& id) {  // block index per row / column, -1 = street
    id.assign(n, -1);
    uint32_t pos = static_cast<uint32_t>(3 + bounded(splitmix64(st), 6)), k = 0;
    while (pos < n) {
      const uint32_t b = static_cast<uint32_t>(32 + bounded(splitmix64(st), 65));
      for (uint32_t x = pos; x < pos + b && x < n; ++x) id[x] = k;
      ++k;
      pos += b + static_cast<uint32_t>(3 + bounded(splitmix64(st), 6));
    }
    return k;
  };
  std::vector<int64_t> rid, cid;
  bands(height, rid);
  const uint32_t ncb = bands(width, cid);
  const uint64_t plaza = splitmix64(st), clutter = splitmix64(st);
  std::vector<uint8_t> occ(static_cast<size_t>(width) * height);
  for (uint32_t r = 0; r < height; ++r)
    for (uint32_t c = 0; c < width; ++c) {
      const uint64_t idx = static_cast<uint64_t>(r) * width + c;
      uint8_t ob = 0;
      if (rid[r] >= 0 && cid[c] >= 0) {
        uint64_t s = plaza ^ (static_cast<uint64_t>(rid[r]) * ncb + static_cast<uint64_t>(cid[c])) * 0xD1B54A32D192ED03ull;
        ob = bounded(splitmix64(s), 100) >= 10;
      }
      if (!ob) {
        uint64_t s = clutter ^ idx * 0x9E3779B97F4A7C15ull;
        ob = bounded(splitmix64(s), 100) < 1;
      }
      occ[idx] = ob;
    }
  return GridMap(width, height, std::move(occ));
}

SourceSet::SourceSet(const GridMap& grid, std::span<const Coord> sources) {
  if (sources.empty()) throw InvalidInputError("SourceSet: at least one source is required");
  coords_.assign(sources.begin(), sources.end());
  for (Coord c : coords_) {
    if (!grid.in_bounds(c)) throw InvalidInputError("SourceSet: source out of bounds " + to_string(c));
    if (grid.is_obstacle(c)) throw InvalidInputError("SourceSet: source on an obstacle " + to_string(c));
  }
  std::sort(coords_.begin(), coords_.end());
  coords_.erase(std::unique(coords_.begin(), coords_.end()), coords_.end());
}

bool SourceSet::contains(Coord c) const noexcept { return std::binary_search(coords_.begin(), coords_.end(), c); }

// -------------------------------------------------------------- activity

ActivityMap::ActivityMap(uint32_t width, uint32_t height, std::vector<uint32_t> values, uint32_t layers_applied)
    : width_(width), height_(height), layers_applied_(layers_applied),
      values_(std::make_shared<detail::LazyValues>()) {
  if (values.size() != static_cast<size_t>(width) * height)
    throw InvalidInputError("ActivityMap: values size does not match width*height");
  std::call_once(values_->once, [&] { values_->v = std::move(values); });
}

ActivityMap::ActivityMap(uint32_t width, uint32_t height, uint32_t layers_applied,
                         std::shared_ptr<detail::DeviceMap> device)
    : width_(width), height_(height), layers_applied_(layers_applied),
      values_(std::make_shared<detail::LazyValues>()), device_(std::move(device)) {}

std::span<const uint32_t> ActivityMap::values() const noexcept {
  std::call_once(values_->once, [&] {
    if (!device_) return;
    std::lock_guard<std::mutex> lk(api_mutex());
    values_->v.resize(static_cast<size_t>(width_) * height_);
    check(am_activity_download(device_->ctx, device_->grid, values_->v.data()), device_->ctx, "activity download");
  });
  return values_->v;
}

ActivityMap ActivityMap::initial(const GridMap& grid, const SourceSet& sources) {
  std::vector<uint32_t> v(grid.cell_count(), 0);
  for (Coord c : sources.coords()) v[grid.index(c)] = 1;
  return ActivityMap(grid.width(), grid.height(), std::move(v), 0);
}

uint32_t ActivityMap::max_value() const noexcept {
  uint32_t m = 0;
  for (uint32_t v : values()) m = std::max(m, v);
  return m;
}

uint64_t ActivityMap::zero_free_cells(const GridMap& grid) const {
  if (grid.width() != width_ || grid.height() != height_) throw InvalidInputError("zero_free_cells: dimension mismatch");
  const auto v = values();
  const auto occ = grid.occupancy();
  uint64_t z = 0;
  for (size_t i = 0; i < v.size(); ++i) z += (occ[i] == 0 && v[i] == 0);
  return z;
}

// ------------------------------------------------------------ propagation

ActivityMap propagate_layer(const ActivityMap& activity, const GridMap& grid, const SourceSet& sources, unsigned) {
  if (activity.width() != grid.width() || activity.height() != grid.height())
    throw InvalidInputError("propagate_layer: activity/grid dimension mismatch");
  const auto in = activity.values();  // before taking the API lock (a lazy download takes it)
  std::lock_guard<std::mutex> lk(api_mutex());
  am_ctx* ctx = default_ctx();
  const auto rc = flatten(sources.coords());
  std::vector<uint32_t> out(grid.cell_count());
  check(am_propagate_layer(ctx, grid.width(), grid.height(), grid.occupancy().data(), rc.data(), sources.size(),
                           in.data(), out.data()),
        ctx, "propagate_layer");
  return ActivityMap(grid.width(), grid.height(), std::move(out), activity.layers_applied() + 1);
}

ActivityMap propagate(const GridMap& grid, const SourceSet& sources, uint32_t layers, Mode mode, unsigned) {
  if (layers == 0) throw InvalidInputError("propagate: L must be >= 1");
  if (layers > kMaxLayers) throw InvalidInputError("propagate: L exceeds kMaxLayers");
  std::lock_guard<std::mutex> lk(api_mutex());
  auto dev = std::make_shared<detail::DeviceMap>(grid, sources);
  am_prop_result r{};
  check(am_propagate(dev->ctx, dev->grid, layers, 0, mode == Mode::kBatched ? AM_MODE_BATCHED : AM_MODE_ITERATIVE, &r),
        dev->ctx, "propagate");
  dev->layers = layers;
  return ActivityMap(grid.width(), grid.height(), layers, std::move(dev));
}

AutoResult propagate_auto(const GridMap& grid, const SourceSet& sources, uint32_t auto_cap, unsigned) {
  if (auto_cap == 0) throw InvalidInputError("propagate_auto: auto_cap must be >= 1");
  if (auto_cap > kMaxLayers) throw InvalidInputError("propagate_auto: auto_cap exceeds kMaxLayers");
  std::lock_guard<std::mutex> lk(api_mutex());
  auto dev = std::make_shared<detail::DeviceMap>(grid, sources);
  am_prop_result r{};
  check(am_propagate(dev->ctx, dev->grid, 0, auto_cap, AM_MODE_BATCHED, &r), dev->ctx, "propagate_auto");
  dev->layers = r.layers_used;
  const AutoStop cause = r.cause == AM_STOP_FILLED ? AutoStop::kFilled
                         : r.cause == AM_STOP_STALLED ? AutoStop::kStalled
                                                      : AutoStop::kCapReached;
  return AutoResult{ActivityMap(grid.width(), grid.height(), r.layers_used, std::move(dev)), r.layers_used, cause};
}

ActivityMap propagate_reference(const GridMap& grid, const SourceSet& sources, uint32_t layers) {
  if (layers == 0 || layers > kMaxLayers) throw InvalidInputError("propagate_reference: L out of range");
  std::lock_guard<std::mutex> lk(api_mutex());
  am_ctx* ctx = default_ctx();
  const auto rc = flatten(sources.coords());
  std::vector<uint32_t> out(grid.cell_count());
  check(am_propagate_reference(ctx, grid.width(), grid.height(), grid.occupancy().data(), rc.data(), sources.size(),
                               layers, out.data()),
        ctx, "propagate_reference");
  return ActivityMap(grid.width(), grid.height(), std::move(out), layers);
}

LayerBound layer_bound(const GridMap& grid) {
  const uint64_t mx = std::max(grid.width(), grid.height()), mn = std::min(grid.width(), grid.height());
  return LayerBound{mx * ((mn + 1) / 2) + mn / 2, static_cast<uint32_t>((3 * mx + 1) / 2),
                    static_cast<uint32_t>(2 * mx)};
}

// ---------------------------------------------------------------- paths

namespace {

std::vector<Path> trace_batch(detail::DeviceMap& dev, std::span<const Coord> targets, uint32_t method, uint64_t seed,
                              std::vector<int32_t>& status) {
  const size_t n = targets.size();
  std::vector<uint32_t> rc(2 * n);
  for (size_t i = 0; i < n; ++i) {
    rc[2 * i] = targets[i].row;
    rc[2 * i + 1] = targets[i].col;
  }
  std::vector<uint64_t> off(n + 1, 0);
  status.assign(n, 0);
  check(am_path_counts(dev.ctx, dev.grid, rc.data(), n, method, seed, off.data(), status.data()), dev.ctx,
        "path counts");
  const uint32_t* pts = dev.trace_buffer(2 * off[n] + 2);  // pinned: the walkers stream the points into it
  check(am_trace_paths(dev.ctx, dev.grid, rc.data(), n, method, seed, off.data(), dev.pts, off[n], status.data()),
        dev.ctx, "trace paths");
  std::vector<Path> paths(n);
  parallel_for(n, [&](size_t i) {
    if (status[i] != AM_OK) return;
    uint64_t end = off[i];  // points removed by device-side straightening of uploaded maps end a path
    while (end < off[i + 1] && pts[2 * end] != 0xFFFFFFFFu) ++end;
    static_assert(sizeof(Coord) == 8, "Coord is {row, col}: the (row, col) pairs are Coord arrays");
    const Coord* first = reinterpret_cast<const Coord*>(pts + 2 * off[i]);
    paths[i].points.assign(first, first + (end - off[i]));
  });
  return paths;
}

Path reconstruct_one(const ActivityMap& activity, const GridMap& grid, const SourceSet& sources, Coord target,
                     uint32_t method, uint64_t seed) {
  if (activity.width() != grid.width() || activity.height() != grid.height())
    throw InvalidInputError("reconstruct: activity/grid dimension mismatch");
  if (!grid.in_bounds(target)) throw InvalidInputError("reconstruct: target out of bounds " + to_string(target));
  if (grid.is_obstacle(target)) throw InvalidInputError("reconstruct: target on an obstacle " + to_string(target));
  std::shared_ptr<detail::DeviceMap> dev = activity.device_map();
  if (!dev || !dev->matches(grid, sources)) {
    const auto vals = activity.values();  // before taking the API lock (lazy download locks it)
    std::lock_guard<std::mutex> lk(api_mutex());
    dev = std::make_shared<detail::DeviceMap>(grid, sources);
    check(am_activity_upload(dev->ctx, dev->grid, vals.data(), activity.layers_applied()), dev->ctx,
          "activity upload");
  }
  std::lock_guard<std::mutex> lk(api_mutex());
  std::vector<int32_t> st;
  auto paths = trace_batch(*dev, std::span<const Coord>(&target, 1), method, seed, st);
  if (st[0] == AM_EUNCOVERED)
    throw UncoveredTargetError("uncovered target " + to_string(target) + ": increase L or target unreachable");
  if (st[0] == AM_EINVAL) throw InvalidInputError("reconstruct: invalid target " + to_string(target));
  if (st[0] != AM_OK) throw Error("reconstruct: activity map has no ascending neighbour on the path");
  return std::move(paths[0]);
}

bool removable(const std::vector<Coord>& p, size_t m, const GridMap* grid, CornerRule rule) {
  const Coord a = p[m - 3], b = p[m - 1];
  const int64_t dr = (int64_t)a.row - b.row, dc = (int64_t)a.col - b.col;
  if (dr * dr + dc * dc != 2) return false;
  if (grid && rule == CornerRule::kStrict && grid->is_obstacle(a.row, b.col) && grid->is_obstacle(b.row, a.col))
    return false;
  return true;
}

Path straighten_impl(const Path& path, const GridMap* grid, CornerRule rule) {
  if (path.points.size() < 3) return path;
  std::vector<Coord> out;
  out.reserve(path.points.size());
  for (const Coord& c : path.points) {  // pin P4 as a single stack pass
    out.push_back(c);
    while (out.size() >= 3 && removable(out, out.size(), grid, rule)) out.erase(out.end() - 2);
  }
  return Path{std::move(out)};
}

}  // namespace

Path reconstruct_simple(const ActivityMap& activity, const GridMap& grid, const SourceSet& sources, Coord target,
                        uint64_t seed) {
  return reconstruct_one(activity, grid, sources, target, AM_METHOD_SIMPLE, seed);
}

Path reconstruct_euclidean(const ActivityMap& activity, const GridMap& grid, const SourceSet& sources, Coord target,
                           CornerRule rule) {
  return straighten(reconstruct_one(activity, grid, sources, target, AM_METHOD_EUCLIDEAN, 0), grid, rule);
}

Path straighten(const Path& path) { return straighten_impl(path, nullptr, CornerRule::kPermissive); }

Path straighten(const Path& path, const GridMap& grid, CornerRule rule) { return straighten_impl(path, &grid, rule); }

PathMetrics path_metrics(const Path& path) {
  PathMetrics m;
  const auto& p = path.points;
  m.steps = p.empty() ? 0 : p.size() - 1;
  uint64_t ax = 0, dg = 0;
  double other = 0.0;
  for (size_t i = 1; i < p.size(); ++i) {
    const int64_t dr = (int64_t)p[i].row - p[i - 1].row, dc = (int64_t)p[i].col - p[i - 1].col;
    const int64_t q = dr * dr + dc * dc;
    if (q == 1) ++ax;
    else if (q == 2) ++dg;
    else other += std::sqrt((double)q);
  }
  m.euclidean_length = (double)ax + (double)dg * 1.4142135623730951 + other;
  return m;
}

// ---------------------------------------------------------------- b200

namespace b200 {

struct PlannerImpl {
  std::shared_ptr<detail::DeviceMap> dev;
  uint32_t width, height;
  // A map returned earlier still refers to `dev` (ActivityMap fetches its values lazily): before the
  // next propagation overwrites the device map, give the planner a fresh one so that map keeps its values.
  // The fresh grid is cloned on the device, so the planner never touches the caller's GridMap after
  // construction (it may die first).
  void own_map() {
    if (dev.use_count() > 1) dev = std::make_shared<detail::DeviceMap>(*dev);
  }
};

Planner::Planner(const GridMap& grid, const SourceSet& sources, DeviceOptions options) {
  std::lock_guard<std::mutex> lk(api_mutex());
  (void)options;
  auto impl = std::make_shared<PlannerImpl>();
  impl->dev = std::make_shared<detail::DeviceMap>(grid, sources);
  impl->width = grid.width();
  impl->height = grid.height();
  impl_ = impl;
}

Planner::~Planner() = default;

AutoResult Planner::propagate_auto(uint32_t auto_cap) {
  if (auto_cap == 0 || auto_cap > kMaxLayers) throw InvalidInputError("propagate_auto: auto_cap out of range");
  auto* p = static_cast<PlannerImpl*>(impl_.get());
  std::lock_guard<std::mutex> lk(api_mutex());
  p->own_map();
  am_prop_result r{};
  check(am_propagate(p->dev->ctx, p->dev->grid, 0, auto_cap, AM_MODE_BATCHED, &r), p->dev->ctx, "propagate_auto");
  p->dev->layers = r.layers_used;
  stats_ = PropagationStats{r.layers_computed, r.cell_bits, r.block_launches, r.layer_launches, r.stencil_ms};
  const AutoStop cause = r.cause == AM_STOP_FILLED ? AutoStop::kFilled
                         : r.cause == AM_STOP_STALLED ? AutoStop::kStalled
                                                      : AutoStop::kCapReached;
  // the returned map shares the planner's device map until the next propagation (own_map)
  return AutoResult{ActivityMap(p->width, p->height, r.layers_used, p->dev), r.layers_used, cause};
}

ActivityMap Planner::propagate(uint32_t layers, Mode mode) {
  if (layers == 0 || layers > kMaxLayers) throw InvalidInputError("propagate: L out of range");
  auto* p = static_cast<PlannerImpl*>(impl_.get());
  std::lock_guard<std::mutex> lk(api_mutex());
  p->own_map();
  am_prop_result r{};
  check(am_propagate(p->dev->ctx, p->dev->grid, layers, 0, mode == Mode::kBatched ? AM_MODE_BATCHED : AM_MODE_ITERATIVE,
                     &r),
        p->dev->ctx, "propagate");
  p->dev->layers = layers;
  stats_ = PropagationStats{r.layers_computed, r.cell_bits, r.block_launches, r.layer_launches, r.stencil_ms};
  return ActivityMap(p->width, p->height, layers, p->dev);
}

std::vector<PlannedPath> Planner::reconstruct_all(std::span<const Coord> targets, Method method, uint64_t seed,
                                                  CornerRule rule) {
  auto* p = static_cast<PlannerImpl*>(impl_.get());
  std::vector<int32_t> st;
  std::vector<Path> paths;
  {
    std::lock_guard<std::mutex> lk(api_mutex());
    paths = trace_batch(*p->dev, targets, method == Method::kSimple ? AM_METHOD_SIMPLE : AM_METHOD_EUCLIDEAN, seed, st);
  }
  std::vector<PlannedPath> out(targets.size());
  for (size_t i = 0; i < targets.size(); ++i) {
    out[i].target = targets[i];
    out[i].status = static_cast<TargetStatus>(st[i]);
    // the map is the device propagation's, so Euclidean paths are already straight (pin P1': two +1 moves
    // cannot span a sqrt(2) pair when 8-adjacent free cells differ by <= 1): no host straightening
    (void)rule;
    if (st[i] == AM_OK) out[i].path = std::move(paths[i]);
  }
  return out;
}

std::vector<TargetReport> Planner::target_reports(std::span<const Coord> targets, Method method, uint64_t seed,
                                                  bool emit_points, CornerRule rule) {
  auto planned = reconstruct_all(targets, method, seed, rule);
  std::vector<TargetReport> out(planned.size());
  for (size_t i = 0; i < planned.size(); ++i) {  // errors in target order, as a sequential loop reports them
    if (planned[i].status == TargetStatus::kInvalid)
      throw InvalidInputError("target out of bounds or on an obstacle " + to_string(planned[i].target));
    if (planned[i].status == TargetStatus::kInternal)
      throw Error("activity map has no ascending neighbour on the path from " + to_string(planned[i].target));
  }
  parallel_for(planned.size(), [&](size_t i) {
    TargetReport& t = out[i];
    t.target = planned[i].target;
    if (planned[i].status != TargetStatus::kOk) return;  // uncovered: recorded, not thrown (validate.hpp:76-77)
    const Path& path = planned[i].path;
    t.covered = true;
    t.reached_source = path.source();
    t.steps = path.steps();
    t.euclidean_length = path_metrics(path).euclidean_length;
    if (emit_points) t.points = std::move(planned[i].path.points);
  });
  return out;
}

}  // namespace b200

// ---------------------------------------------------------------- map / scene text (mapio.hpp)

namespace {

// device parse of `text`; the scene handle is released on every path
struct ParsedScene {
  am_ctx* ctx = nullptr;
  am_scene* sc = nullptr;
  am_parse_info info{};
  ~ParsedScene() {
    if (sc) am_scene_destroy(ctx, sc);
  }
};

void parse_text(std::string_view text, uint32_t format, ParsedScene& ps) {
  ps.ctx = default_ctx();
  const am_status st = am_scene_parse(ps.ctx, text.data(), text.size(), format, &ps.sc, &ps.info);
  if (st == AM_OK) return;
  if (st == AM_EINVAL && ps.info.error_line)
    throw ParseError(ps.info.error, ps.info.error_line, ps.info.error_column);
  if (st == AM_EINVAL && ps.info.error[0]) throw InvalidInputError(ps.info.error);
  throw_status(st, ps.ctx, "parse");
}

std::string emit_text(uint32_t format, const GridMap& grid, const std::vector<uint32_t>& src,
                      const std::vector<uint32_t>& tgt) {
  am_ctx* ctx = default_ctx();
  uint64_t n = 0;
  const auto occ = grid.occupancy();
  check(am_emit_text(ctx, format, grid.width(), grid.height(), occ.data(), src.data(), src.size() / 2, tgt.data(),
                     tgt.size() / 2, nullptr, 0, &n),
        ctx, "emit");
  std::string out(n, '\0');
  check(am_emit_text(ctx, format, grid.width(), grid.height(), occ.data(), src.data(), src.size() / 2, tgt.data(),
                     tgt.size() / 2, out.data(), n, &n),
        ctx, "emit");
  return out;
}

}  // namespace

GridMap parse_movingai(std::string_view text) {
  std::lock_guard<std::mutex> lk(api_mutex());
  ParsedScene ps;
  parse_text(text, AM_FORMAT_MOVINGAI, ps);
  std::vector<uint8_t> occ(static_cast<size_t>(ps.info.width) * ps.info.height);
  check(am_scene_download(ps.ctx, ps.sc, occ.data(), nullptr, nullptr), ps.ctx, "scene download");
  return GridMap(ps.info.width, ps.info.height, std::move(occ));
}

std::string emit_movingai(const GridMap& grid) {
  std::lock_guard<std::mutex> lk(api_mutex());
  return emit_text(AM_FORMAT_MOVINGAI, grid, {}, {});
}

Scene parse_ascii_scene(std::string_view text) {
  std::unique_lock<std::mutex> lk(api_mutex());
  ParsedScene ps;
  parse_text(text, AM_FORMAT_ASCII_SCENE, ps);
  std::vector<uint8_t> occ(static_cast<size_t>(ps.info.width) * ps.info.height);
  std::vector<uint32_t> src(2 * ps.info.n_sources), tgt(2 * ps.info.n_targets);
  check(am_scene_download(ps.ctx, ps.sc, occ.data(), src.data(), tgt.data()), ps.ctx, "scene download");
  lk.unlock();
  std::vector<Coord> s(ps.info.n_sources), t(ps.info.n_targets);
  for (size_t i = 0; i < s.size(); ++i) s[i] = Coord{src[2 * i], src[2 * i + 1]};
  for (size_t i = 0; i < t.size(); ++i) t[i] = Coord{tgt[2 * i], tgt[2 * i + 1]};
  GridMap g(ps.info.width, ps.info.height, std::move(occ));
  SourceSet set(g, s);
  return Scene{std::move(g), std::move(set), std::move(t)};
}

std::string emit_ascii_scene(const Scene& scene) {
  std::lock_guard<std::mutex> lk(api_mutex());
  return emit_text(AM_FORMAT_ASCII_SCENE, scene.grid, flatten(scene.sources.coords()), flatten(scene.targets));
}

std::string export_pgm(const ActivityMap& activity) {
  const auto& dev = activity.device_map();
  if (dev) {
    std::lock_guard<std::mutex> lk(api_mutex());
    uint64_t n = 0;
    check(am_activity_export_pgm(dev->ctx, dev->grid, nullptr, 0, &n), dev->ctx, "export_pgm");
    std::string out(n, '\0');
    check(am_activity_export_pgm(dev->ctx, dev->grid, reinterpret_cast<uint8_t*>(out.data()), n, &n), dev->ctx,
          "export_pgm");
    return out;
  }
  const auto vals = activity.values();
  std::lock_guard<std::mutex> lk(api_mutex());
  am_ctx* ctx = default_ctx();
  uint64_t n = 0;
  check(am_export_pgm(ctx, activity.width(), activity.height(), vals.data(), nullptr, 0, &n), ctx, "export_pgm");
  std::string out(n, '\0');
  check(am_export_pgm(ctx, activity.width(), activity.height(), vals.data(), reinterpret_cast<uint8_t*>(out.data()), n,
                      &n),
        ctx, "export_pgm");
  return out;
}

}  // namespace actmap

// ------------------------------------------------- C-ABI host helpers
extern "C" {

am_status am_random_maze(uint32_t w, uint32_t h, double density, uint64_t seed, uint8_t* occ) {
  if (!occ) return AM_EINVAL;
  try {
    const auto g = actmap::random_maze(w, h, density, seed);
    std::memcpy(occ, g.occupancy().data(), g.cell_count());
    return AM_OK;
  } catch (const actmap::InvalidInputError&) {
    return AM_EINVAL;
  } catch (...) {
    return AM_EINTERNAL;
  }
}

am_status am_kruskal_maze(uint32_t w, uint32_t h, uint64_t seed, uint8_t* occ) {
  if (!occ) return AM_EINVAL;
  try {
    const auto g = actmap::kruskal_maze(w, h, seed);
    std::memcpy(occ, g.occupancy().data(), g.cell_count());
    return AM_OK;
  } catch (const actmap::InvalidInputError&) {
    return AM_EINVAL;
  } catch (...) {
    return AM_EINTERNAL;
  }
}

am_status am_city_grid(uint32_t w, uint32_t h, uint64_t seed, uint8_t* occ) {
  if (!occ) return AM_EINVAL;
  try {
    const auto g = actmap::city_grid(w, h, seed);
    std::memcpy(occ, g.occupancy().data(), g.cell_count());
    return AM_OK;
  } catch (const actmap::InvalidInputError&) {
    return AM_EINVAL;
  } catch (...) {
    return AM_EINTERNAL;
  }
}

am_status am_comb_maze(uint32_t w, uint32_t h, uint8_t* occ) {
  if (!occ) return AM_EINVAL;
  try {
    const auto g = actmap::comb_maze(w, h);
    std::memcpy(occ, g.occupancy().data(), g.cell_count());
    return AM_OK;
  } catch (const actmap::InvalidInputError&) {
    return AM_EINVAL;
  } catch (...) {
    return AM_EINTERNAL;
  }
}

am_status am_straighten(const uint32_t* pts, uint64_t n, const uint8_t* occ, uint32_t w, uint32_t h, uint32_t rule,
                        uint32_t* out, uint64_t* n_out) {
  if ((n && (!pts || !out)) || !n_out) return AM_EINVAL;
  try {
    actmap::Path p;
    p.points.resize(n);
    for (uint64_t i = 0; i < n; ++i) p.points[i] = actmap::Coord{pts[2 * i], pts[2 * i + 1]};
    actmap::Path s;
    if (occ) {
      actmap::GridMap g(w, h, std::vector<uint8_t>(occ, occ + (size_t)w * h));
      s = actmap::straighten(p, g, rule ? actmap::CornerRule::kPermissive : actmap::CornerRule::kStrict);
    } else {
      s = actmap::straighten(p);
    }
    for (size_t i = 0; i < s.points.size(); ++i) {
      out[2 * i] = s.points[i].row;
      out[2 * i + 1] = s.points[i].col;
    }
    *n_out = s.points.size();
    return AM_OK;
  } catch (const actmap::InvalidInputError&) {
    return AM_EINVAL;
  } catch (...) {
    return AM_EINTERNAL;
  }
}

am_status am_path_metrics(const uint32_t* pts, uint64_t n, uint64_t* steps, double* length) {
  if ((n && !pts) || !steps || !length) return AM_EINVAL;
  actmap::Path p;
  p.points.resize(n);
  for (uint64_t i = 0; i < n; ++i) p.points[i] = actmap::Coord{pts[2 * i], pts[2 * i + 1]};
  const auto m = actmap::path_metrics(p);
  *steps = m.steps;
  *length = m.euclidean_length;
  return AM_OK;
}

}  // extern "C"
