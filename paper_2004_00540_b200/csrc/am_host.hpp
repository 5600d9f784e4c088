// am_host.hpp -- host-side state shared by capi.cu (single grid, propagation
// driver, paths) and multigpu.cu (row slabs: in-process groups and NCCL).
#pragma once

#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/actmap_b200.h"
#include "am_internal.cuh"

namespace am {
constexpr int kLag = 2;        // blocks in flight before the host reads a fixed-point flag (dense)
#ifndef AM_LAG_TILES
#define AM_LAG_TILES 24
#endif
constexpr int kLagTiles = AM_LAG_TILES;  // same, active-tile mode (< kFlagSlots)
struct Comm;             // NCCL communicator wrapper (multigpu.cu)
struct HostPool;         // host worker threads (upload.cu)
void host_pool_destroy(HostPool* p);
struct PeerLink;         // peer-memory slab transport state (multigpu.cu)
// bit-plane propagation state of a single grid (bits.cu), allocated on first use
struct BitState {
  BitGeo bg{};
  BitBook bk{};
  int ctas = 0;
  uint32_t* own_t = nullptr;  // time planes when the second field is too small for them
  uint64_t free_cells = 0;    // free cells of the grid (counted when the free plane is built)
  bool planes_ready = false;  // the free plane of the grid's occupancy is built (once per grid)
};
void peer_destroy(PeerLink* p);
// Host side of a grid's fixed-point slots: pinned device-mapped mirror + one
// event per slot.  Pinning and event creation are slow, so contexts recycle
// these across grids.
struct FlagSet {
  uint32_t* h = nullptr;     // pinned, device-mapped mirror
  uint32_t* hdev = nullptr;  // its device address
  cudaEvent_t ev[kFlagSlots] = {};
};
}  // namespace am

struct am_ctx {
  int device = 0;
  uint32_t flags = 0;
  cudaStream_t stream = nullptr;
  int sms = 148;
  int warp_slots = 0;
  uint64_t launches = 0;
  std::string err;
  struct Timer {
    cudaEvent_t a, b;
  };
  std::vector<Timer> timers;
  am::Comm* comm = nullptr;  // set by am_comm_init
  cudaMemPool_t pool = nullptr;  // every device buffer of the context's grids (am::dmalloc)
  std::vector<am::FlagSet*> flag_sets;  // recycled FlagSets of destroyed grids
  cudaStream_t copy_stream = nullptr;   // map downloads: D2H copies overlapping the chunk decode
  cudaEvent_t copy_ev[8] = {};
  // packed occupancy upload (upload.cu): host workers, pinned staging, device copy of the packed rows
  am::HostPool* hpool = nullptr;
  uint32_t* h_pack = nullptr;
  size_t h_pack_cap = 0;
  uint32_t* d_pack = nullptr;
  size_t d_pack_cap = 0;
  uint32_t pack_rows = 0, pack_w = 0;  // the rows d_pack holds (valid until the next upload)
  uint64_t h2d_bytes = 0;              // host-to-device bytes copied by this context
  cudaStream_t map_stream = nullptr;   // k_bits_finalize (field encoding) beside the path walkers
};

struct am_grid {
  am::Geo g{};
  int cell_bits = 16;
  void* val[2] = {nullptr, nullptr};
  int cur = 0;
  uint8_t* srcmask = nullptr;        // pitched 0/1 (owned rows + halo rows for slabs)
  uint8_t* rowsrc = nullptr;         // per band and allocated row: a source in the band's columns (Geo::rowsrc_bytes)
  uint8_t* occ = nullptr;            // dense owned rows (re-initialisation / plain maps)
  uint32_t* src_rc = nullptr;        // the SourceSet, global (row, col) pairs (re-initialisation)
  uint64_t n_src = 0;
  uint8_t* srcmask_dense = nullptr;  // dense owned rows (plain maps)
  uint32_t* d_flags = nullptr;       // kFlagWords: fixed-point slots, CTA arrival counter, neighbour receive rings
  am::FlagSet* fs = nullptr;         // host mirror + events of the slots (borrowed from the context)
  uint32_t* plain = nullptr;         // caller-uploaded dense map
  int plain_active = 0;
  uint32_t plain_layers = 0;
  int have_map = 0;
  int dirty[2] = {0, 0};    // buffer reused as download staging: padding no longer unflagged
  uint32_t computed = 0;    // layers represented by val[cur]
  uint32_t layers_used = 0; // logical layers (val[cur] minus rollback)
  // row-slab membership: this grid holds rows [row0, row0 + g.H) of a total_h-row grid
  int slab = 0;
  uint32_t total_h = 0, row0 = 0;
  // active-tile skipping state (single grids; stencil.cu k_tiles_*)
  unsigned long long* t_state = nullptr;     // per tile: old << 32 | cur (am::TileBook)
  uint32_t* t_sched = nullptr;               // per tile: index + 1 of the block it is listed for
  uint32_t* t_list[2] = {nullptr, nullptr};  // work lists (band << 16 | chunk) by block parity
  uint32_t* t_count = nullptr;               // [6] list lengths, item fetch counters (TileBook::count)
  unsigned long long* t_processed = nullptr; // tiles processed (statistics)
  uint32_t t_blk = 0;                        // index of the next tile block (list / counter selection)
  void* t_bnd = nullptr;                     // slabs: first / last kK rows gathered for the neighbours (2 x kK x pitch)
  uint8_t* t_src = nullptr;                  // per tile: a source in its staged rows (TileBook::tsrc)
  am::PeerLink* peer = nullptr;              // slabs: peer-memory transport (am_peer_connect)
  am::BitState* bits = nullptr;              // bit-plane propagation (single grids, 16-bit runs)
  int bits_map = 0;                          // val[0] came from a bit-plane run whose planes are intact
  cudaEvent_t map_ev = nullptr;              // recorded on ctx->map_stream after the field encoding
  int map_pending = 0;                       // ctx->stream has not waited on map_ev yet
  am::TileBook book() const {
    return am::TileBook{t_state, t_sched, {t_list[0], t_list[1]}, t_count, t_processed, t_src};
  }
  // scratch for path extraction
  uint32_t* d_tgt = nullptr;
  uint64_t* d_counts = nullptr;
  uint32_t* d_sched = nullptr;  // launch_trace's longest-first scheduling (kTraceSchedWords)
  uint64_t* d_offsets = nullptr;
  int32_t* d_status = nullptr;
  uint64_t tgt_cap = 0;
  uint32_t* d_pts = nullptr;
  uint64_t pts_cap = 0;
};

namespace am {

// Stream-ordered allocation from the context's pool: memory released by a
// destroyed grid is reused by the next one without a driver round trip.
template <class T>
inline cudaError_t dmalloc(am_ctx* c, T** p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) return cudaSuccess;
  return cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, c->pool, c->stream);
}
inline void dfree(am_ctx* c, void* p) {
  if (p) cudaFreeAsync(p, c->stream);
}

inline am_status fail(am_ctx* ctx, am_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return st;
}

inline bool dims_ok(uint32_t w, uint32_t h) { return w >= 1 && h >= 1 && w <= 65535 && h <= 65535; }

// rows [first, last) of slab r out of n over h rows
// Slab boundaries fall on tile-chunk multiples (kTileRows) whenever every
// slab keeps at least two chunks, so active-tile skipping works across slabs.
inline void slab_rows(uint32_t h, uint32_t n, uint32_t r, uint32_t* first, uint32_t* last) {
  auto cut = [&](uint32_t k) -> uint32_t {
    uint64_t b = (uint64_t)h * k / n;
    if (k > 0 && k < n && h >= 2u * kTileRows * n) b = (b + kTileRows / 2) / kTileRows * kTileRows;
    return (uint32_t)b;
  };
  *first = cut(r);
  *last = cut(r + 1);
}

// Halo transport used by the propagation driver between blocks.
struct Transport {
  virtual ~Transport() = default;
  // enqueue the K-row halo refresh of every local slab (reads current buffers)
  virtual am_status exchange() = 0;
  // active tiles: send each slab's gathered boundary rows (t_bnd) into its
  // neighbours' halo rows of field 0
  virtual am_status exchange_tiles() = 0;
  // make the per-slab device word *w (one per local slab) global: min or max over all slabs
  virtual am_status reduce(std::vector<uint32_t*>& words, bool take_max) = 0;
  // The per-block fixed-point words travel with the halo rows instead of an
  // all-reduce per block: exchange() / exchange_tiles() also send every slab's
  // kFlagSlots slot words to both neighbours and fold the neighbours' words in
  // (d_flags receive rings + launch_flags_merge), one hop per exchange, so a
  // block's word is the minimum over all slabs after span() - 1 further
  // exchanges.  exchange_flags() is such an exchange without the rows.
  virtual uint32_t span() const = 0;  // slabs in the chain
  virtual am_status exchange_flags() = 0;
  // local values must still be combined on the host (in-process groups)
  virtual bool host_combine() const = 0;
  // a one-slab-per-process transport whose slab has a neighbour below it
  // (its bottom halo holds that neighbour's rows, not padding)
  virtual bool lower_neighbour() const { return false; }
  // every slab of the chain (all ranks) meets its lower neighbour on a tile-chunk boundary, so every
  // rank runs the same mode (active tiles or dense) and issues the same sequence of exchanges
  virtual bool chain_tiles_ok() const { return true; }
  // where the boundary kernel stores the slab's first (side 0) / last (side 1) kK rows for the next
  // exchange_tiles(); nullptr: the slab's own t_bnd (the transport moves them)
  virtual void* boundary_dst(int side) { (void)side; return nullptr; }
};

struct SlabRef {
  am_ctx* ctx;
  am_grid* g;
};

// am_trace_paths with an optional maze-local coordinate pass (cell_h/cell_w > 0, am_batch)
am_status trace_paths_host(am_ctx* ctx, am_grid* g, const uint32_t* tgt, uint64_t n, uint32_t method, uint64_t seed,
                           const uint64_t* offsets, uint32_t* pts, uint64_t cap, int32_t* status, uint32_t cell_h,
                           uint32_t cell_w);

Transport* make_peer_transport(am_ctx* ctx, am_grid* g);
// per-grid path-extraction scratch (targets, counts, offsets, status) for n targets
am_status trace_scratch(am_ctx* ctx, am_grid* g, uint64_t n);

// The propagation driver (capi.cu): runs slabs in lock step, 1 slab = single grid.
am_status drive_propagation(std::vector<SlabRef>& slabs, Transport* tr, uint32_t layers, uint32_t auto_cap,
                            uint32_t mode, am_prop_result* res);
am_status grid_create_rows(am_ctx* ctx, uint32_t W, uint32_t H_total, uint32_t row0, uint32_t row1,
                           const uint8_t* occ_full, const uint32_t* src, uint64_t n_src, bool device_ptrs,
                           bool slab, am_grid** out);
am_status set_cell_bits(am_ctx* ctx, am_grid* g, int cell_bits);
// bit-plane state + the grid's free plane (capi.cu); packed: the grid's occupancy as packed rows
// (upload.cu) to build it from, else the dense bytes are read
am_status bits_alloc(am_ctx* ctx, am_grid* g, const uint32_t* packed = nullptr);
// Orders the context stream after the grid's field encoding (k_bits_finalize on the map stream): every
// entry point that reads or rewrites the field calls this first; path counts and walks read the planes
// and join after their launches.
am_status join_map(am_ctx* ctx, am_grid* g);
am_status upload_occupancy_packed(am_ctx* ctx, const uint8_t* occ, uint32_t W, uint32_t H, uint8_t* d_occ);

}  // namespace am

#define CK(call)                                                                                     \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) {                                                                         \
      (void)cudaGetLastError();                                                                      \
      return am::fail(ctx, e_ == cudaErrorMemoryAllocation ? AM_EOOM : AM_ECUDA, "%s: %s (%s:%d)", #call, \
                      cudaGetErrorString(e_), __FILE__, __LINE__);                                   \
    }                                                                                                \
  } while (0)

#define CKL()                  \
  do {                         \
    ++ctx->launches;           \
    CK(cudaPeekAtLastError()); \
  } while (0)
