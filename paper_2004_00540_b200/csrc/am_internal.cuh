// am_internal.cuh -- device layout, cell encoding and kernel declarations
// shared by the sm_100a kernels and the C-ABI host code.
//
// Device layout.  The reference map is a dense row-major
// uint32 field (activity.hpp:51) plus a dense uint8 occupancy grid
// (grid.hpp:56).  On the device one pitched field carries BOTH: every free
// cell has its top bit set ("flag") and its activity a in the low bits; every
// obstacle or padding cell has the flag clear and is semantically 0.  Then the
// layer step  out = max3x3(in) & (in_center | LOWMASK)  is exactly
// propagate_layer (propagate.hpp:34-38): a free centre keeps the flagged max
// of its neighbourhood (unflagged obstacles can never win against the
// centre's own flagged value), an obstacle centre loses its flag.  Sources
// add +1 (rare; see the source-row flags).  No occupancy bytes are read
// inside the stencil at all.
//
// Cell width: 16-bit (a <= 0x7FFF) while layers+1 <= 32767, packed two
// independent tiles per 32-bit word ("u16x2 tile pairs": lo half = tile A,
// hi half = tile B, so the 3x3 max never needs a byte permute); promoted
// exactly to 32-bit cells (a <= 2^31-1 = kMaxLayers+1) beyond that.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace am {

constexpr uint32_t kFlag16 = 0x8000u;
constexpr uint32_t kLow16x2 = 0x7FFF7FFFu;
constexpr uint32_t kFlag32 = 0x80000000u;
constexpr uint32_t kLow32 = 0x7FFFFFFFu;
constexpr uint32_t kMax16Activity = 0x7FFFu;      // largest a representable in 16-bit cells
constexpr uint32_t kMaxLayers = 2147483646u;      // propagate.hpp:15-16

// Temporal-block kernel shape: each warp streams a vertical band of
// 32*kWPL cells (kK-cell halo each side) down a row segment, running kK
// layers per HBM round trip in registers.
constexpr int kWPL = 8;          // words per lane
constexpr int kK = 8;            // layers per block (= halo depth)
constexpr int kBand = 32 * kWPL; // band width in cells (incl. halo)
constexpr int kBandUseful = kBand - 2 * kK;
constexpr int kBlockThreads = 128;

// Active-tile skipping works on tiles of kTileRows rows x kTileCols columns,
// streamed by warps with kTileWPL words per lane: narrower than the dense
// bands, so a frontier activates fewer cells and a warp's item is shorter.
#ifndef AM_TILE_ROWS
#define AM_TILE_ROWS 32
#endif
#ifndef AM_TILE_WPL
#define AM_TILE_WPL 4
#endif
constexpr int kTileRows = AM_TILE_ROWS;
constexpr int kTileWPL = AM_TILE_WPL;
constexpr int kTileCols = 32 * kTileWPL - 2 * kK;  // useful columns of a tile band
#ifndef AM_TILE_CTAS
#define AM_TILE_CTAS 3  // 4 warps x 12 KB staged tiles each, <= 168 registers
#endif
constexpr int kTileCtasPerSm = AM_TILE_CTAS;  // k_block_tiles is persistent: this many CTAs per SM
#ifndef AM_TILE_THREADS
#define AM_TILE_THREADS 128
#endif
constexpr int kTileThreads = AM_TILE_THREADS;  // threads per k_block_tiles CTA (one item per warp)

// Fixed-point word slots per grid (a ring the host reads lagged).  A grid's
// d_flags holds the slots, the CTA arrival counter (FlagSink::done), and two
// receive rings for the neighbours' slots (row slabs: the words travel with the
// halo rows, see Transport in am_host.hpp).
constexpr int kFlagSlots = 64;
constexpr int kFlagRecvUp = kFlagSlots + 1;
constexpr int kFlagRecvDn = 2 * kFlagSlots + 1;
constexpr int kFlagWords = 3 * kFlagSlots + 1;

struct Geo {
  uint32_t W, H;          // grid extent (cells)
  uint32_t pad;           // = kK: rows above / cols left of the grid
  uint32_t pitch;         // elements per allocated row
  uint32_t rows;          // allocated rows
  uint32_t nbands;        // vertical bands of kBandUseful cells
  uint32_t nseg;          // row segments (even)
  uint32_t seg_len;       // rows per segment (even)
  uint32_t nchunks;       // row chunks of kTileRows (tile rows)
  uint32_t tbands;        // tile bands of kTileCols columns
  __host__ __device__ uint32_t ntiles() const { return tbands * nchunks; }
  // per-band source-row flags (rowsrc): one byte per allocated row for each
  // dense band, then for each tile band; set where the band's streamed
  // columns (useful + halo) hold a source in that row
  __host__ __device__ size_t rowsrc_bytes() const { return (size_t)(nbands + tbands) * rows; }
  __host__ __device__ size_t dense_rowsrc(uint32_t band) const { return (size_t)band * rows; }
  __host__ __device__ size_t tile_rowsrc(uint32_t tband) const { return (size_t)(nbands + tband) * rows; }
  __host__ __device__ size_t idx(uint32_t r, uint32_t c) const {
    return (size_t)(r + pad) * pitch + (c + pad);
  }
};

Geo make_geo(uint32_t W, uint32_t H, int num_sms);

// Where a blocked launch leaves its fixed-point word (min over covered cells
// of a-1): `word` is the device slot the warps atomicMin into.  With `host`
// set, the last CTA to finish copies the word into that host-mapped pinned
// slot and re-arms word (all ones) and `done` (0), so the driver reads the
// signal after an event without a copy-engine op between launches.
struct FlagSink {
  uint32_t* word;
  uint32_t* done;  // CTA arrival counter, 0 between launches
  uint32_t* host;  // mapped mirror slot, or null (word left for the caller)
};

// Active-tile bookkeeping (stencil.cu k_block_tiles / k_tiles_*).  A tile's
// state word is  old << 32 | cur  with cur = layer << 1 | home field of the
// tile's latest values; a tile processed in the running block writes
// cur = (l0 + kK) << 1 | home^1 and keeps its pre-block word in `old`, so a
// neighbour reading it during the same block can still tell the values it
// must read (cur's layer == l0 + kK marks "processed in this block").  Work
// lists are pushed by the processed tiles themselves: block `blk` reads
// list[blk & 1] / count[blk % 3], appends to list[(blk+1) & 1] /
// count[(blk+1) % 3] (deduplicated by sched[t] = the index + 1 of the block
// a tile is listed for) and clears count[(blk+2) % 3].
struct TileBook {
  unsigned long long* state;
  uint32_t* sched;
  uint32_t* list[2];
  uint32_t* count;                // [6]: list lengths [0..2], item fetch counters [3..5] (both by block mod 3)
  unsigned long long* processed;  // tiles processed (statistics)
  const uint8_t* tsrc;            // per tile: a source lies in the rows its items stage (static)
};
// list entries: band << 16 | chunk, plus kListSrc when the tile's tsrc is set (the item takes the source path
// without reading the per-row flags first)
constexpr uint32_t kListSrc = 1u << 31;
constexpr uint32_t kListBand = 0x7FFFu;

// ---- kernels (stencil.cu) ----
// layer 0 (initial, activity.hpp:21): flag on free cells; then +1 at the sources of rows
// [row0, row0 + g.H) (src_rc: n global (row, col) pairs, already validated)
void launch_init(const Geo& g, const uint8_t* d_occ_dense, void* d_val, int cell_bits, cudaStream_t s);
void launch_src_init(const Geo& g, const uint32_t* src_rc, uint64_t n, uint32_t row0, void* d_val, int cell_bits,
                     cudaStream_t s);
void launch_srcmask_rows(const Geo& g, uint32_t total_h, uint32_t row0, const uint32_t* d_src_rc, uint64_t n,
                         uint8_t* d_dense, const uint8_t* d_occ, uint8_t* d_srcmask, uint8_t* d_rowsrc, int* d_err,
                         cudaStream_t s);
void launch_block(const Geo& g, int cell_bits, bool slab, const void* in, void* out, const uint8_t* srcmask,
                  const uint8_t* rowsrc, FlagSink flag, cudaStream_t s);
void launch_layer(const Geo& g, int cell_bits, const void* in, void* out, const uint8_t* srcmask,
                  uint32_t* flag, cudaStream_t s);
// active-tile skipping (stencil.cu)
// lists the tiles of block 0: the 3x3 tile neighbourhood of every tile holding a source
void launch_tiles_init(const Geo& g, const uint8_t* srcmask, TileBook book, cudaStream_t s);
// TileBook::tsrc from the per-band source-row flags (after launch_srcmask_rows)
void launch_tile_src(const Geo& g, const uint8_t* rowsrc, uint8_t* tsrc, cudaStream_t s);
// every tile current at `layer` in field `home`, all listed for block blk
void launch_tiles_all(const Geo& g, TileBook book, uint32_t blk, uint32_t layer, int home, cudaStream_t s);
// pdl: launch with programmatic stream serialization (back-to-back tile blocks on one stream)
// prev: the previous tile block's word, published (host + re-arm) by this launch; flag.host must be null
void launch_block_tiles(const Geo& g, int cell_bits, int ctas, void* f0, void* f1, const uint8_t* srcmask,
                        const uint8_t* rowsrc, TileBook book, uint32_t blk, uint32_t l0, FlagSink flag,
                        FlagSink prev, bool pdl, cudaStream_t s);
// publishes a word the way the last CTA of a blocked launch would (FlagSink)
void launch_publish_flag(FlagSink f, cudaStream_t s);
// slots[k] = min(slots[k], received from above[k], received from below[k]) for every slot
void launch_flags_merge(uint32_t* d_flags, cudaStream_t s);
// zero (nullable): also ORs 1 into *zero if a free cell is still uncovered (fused k_zero_check)
void launch_tiles_finalize(const Geo& g, int cell_bits, unsigned long long* state, void* f0, void* f1, int dst,
                           uint32_t l, uint32_t* zero, cudaStream_t s);
// row slabs with active tiles: the slab's first / last kK rows at layer l into
// bnd (2 x kK x pitch, the halo rows its neighbours read), and the list entry
// of every boundary tile a frontier cell in the received halo rows can reach
void launch_tiles_boundary(const Geo& g, int cell_bits, const unsigned long long* state, void* f0, void* f1,
                           uint32_t l, void* dst_top, void* dst_bottom, cudaStream_t s);
// min (take_max = 0) or max over n words into *out
void launch_peer_reduce(const uint32_t* vals, uint32_t n, int take_max, uint32_t* out, cudaStream_t s);
void launch_tiles_halo_scan(const Geo& g, int cell_bits, const void* f0, TileBook book, uint32_t blk, cudaStream_t s);
void launch_promote(const Geo& g, const uint16_t* in, uint32_t* out, cudaStream_t s);
void launch_zero_check(const Geo& g, int cell_bits, const void* val, uint32_t* flag, cudaStream_t s);
void launch_decode(const Geo& g, int cell_bits, const void* val, uint32_t rollback, uint32_t r0, uint32_t r1,
                   uint32_t* dense_rows, cudaStream_t s);
int block_kernel_blocks_per_sm(int cell_bits);
void launch_encode_dense(const Geo& g, const uint32_t* dense, const uint8_t* occ_dense, uint32_t* val32,
                         cudaStream_t s);
void launch_plain_layer(uint32_t W, uint32_t H, const uint8_t* occ, const uint8_t* srcmask_dense,
                        const uint32_t* in, uint32_t* out, cudaStream_t s);
void launch_sentinel_layer(uint32_t W, uint32_t H, const uint8_t* occ, const uint8_t* srcmask_dense,
                           const int32_t* in, int32_t* out, cudaStream_t s);
void launch_srcmask_dense(uint32_t W, uint32_t H, const uint32_t* d_src_rc, uint64_t n, uint8_t* d_srcmask,
                          const uint8_t* d_occ, int* d_err, cudaStream_t s);

// ---- bit-plane propagation (bits.cu) ----
// Tiles of kBTR rows x kBTW words (32 cells each); a warp holds a tile plus a
// kBK-deep halo (32*kBRPL rows, kBTW+2 words) and runs kBK layers per launch.
#ifndef AM_BK
#define AM_BK 16
#endif
#ifndef AM_BRPL
#define AM_BRPL 2
#endif
#ifndef AM_BITS_PCM
#define AM_BITS_PCM 1
#endif
constexpr int kBK = AM_BK;
constexpr int kBRPL = AM_BRPL;
constexpr int kBTW = 4;
constexpr int kBTR = 32 * kBRPL - 2 * kBK;
// time planes: bit k < kBTPlanes of t - 1 per cell (t = the layer a cell was covered at); word slots
// kBTPlanes .. 15 of a row word's 16 are unused during the run (k_bits_finalize puts covered / free there)
constexpr int kBTPlanes = 14;
constexpr uint32_t kBTSrcU = (1u << kBTPlanes) - 1u;     // sources' t - 1 (== -1 mod 2^kBTPlanes)
constexpr uint32_t kBitsMaxRef = (1u << kBTPlanes) - 2u;  // layers a bit-plane run represents (16382)
struct BitGeo {
  uint32_t W, H;
  uint32_t nchunks, tbands;  // tile rows / tile columns
  uint32_t wpr;              // plane words per row (tbands * kBTW)
  uint32_t rows;             // plane rows (nchunks * kBTR)
  __host__ __device__ uint32_t ntiles() const { return nchunks * tbands; }
  __host__ __device__ size_t plane_words() const { return (size_t)rows * wpr; }
  // plane word (row, word) of P: column-major (a word column's rows contiguous), so the lane-per-row
  // accesses of the tile kernel and the walkers touch 8 lines per warp instead of 32 (AM_BITS_PCM)
  __host__ __device__ size_t pidx(uint32_t row, uint32_t word) const {
#if AM_BITS_PCM
    return (size_t)word * rows + row;
#else
    return (size_t)row * wpr + word;
#endif
  }
  // row word (row, word) of the time planes T (16 words each): row-major
  __host__ __device__ size_t tidx(uint32_t row, uint32_t word) const { return (size_t)row * wpr + word; }
};
BitGeo make_bit_geo(uint32_t W, uint32_t H);
// Device state of a bit-plane run.  State words and lists work as in TileBook
// (state = old << 32 | cur, cur = (index + 1 of the block that last processed the
// tile) << 1 | home plane; lists / counts by block parity / block mod 3).  cur = 0: no block of this run
// has processed the tile and it holds no source, so its coverage words are stale and read as empty (runs
// reset only the states, never the planes).
struct BitBook {
  uint4* P;                    // plane words {covered (home 0), covered (home 1), free, -}; free is built once per grid
  uint32_t* T;                 // time planes: 16 words per plane word (bit k of t - 1 of its 32 cells)
  unsigned long long* state;
  uint32_t* sched;
  uint32_t* list[2];
  uint32_t* count;             // [12]: [0..2] items per block, [3..5] fetch counters, [6..8] k_bits_run flags
  unsigned long long* stat;    // [0] tiles processed, [1] cells covered, [2] free cells
  uint32_t* hcount;            // mapped host mirror (device address) of each block's items by slot, or null
};
int bits_ctas_per_sm();
void launch_bits_init(const BitGeo& bg, const uint8_t* occ, BitBook bk, cudaStream_t s);
// the same from packed rows (bit = obstacle, (W + 31) / 32 words per row; upload.cu)
void launch_bits_init_packed(const BitGeo& bg, const uint32_t* packed, BitBook bk, cudaStream_t s);
void launch_bits_sources(const BitGeo& bg, const uint32_t* rc, uint64_t n, BitBook bk, cudaStream_t s);
void launch_bits_tiles(const BitGeo& bg, int ctas, BitBook bk, uint32_t blk, uint32_t nl, FlagSink flag,
                       FlagSink prev, cudaStream_t s);
// k_bits_run: CTAs per cluster it can run with (0: no cluster fits), the tiles one pass of its warps covers
int bits_run_cluster();
uint32_t bits_run_warps(int cluster);
void launch_bits_run(const BitGeo& bg, int cluster, BitBook bk, uint32_t blk, uint32_t blk_end, uint32_t nmax,
                     bool autom, uint32_t seq, uint32_t* rec, cudaStream_t s);
// the encoded 16-bit field (values relative to lref layers) from the planes
void launch_bits_finalize(const BitGeo& bg, const Geo& g, BitBook bk, uint32_t lref, uint16_t* field, int sms,
                          cudaStream_t s);

// ---- path extraction (trace.cu) ----
// A map distributed over row slabs (peer transport): grid row r lives in slab s with row0[s] <= r <
// row0[s+1], at base[s] + (r - row0[s]) * pitch cells (base: the slabs' published rows, peer-mapped);
// rows outside the grid read the zero row.  Device memory, built by am_peer_connect.
constexpr uint32_t kSlabDirMax = 64;
struct SlabDir {
  uint32_t n;
  uint32_t row0[kSlabDirMax + 1];
  const void* base[kSlabDirMax];
  const void* zero;  // one zero row (pitch cells of either width)
};
struct MapView {
  const void* val;        // encoded pitched field (cell_bits 16/32) or plain dense uint32 (cell_bits 0)
  const uint8_t* srcmask; // pitched (encoded) or dense (plain)
  Geo g;
  int cell_bits;          // 16, 32, or 0 = plain dense uint32 + dense occupancy
  const uint8_t* occ;     // plain mode only: dense occupancy
  uint32_t layers;        // layers represented by the values (for point counts)
  const SlabDir* dir = nullptr;  // encoded maps only: the field is distributed over row slabs (val unused)
  uint32_t cell_h = 0, cell_w = 0;  // > 0: mazes packed on this lattice, paths written maze-local
  // maps of a bit-plane run (bits.cu) whose planes are intact: path counts and walkers read the planes
  // (the encoded field may still be in flight on the map stream)
  const uint4* bp = nullptr;                 // {covered (home 0), covered (home 1), free, -} per plane word
  const uint32_t* bt = nullptr;              // time planes, 16 words per plane word
  const unsigned long long* bstate = nullptr;  // tile states (home plane; 0: nothing covered)
  BitGeo bg{};
  // covered / free bits and t - 1 of cell (r, c) of a bit-plane map (r < H, c < W)
  __device__ __forceinline__ uint32_t bword(uint32_t r, uint32_t c, uint32_t* free_bit) const {
    const uint4 p = bp[bg.pidx(r, c >> 5)];
    const uint32_t st = (uint32_t)bstate[(r / kBTR) * bg.tbands + (c >> 5) / kBTW];
    *free_bit = (p.z >> (c & 31)) & 1u;
    const uint32_t cov = st == 0u ? 0u : (st & 1u) ? p.y : p.x;
    return (cov >> (c & 31)) & 1u;
  }
  __device__ __forceinline__ uint32_t bu(uint32_t r, uint32_t c) const {
    const uint32_t* t = bt + bg.tidx(r, c >> 5) * 16;
    uint32_t u = 0;
    for (int k = 0; k < kBTPlanes; ++k) u |= ((t[k] >> (c & 31)) & 1u) << k;
    return u;
  }
  // allocated row arow of an encoded field (cell 0 = allocated column 0)
  template <typename T>
  __device__ __forceinline__ const T* row(int arow) const {
    if (!dir) return static_cast<const T*>(val) + (size_t)arow * g.pitch;
    const int r = arow - (int)g.pad;
    if (r < 0 || r >= (int)g.H) return static_cast<const T*>(dir->zero);
    uint32_t s = 0;
    while (s + 1 < dir->n && (uint32_t)r >= dir->row0[s + 1]) ++s;
    return static_cast<const T*>(dir->base[s]) + (size_t)((uint32_t)r - dir->row0[s]) * g.pitch;
  }
};
void launch_path_counts(const MapView& m, const uint32_t* tgt_rc, uint64_t n, int method, uint64_t seed,
                        uint64_t* counts, int32_t* status, cudaStream_t s);
void launch_scan(const uint64_t* counts, uint64_t n, uint64_t* offsets, cudaStream_t s);
void launch_trace(const MapView& m, const uint32_t* tgt_rc, uint64_t n, int method, uint64_t seed,
                  const uint64_t* offsets, uint32_t* pts_rc, int32_t* status, cudaStream_t s,
                  uint64_t pts_capacity = ~0ull, uint32_t* order = nullptr, uint32_t* sched = nullptr, int sms = 0);
// scratch of launch_trace's longest-first scheduling: order (n words) and sched (this many words)
constexpr int kTraceSchedWords = 1024 + 2;

}  // namespace am
