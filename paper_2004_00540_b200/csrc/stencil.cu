// stencil.cu -- sm_100a kernels for the oMAP layer stack (propagate.hpp:34-68).
//
// K1+K2: a warp streams a band of cells down a run of rows and applies kK
// pool+add+ReLU layers per HBM round trip entirely in registers (per-layer
// 3-row window, warp-shuffle horizontal halo), writes the useful middle of
// the band and folds the fixed-point signal (min over covered cells of a-1)
// into one atomicMin per warp.  k_block sweeps every band of the grid (dense
// mode, 240-column bands); k_block_tiles runs only the active 32x112 tiles
// (exact skipping: quiet tiles advance lazily through a per-tile lag) and
// lists the next block's tiles itself.  See DESIGN.md §4.
#include <cuda.h>  // CUtensorMap (TMA descriptors; encoded through the runtime's driver entry point)

#include <cstdio>
#include <cstdlib>

#include "am_internal.cuh"

// AM_TMA=1: the active-tile items stage their rows with TMA (cp.async.bulk.tensor.2d, one 128 x 8 box of
// 16-bit cells per 8-row slot, completion on a per-warp mbarrier) wherever all 128 columns of a slot's
// region live in the same ping-pong field; regions split across fields (the neighbour bands' halo columns
// in the other field) keep the per-lane 16 B cp.async.  AM_TMA=0: cp.async only (the A/B baseline).
#ifndef AM_TMA
#define AM_TMA 0  // measured: +2-4% on C4 / C2 / C3; tools/build_variant.sh tma "-DAM_TMA=1"
#endif

namespace am {

Geo make_geo(uint32_t W, uint32_t H, int warp_slots) {
  Geo g{};
  g.W = W;
  g.H = H;
  g.pad = kK;
  g.nbands = (W + kBandUseful - 1) / kBandUseful;
  g.tbands = (W + kTileCols - 1) / kTileCols;
  uint32_t need = g.nbands * kBandUseful + 2 * kK;
  const uint32_t tneed = g.tbands * kTileCols + 2 * kK;
  uint32_t minw = W + 2 * kK;
  if (need < minw) need = minw;
  if (need < tneed) need = tneed;
  g.pitch = (need + 63) / 64 * 64;
  // one wave of warps: pairs of row segments per band
  uint32_t pairs = warp_slots > 0 ? (uint32_t)warp_slots / g.nbands : 1;
  if (pairs < 1) pairs = 1;
  uint32_t seg = (H + 2 * pairs - 1) / (2 * pairs);
  if (seg < 64) seg = 64;
  seg = (seg + 1) & ~1u;
  uint32_t nseg = (H + seg - 1) / seg;
  nseg = (nseg + 1) & ~1u;
  g.seg_len = seg;
  g.nseg = nseg;
  g.nchunks = (H + kTileRows - 1) / kTileRows;
  const uint32_t body = nseg * seg > g.nchunks * kTileRows ? nseg * seg : g.nchunks * kTileRows;
  g.rows = body + 2 * kK;
  return g;
}

// ------------------------------------------------------------------ traits
template <int CB>
struct Cell;

template <>
struct Cell<16> {
  using T = uint16_t;
  static constexpr uint32_t LOW = kLow16x2;
  __device__ __forceinline__ static uint32_t max3(uint32_t a, uint32_t b, uint32_t c) {
    return __vimax3_u16x2(a, b, c);
  }
  // running min over halves of (v - 0x8001) mod 2^16: a-1 for flagged cells,
  // >= 0x7FFF for unflagged ones (obstacles, padding, garbage).
  __device__ __forceinline__ static uint32_t acc_min(uint32_t v, uint32_t acc) {
    return __viaddmin_u16x2(v, 0x7FFF7FFFu, acc);
  }
  __device__ __forceinline__ static uint32_t fold(uint32_t acc) {
    uint32_t lo = acc & 0xFFFFu, hi = acc >> 16;
    return lo < hi ? lo : hi;
  }
  __device__ __forceinline__ static uint32_t vmin(uint32_t a, uint32_t b) { return __vminu2(a, b); }
};

template <>
struct Cell<32> {
  using T = uint32_t;
  static constexpr uint32_t LOW = kLow32;
  __device__ __forceinline__ static uint32_t max3(uint32_t a, uint32_t b, uint32_t c) {
    return __vimax3_u32(a, b, c);
  }
  __device__ __forceinline__ static uint32_t acc_min(uint32_t v, uint32_t acc) {
    return __viaddmin_u32(v, 0x7FFFFFFFu, acc);
  }
  __device__ __forceinline__ static uint32_t fold(uint32_t acc) { return acc; }
  __device__ __forceinline__ static uint32_t vmin(uint32_t a, uint32_t b) { return a < b ? a : b; }
};

// Each working warp calls this exactly once (m = its min, from lane 0); the
// last of `arrivals` to arrive publishes the word (see FlagSink).  PER_CTA:
// every thread of every CTA calls it and one arrival is counted per CTA
// (fewer same-address atomics); otherwise one arrival per working warp.
template <bool PER_CTA>
__device__ __forceinline__ void publish_flag(const FlagSink& f, uint32_t m, uint32_t arrivals) {
  if ((threadIdx.x & 31) == 0 && m != 0xFFFFFFFFu) atomicMin(f.word, m);
  if (!f.host) return;  // uniform
  if (PER_CTA) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x != 0) return;
  } else {
    if ((threadIdx.x & 31) != 0) return;
    __threadfence();
  }
  if (atomicAdd(f.done, 1u) == arrivals - 1) {  // every warp's min is in word
    __threadfence();
    const uint32_t v = atomicExch(f.word, 0xFFFFFFFFu);
    *reinterpret_cast<volatile uint32_t*>(f.host) = v;
    atomicExch(f.done, 0u);
  }
}

// ------------------------------------------------------------- init / misc
// SourceSet rasterisation for the grid rows [row0, row0+H) of a total_h-row
// grid (grid.hpp:78-90): validates every source, marks owned sources in the
// dense mask, and marks owned + halo-band sources in the pitched mask and
// the per-band row flags (a slab recomputes its halo rows inside a block).
__global__ void k_srcmask_rows(Geo g, uint32_t total_h, uint32_t row0, const uint32_t* __restrict__ rc, uint64_t n,
                               uint8_t* __restrict__ dense, const uint8_t* __restrict__ occ,
                               uint8_t* __restrict__ srcmask, uint8_t* __restrict__ rowsrc, int* __restrict__ err) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t r = rc[2 * i], c = rc[2 * i + 1];
  if (r >= total_h || c >= g.W) {
    atomicOr(err, 1);
    return;
  }
  const long local = (long)r - (long)row0;
  if (local >= 0 && local < (long)g.H) {
    if (occ[(size_t)local * g.W + c]) {
      atomicOr(err, 1);
      return;
    }
    dense[(size_t)local * g.W + c] = 1;
  }
  const long arow = local + g.pad;
  if (arow >= 0 && arow < (long)g.rows) {
    const uint32_t ac = c + g.pad;  // allocated column
    srcmask[(size_t)arow * g.pitch + ac] = 1;
    // bands whose streamed columns [b*useful, b*useful + width) hold ac
    const int db0 = ac >= (uint32_t)kBand ? (int)((ac - kBand) / kBandUseful) + 1 : 0;
    for (int b = db0; b <= (int)(ac / kBandUseful) && b < (int)g.nbands; ++b) rowsrc[g.dense_rowsrc(b) + arow] = 1;
    constexpr uint32_t kTW = 32 * kTileWPL;
    const int tb0 = ac >= kTW ? (int)((ac - kTW) / kTileCols) + 1 : 0;
    for (int b = tb0; b <= (int)(ac / kTileCols) && b < (int)g.tbands; ++b) rowsrc[g.tile_rowsrc(b) + arow] = 1;
  }
}

// layer-0 field (activity.hpp:20-21): free = flag|[source], obstacle = 0.
// 8 cells per thread (one 16 B / 32 B store); cells past the grid edge are
// written as padding (0).
template <int CB>
__global__ void k_init(Geo g, const uint8_t* __restrict__ occ, typename Cell<CB>::T* __restrict__ val) {
  const uint32_t c0 = 8 * (blockIdx.x * blockDim.x + threadIdx.x);
  const uint32_t r = blockIdx.y;
  if (c0 >= g.W) return;
  const uint8_t* o = occ + (size_t)r * g.W + c0;
  const size_t i = g.idx(r, c0);
  const uint32_t flag = CB == 16 ? kFlag16 : kFlag32;
  uint32_t v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = (c0 + k < g.W && !o[k]) ? flag : 0u;
  if constexpr (CB == 16) {
    *reinterpret_cast<uint4*>(val + i) =
        make_uint4(v[0] | v[1] << 16, v[2] | v[3] << 16, v[4] | v[5] << 16, v[6] | v[7] << 16);
  } else {
    reinterpret_cast<uint4*>(val + i)[0] = make_uint4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<uint4*>(val + i)[1] = make_uint4(v[4], v[5], v[6], v[7]);
  }
}

// the sources of the grid's rows start at 1 (free cells: validated at grid creation)
template <int CB>
__global__ void k_src_init(Geo g, const uint32_t* __restrict__ rc, uint64_t n, uint32_t row0,
                           typename Cell<CB>::T* __restrict__ val) {
  const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t r = rc[2 * k], c = rc[2 * k + 1];
  if (r < row0 || r >= row0 + g.H) return;
  val[g.idx(r - row0, c)] = (CB == 16 ? kFlag16 : kFlag32) | 1u;
}

// ----------------------------------------------------------- K1+K2 block
template <int CB, int WPL>
struct Rows;

// 16-bit cells: word w of a lane holds cell w of tile A (lo) and of tile B
// (hi); a lane's WPL cells of one tile row are WPL*2 contiguous bytes.
template <int WPL>
struct Rows<16, WPL> {
  static_assert(WPL == 4 || WPL == 8, "lane width");
  __device__ __forceinline__ static void store(const uint32_t (&x)[WPL], uint16_t* pa, uint16_t* pb, bool wa,
                                               bool wb) {
    uint32_t A[WPL / 2], B[WPL / 2];
#pragma unroll
    for (int i = 0; i < WPL / 2; ++i) {
      A[i] = __byte_perm(x[2 * i], x[2 * i + 1], 0x5410);
      B[i] = __byte_perm(x[2 * i], x[2 * i + 1], 0x7632);
    }
    if constexpr (WPL == 8) {
      if (wa) *reinterpret_cast<uint4*>(pa) = make_uint4(A[0], A[1], A[2], A[3]);
      if (wb) *reinterpret_cast<uint4*>(pb) = make_uint4(B[0], B[1], B[2], B[3]);
    } else {
      if (wa) *reinterpret_cast<uint2*>(pa) = make_uint2(A[0], A[1]);
      if (wb) *reinterpret_cast<uint2*>(pb) = make_uint2(B[0], B[1]);
    }
  }
  // words restricted to the valid tiles (an invalid half becomes 0 = unflagged)
  __device__ __forceinline__ static uint32_t valid_bits(bool wa, bool wb) {
    return (wa ? 0x0000FFFFu : 0u) | (wb ? 0xFFFF0000u : 0u);
  }
  __device__ __forceinline__ static void src_words(const uint8_t* sa, const uint8_t* sb, uint32_t (&s)[WPL]) {
    uint32_t a4[2], b4[2];
    if constexpr (WPL == 8) {
      const uint2 A = *reinterpret_cast<const uint2*>(sa), B = *reinterpret_cast<const uint2*>(sb);
      a4[0] = A.x, a4[1] = A.y, b4[0] = B.x, b4[1] = B.y;
    } else {
      a4[0] = *reinterpret_cast<const uint32_t*>(sa), b4[0] = *reinterpret_cast<const uint32_t*>(sb);
      a4[1] = b4[1] = 0;
    }
#pragma unroll
    for (int w = 0; w < WPL; ++w) {
      uint32_t ab = (a4[w / 4] >> (8 * (w % 4))) & 0xFFu, bb = (b4[w / 4] >> (8 * (w % 4))) & 0xFFu;
      s[w] = ab | (bb << 16);
    }
  }
};

template <int WPL>
struct Rows<32, WPL> {
  static_assert(WPL == 4 || WPL == 8, "lane width");
  __device__ __forceinline__ static void store(const uint32_t (&x)[WPL], uint32_t* pa, uint32_t*, bool wa, bool) {
    if (!wa) return;
    reinterpret_cast<uint4*>(pa)[0] = make_uint4(x[0], x[1], x[2], x[3]);
    if constexpr (WPL == 8) reinterpret_cast<uint4*>(pa)[1] = make_uint4(x[4], x[5], x[6], x[7]);
  }
  __device__ __forceinline__ static uint32_t valid_bits(bool wa, bool) { return wa ? 0xFFFFFFFFu : 0u; }
  __device__ __forceinline__ static void src_words(const uint8_t* sa, const uint8_t*, uint32_t (&s)[WPL]) {
    uint32_t a4[2];
    if constexpr (WPL == 8) {
      const uint2 A = *reinterpret_cast<const uint2*>(sa);
      a4[0] = A.x, a4[1] = A.y;
    } else {
      a4[0] = *reinterpret_cast<const uint32_t*>(sa), a4[1] = 0;
    }
#pragma unroll
    for (int w = 0; w < WPL; ++w) s[w] = (a4[w / 4] >> (8 * (w % 4))) & 0xFFu;
  }
};

// Layer j of one streaming step (see stream_step), no sources.
template <int CB, int PH, int WPL>
__device__ __forceinline__ void stream_layer(int j, uint32_t (&x)[WPL], uint32_t (&P0)[kK][WPL],
                                             uint32_t (&P1)[kK][WPL]) {
  using C = Cell<CB>;
  uint32_t v[WPL];
#pragma unroll
  for (int w = 0; w < WPL; ++w) v[w] = C::max3(P0[j][w], P1[j][w], x[w]);
  const uint32_t left = __shfl_up_sync(0xffffffffu, v[WPL - 1], 1);
  const uint32_t right = __shfl_down_sync(0xffffffffu, v[0], 1);
#pragma unroll
  for (int w = 0; w < WPL; ++w) {
    if (PH == 0) P0[j][w] = x[w];
    else P1[j][w] = x[w];
  }
#pragma unroll
  for (int w = 1; w < WPL - 1; ++w) x[w] = C::max3(v[w - 1], v[w], v[w + 1]) & ((PH == 0 ? P1[j][w] : P0[j][w]) | C::LOW);
  x[0] = C::max3(left, v[0], v[1]) & ((PH == 0 ? P1[j][0] : P0[j][0]) | C::LOW);
  x[WPL - 1] = C::max3(v[WPL - 2], v[WPL - 1], right) & ((PH == 0 ? P1[j][WPL - 1] : P0[j][WPL - 1]) | C::LOW);
}

// Steps t (x0, window slot PH 0) and t+1 (x1, slot PH 1) without sources,
// skewed: step t+1's layer j only needs step t's layer j-1, so layer j of
// step t and layer j-1 of step t+1 are independent and issue side by side
// (a warp issues in order; this halves the dependent chain per row pair).
template <int CB, int WPL>
__device__ __forceinline__ void stream_step2(uint32_t (&x0)[WPL], uint32_t (&x1)[WPL], uint32_t (&P0)[kK][WPL],
                                             uint32_t (&P1)[kK][WPL]) {
#pragma unroll
  for (int j = 0; j <= kK; ++j) {
    if (j < kK) stream_layer<CB, 0, WPL>(j, x0, P0, P1);
    if (j >= 1) stream_layer<CB, 1, WPL>(j - 1, x1, P0, P1);
  }
}

// One streaming step: x holds the newly loaded row (layer 0, row t); layer j
// produces row t-j from layer j-1's rows t-j-1, t-j (window) and t-j+1 (x).
// PH selects which window slot holds the older row (it is overwritten).
template <int CB, int PH, bool SRC, int WPL>
__device__ __forceinline__ void stream_step(uint32_t (&x)[WPL], uint32_t (&P0)[kK][WPL],
                                            uint32_t (&P1)[kK][WPL], uint32_t srcbits,
                                            const uint8_t* sA, const uint8_t* sB, size_t pitch, int lane) {
  using C = Cell<CB>;
#pragma unroll
  for (int j = 0; j < kK; ++j) {
    uint32_t v[WPL];
#pragma unroll
    for (int w = 0; w < WPL; ++w) v[w] = C::max3(P0[j][w], P1[j][w], x[w]);
    const uint32_t left = __shfl_up_sync(0xffffffffu, v[WPL - 1], 1);
    const uint32_t right = __shfl_down_sync(0xffffffffu, v[0], 1);
    // the older window row is dead once v exists: it takes this layer's input row
#pragma unroll
    for (int w = 0; w < WPL; ++w) {
      if (PH == 0) P0[j][w] = x[w];
      else P1[j][w] = x[w];
    }
    // interior words first: they do not wait for the shuffles
#pragma unroll
    for (int w = 1; w < WPL - 1; ++w) {
      const uint32_t ctr = PH == 0 ? P1[j][w] : P0[j][w];  // layer j-1, row t-j-1+1
      x[w] = C::max3(v[w - 1], v[w], v[w + 1]) & (ctr | C::LOW);
    }
    x[0] = C::max3(left, v[0], v[1]) & ((PH == 0 ? P1[j][0] : P0[j][0]) | C::LOW);
    x[WPL - 1] = C::max3(v[WPL - 2], v[WPL - 1], right) & ((PH == 0 ? P1[j][WPL - 1] : P0[j][WPL - 1]) | C::LOW);
    if (SRC && ((srcbits >> (j + 1)) & 1u)) {  // row t-(j+1) holds a source (warp-uniform, rare)
      uint32_t s[WPL];
      const size_t off = (size_t)(j + 1) * pitch;
      Rows<CB, WPL>::src_words(sA - off, sB - off, s);
#pragma unroll
      for (int w = 0; w < WPL; ++w) x[w] += s[w];
    }
  }
  (void)lane;
}

// ---- cp.async staging (per-lane 16 / 8 B pieces into shared memory) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// ---- TMA staging (active tiles, 16-bit cells) ----
struct TileMaps {
  CUtensorMap box8[2];  // field 0 / field 1: 2-D (pitch x rows) u16, box = 128 columns x 8 rows (2 KB)
};

struct TmaStage {
  const TileMaps* tm;  // the kernel's __grid_constant__ descriptors
  uint32_t mbA, mbB;   // this warp's mbarriers (shared addresses): rows 0..31 / rows 32..47 of a staging
  uint32_t parity;     // phase parity of the current staging (every staging arrives on both exactly once)
};

#if AM_TMA
constexpr int kSlotRows = 8;
constexpr int kSlotBytes = kSlotRows * 32 * kTileWPL * 2;  // one 8-row slot of the warp's 128-column band

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "MBAR_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra MBAR_WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// one 128-column x 8-row box of a field into shared memory, completing on bar
__device__ __forceinline__ void tma_box8(uint32_t dst, const CUtensorMap* map, uint32_t x, uint32_t y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
// Issue the TMA part of a staging of `nslots` (<= 6) 8-row slots (slot s = staged rows 8s..8s+7, band
// column x, allocated row y0 + 8s) into buf; slot s reads region reg(s).  A region goes through TMA when
// all 32 compute lanes' homes (bit r of `homes`) agree; returns the mask of TMA regions.  Lanes 0-3 arrive
// on mbA (init count 4) and lanes 4-5 on mbB (count 2), each with its own slot's bytes (0 when the slot
// is absent or copied by cp.async), so every staging completes one phase of each barrier and no lane
// waits for another before issuing.
template <class Reg>
__device__ __forceinline__ uint32_t tma_stage(const TmaStage& ts, uint32_t homes, uint8_t* buf, uint32_t x, uint32_t y0,
                                              int nslots, Reg reg) {
  const int lane = threadIdx.x & 31;
  uint32_t tmask = 0, fld = 0;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const uint32_t m = __ballot_sync(0xffffffffu, (homes >> r) & 1u);
    if (m == 0u || m == 0xffffffffu) tmask |= 1u << r;
    if (m) fld |= 1u << r;
  }
  if (lane < 6) {
    const int r = lane < nslots ? reg(lane) : 0;
    const bool tma = lane < nslots && ((tmask >> r) & 1u);
    const uint32_t bar = lane < 4 ? ts.mbA : ts.mbB;
    // the previous item's generic-proxy reads of buf (ordered by the caller's __syncwarp) come first
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_expect(bar, tma ? kSlotBytes : 0u);
    if (tma)
      tma_box8(smem_u32(buf) + lane * kSlotBytes, &ts.tm->box8[(fld >> r) & 1u], x, y0 + kSlotRows * lane, bar);
  }
  return tmask;
}
#endif  // AM_TMA

#ifndef AM_STAGES
#define AM_STAGES 4
#endif
#ifndef AM_ST128
#define AM_ST128 0  // 1: tile outputs as 16 B stores (lane pairs swap halves)
#endif
#ifndef AM_TILE_STAGES
#define AM_TILE_STAGES 4
#endif
#ifndef AM_SKEW
#define AM_SKEW 1
#endif
#ifndef AM_QUARTERS
#define AM_QUARTERS 1  // light blocks run two quarter items per tile
#endif
#ifndef AM_PAIRS
#define AM_PAIRS 0  // 1: heavy blocks run two whole tiles per item (C4 -1.4%, C5 +50%: source tiles serialise)
#endif
#ifndef AM_PAIR_MIN4
#define AM_PAIR_MIN4 6  // pairs from this many quarter warp slots of tiles on (below: halves, shorter latency)
#endif
#ifndef AM_QUARTER_SLOTS
#define AM_QUARTER_SLOTS 1  // quarter items while they fit this many times into the warp slots
#endif


constexpr int kStages = AM_STAGES;                 // rows in flight per warp (dense sweep)
constexpr int kTileStages = AM_TILE_STAGES;        // rows in flight per warp (active tiles: few warps per SM)
// one stage = one u32 row of the warp's band, or the A+B pair of u16 rows
template <int WPL>
constexpr int stage_bytes() { return 32 * WPL * 4; }
constexpr int kWarpsPerCta = kBlockThreads / 32;
constexpr int kBlockSmem = kWarpsPerCta * kStages * stage_bytes<kWPL>();
constexpr int kTileWarpSmemRing = kTileStages * stage_bytes<kTileWPL>();

template <int CB, int WPL>
__device__ __forceinline__ void stage_words(const uint8_t* stage, int lane, uint32_t (&x)[WPL]) {
  constexpr int kLaneBytes = WPL * CB / 8;  // one tile row of this lane
  uint32_t A[4], B[4];
  if constexpr (CB == 16) {
    if constexpr (WPL == 8) {
      const uint4 a = reinterpret_cast<const uint4*>(stage)[lane];
      const uint4 b = reinterpret_cast<const uint4*>(stage + 32 * kLaneBytes)[lane];
      A[0] = a.x, A[1] = a.y, A[2] = a.z, A[3] = a.w, B[0] = b.x, B[1] = b.y, B[2] = b.z, B[3] = b.w;
    } else {
      const uint2 a = reinterpret_cast<const uint2*>(stage)[lane];
      const uint2 b = reinterpret_cast<const uint2*>(stage + 32 * kLaneBytes)[lane];
      A[0] = a.x, A[1] = a.y, B[0] = b.x, B[1] = b.y;
    }
#pragma unroll
    for (int i = 0; i < WPL / 2; ++i) {
      x[2 * i] = __byte_perm(A[i], B[i], 0x5410);
      x[2 * i + 1] = __byte_perm(A[i], B[i], 0x7632);
    }
  } else {
    const uint4 a = reinterpret_cast<const uint4*>(stage + lane * kLaneBytes)[0];
    x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w;
    if constexpr (WPL == 8) {
      const uint4 b = reinterpret_cast<const uint4*>(stage + lane * kLaneBytes)[1];
      x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
    }
  }
}

#ifndef AM_BLOCK_MINB
#define AM_BLOCK_MINB 3  // CTAs per SM the register budget is sized for (12 warps, <= 170 regs)
#endif
// SLAB=false: rows past the grid are padding (unflagged centres compute to
// unflagged values), so they may be stored and folded into the flag
// unchanged.  SLAB=true: the rows below the slab are a neighbour's halo
// (flagged data) and must be neither stored nor counted.
// One work item per warp: tile A = band bA, allocated rows [rA, rA+rows+2K)
// (rows of output), tile B likewise in the hi halves (16-bit cells; 32-bit
// cells process A only).  Returns the warp's running u16x2/u32 minimum of
// (a-1) over its stored cells (lo half = A, hi half = B).
// LAG (active-tile mode): lagw[0..2] are this lane's per-half lags of the
// tiles it reads above / inside / below the item (lane 0 and 31 read the
// neighbouring bands); they are added to covered cells as rows arrive.
template <int CB>
__device__ __forceinline__ uint32_t add_lag(uint32_t w, uint32_t lagw);
// Field selection (active-tile mode): the two ping-pong fields are `in` and
// `in + delta`; bit r of `homes` (r = 0 above, 1 inside, 2 below the item)
// says tile A's region r is read from the second field, bits 3..5 the same
// for B, bit 6 / 7 that A's / B's output goes to `out + delta`.
template <int CB, bool SLAB, bool LAG = false, int ST = kStages, int WPL = kWPL, int RS = ST * stage_bytes<WPL>()>
__device__ __forceinline__ uint32_t stream_item(const Geo& g, const typename Cell<CB>::T* __restrict__ in,
                                                typename Cell<CB>::T* __restrict__ out,
                                                const uint8_t* __restrict__ srcmask,
                                                const uint8_t* __restrict__ rfA, const uint8_t* __restrict__ rfB,
                                                uint32_t bA, uint32_t rA,
                                                uint32_t bB, uint32_t rB, uint32_t rows, bool hasB,
                                                uint32_t lag0 = 0, uint32_t lag1 = 0, uint32_t lag2 = 0,
                                                ptrdiff_t delta = 0, uint32_t homes = 0, uint32_t* edge_min = nullptr) {
  uint32_t accTop = 0xFFFFFFFFu, accBot = 0xFFFFFFFFu;  // LAG: minima over the first / last kK output rows
  using C = Cell<CB>;
  using T = typename C::T;
  const int lane = threadIdx.x & 31;
  constexpr uint32_t kUseful = 32 * WPL - 2 * kK;  // useful columns of the band
  const uint32_t colA = bA * kUseful + lane * WPL;   // allocated column of this lane's first cell
  const uint32_t colB = bB * kUseful + lane * WPL;
  const uint32_t T_steps = rows + 2 * kK;
  const size_t pitch = g.pitch;

  const T* pA = in + (size_t)rA * pitch + colA;
  const T* pB = in + (size_t)rB * pitch + colB;
  T* oA = out + (size_t)rA * pitch + colA + ((homes >> 6) & 1u ? delta : 0);  // output row of step t: rA + t - kK
  T* oB = out + (size_t)rB * pitch + colB + ((homes >> 7) & 1u ? delta : 0);
  const uint8_t* sA = srcmask + (size_t)rA * pitch + colA;
  const uint8_t* sB = srcmask + (size_t)rB * pitch + colB;
  const bool store_lane = lane >= kK / WPL && lane < 32 - kK / WPL;

  uint32_t P0[kK][WPL], P1[kK][WPL];
#pragma unroll
  for (int j = 0; j < kK; ++j)
#pragma unroll
    for (int w = 0; w < WPL; ++w) P0[j][w] = P1[j][w] = 0u;
  uint32_t acc = 0xFFFFFFFFu;
  uint32_t srcbits = 0;

  // Each lane streams its own 16-32 B of every row through a private kStages
  // deep shared-memory ring with cp.async (LDGSTS): the copies run
  // kStages-1 rows ahead without holding registers, and since no lane reads
  // another lane's slot no barrier or fence is needed.
  extern __shared__ __align__(128) uint8_t smem_raw[];
  constexpr int kSB = stage_bytes<WPL>();
  constexpr int kLaneBytes = WPL * CB / 8;  // one tile row of this lane
  uint8_t* ring = smem_raw + (threadIdx.x >> 5) * RS;  // RS: bytes of shared memory per warp
  auto issue = [&](uint32_t step) {
    uint8_t* dst = ring + (step % ST) * kSB;
    if (step < T_steps) {
      const size_t off = (size_t)step * pitch;
      const T* a = pA + off;
      const T* b = pB + off;
      if constexpr (LAG) {
        const uint32_t reg = step < (uint32_t)kK ? 0u : (step < kK + rows ? 1u : 2u);
        if ((homes >> reg) & 1u) a += delta;
        if ((homes >> (3 + reg)) & 1u) b += delta;
      }
      if constexpr (kLaneBytes == 8) {
        cp_async8(dst + lane * 8, a);
        cp_async8(dst + 32 * 8 + lane * 8, b);
      } else if constexpr (CB == 16) {
        cp_async16(dst + lane * 16, a);
        cp_async16(dst + 32 * 16 + lane * 16, b);
      } else {
        cp_async16(dst + lane * kLaneBytes, a);
        if constexpr (kLaneBytes == 32) cp_async16(dst + lane * 32 + 16, a + 16 / sizeof(T));
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) issue(s);
  // source-row flags arrive as a 32-row ballot window, loaded one window ahead
  auto row_flag = [&](uint32_t step) -> uint32_t {
    if (step >= T_steps) return 0u;
    uint32_t f = rfA[rA + step];
    if (CB == 16) f |= rfB[rB + step];
    return f;
  };
  uint32_t flag_lane = row_flag(lane), flag_win = 0;
  // Output row handling of step tt (x = the row after the last layer).
  auto emit = [&](uint32_t tt, const uint32_t (&x)[WPL]) {
    if (!(tt >= 2 * kK && tt < 2 * kK + rows && store_lane)) return;
    const size_t roff = (size_t)tt * pitch;
    if constexpr (LAG) {  // also track the first / last kK output rows (tile edge regions)
      Rows<CB, WPL>::store(x, oA + roff - (size_t)kK * pitch, oB + roff - (size_t)kK * pitch, true, hasB);
      uint32_t rm = 0xFFFFFFFFu;
#pragma unroll
      for (int w = 0; w < WPL; ++w) rm = C::acc_min(x[w], rm);
      acc = C::vmin(acc, rm);
      const uint32_t orow = tt - 2 * kK;
      if (orow < (uint32_t)kK) accTop = C::vmin(accTop, rm);
      if (orow >= rows - kK) accBot = C::vmin(accBot, rm);
    } else if constexpr (!SLAB) {
      Rows<CB, WPL>::store(x, oA + roff - (size_t)kK * pitch, oB + roff - (size_t)kK * pitch, true, hasB);
#pragma unroll
      for (int w = 0; w < WPL; ++w) acc = C::acc_min(x[w], acc);
    } else {
      const uint32_t orow = tt - 2 * kK;
      const bool wa = rA + orow < g.H, wb = rB + orow < g.H;
      Rows<CB, WPL>::store(x, oA + roff - (size_t)kK * pitch, oB + roff - (size_t)kK * pitch, wa, wb);
      const uint32_t keep = Rows<CB, WPL>::valid_bits(wa, wb);
#pragma unroll
      for (int w = 0; w < WPL; ++w) acc = C::acc_min(x[w] & keep, acc);
    }
  };
  constexpr uint32_t kInFlight = ((1u << kK) - 1u) << 1;  // rows t-1 .. t-kK of a step's srcbits
  // Two steps per iteration.  On the common path (no source row in flight)
  // both steps sit in one branch-free block, so the scheduler overlaps step
  // t+1's early layers with step t's late ones (they are independent).
  for (uint32_t t = 0; t < T_steps; t += 2) {
    if ((t & 31u) == 0) {
      flag_win = __ballot_sync(0xffffffffu, flag_lane != 0u);
      flag_lane = row_flag(t + 32 + lane);
    }
    uint32_t x0[WPL], x1[WPL];
    issue(t + ST - 1);  // refills the slot consumed by the previous step
    asm volatile("cp.async.wait_group %0;" ::"n"(ST - 1) : "memory");
    stage_words<CB, WPL>(ring + (t % ST) * kSB, lane, x0);
    issue(t + ST);  // the slot of row t, now in registers
    asm volatile("cp.async.wait_group %0;" ::"n"(ST - 1) : "memory");
    stage_words<CB, WPL>(ring + ((t + 1) % ST) * kSB, lane, x1);
    if constexpr (LAG) {
      auto lag_of = [&](uint32_t tt) { return tt < (uint32_t)kK ? lag0 : (tt < kK + rows ? lag1 : lag2); };
      const uint32_t l0w = lag_of(t), l1w = lag_of(t + 1);
      if (__any_sync(0xffffffffu, (l0w | l1w) != 0u)) {
#pragma unroll
        for (int w = 0; w < WPL; ++w) {
          x0[w] = add_lag<CB>(x0[w], l0w);
          x1[w] = add_lag<CB>(x1[w], l1w);
        }
      }
    }
    const uint32_t sb0 = (srcbits << 1) | ((flag_win >> (t & 31u)) & 1u);
    const uint32_t sb1 = (sb0 << 1) | ((flag_win >> ((t + 1) & 31u)) & 1u);
    srcbits = sb1;
    const size_t r0 = (size_t)t * pitch, r1 = r0 + pitch;
    // only steps that touch a source row pay for the +1 (warp-uniform)
    if (__any_sync(0xffffffffu, ((sb0 | sb1) & kInFlight) != 0u)) {
      stream_step<CB, 0, true, WPL>(x0, P0, P1, sb0, sA + r0, sB + r0, pitch, lane);
      stream_step<CB, 1, true, WPL>(x1, P0, P1, sb1, sA + r1, sB + r1, pitch, lane);
    } else {
#if AM_SKEW
      stream_step2<CB, WPL>(x0, x1, P0, P1);
#else
      stream_step<CB, 0, false, WPL>(x0, P0, P1, sb0, sA + r0, sB + r0, pitch, lane);
      stream_step<CB, 1, false, WPL>(x1, P0, P1, sb1, sA + r1, sB + r1, pitch, lane);
#endif
    }
    emit(t, x0);
    emit(t + 1, x1);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if constexpr (LAG) {
    edge_min[0] = accTop;
    edge_min[1] = accBot;
  }
  return acc;
}

// ---- active tiles, 16-bit cells: one tile per warp, staged whole ---------
//
// The two u16 halves of every word carry the tile's upper half (rows 0-15,
// lo) and lower half (rows 16-31, hi): both stream 16 + 2K = 32 steps, so an
// item is short (latency) and the block has one item per active tile (warps
// to hide it).  The tile's rows -8..39 (its own 32 + K above + K below) are
// staged in shared memory up front with 16 B cp.async.cg (lanes 0-15 copy
// one 256 B row, 16-31 the next; two commit groups), then the steps run in
// four compile-time phases: which region each half reads (lag) and which
// output minima a step feeds.  Items whose rows hold a source take the
// general stream_item path (same halves).
constexpr int kHalfRows = kTileRows / 2;                   // rows per half
constexpr int kTileSteps = kHalfRows + 2 * kK;             // steps per item
constexpr int kStageRows = kTileRows + 2 * kK;             // rows staged (-K .. kTileRows+K-1)
constexpr int kTileRowBytes = 32 * kTileWPL * 2;           // one u16 row of the warp's band
constexpr int kTileBufBytes = kStageRows * kTileRowBytes;  // 12 KB
constexpr int kPairSteps = kTileRows + 2 * kK;             // steps of a pair item (48)
static_assert(kTileWPL == 4, "the staged item path loads 8 B per lane and tile row");
static_assert(kHalfRows == 2 * kK, "phase layout: 16-row halves with K = 8");
// heavy blocks, pairs of tiles (see tile_pair16): 32 staged rows of A + B (a ring over 48 steps)
constexpr int kPairRowBytes = 2 * kTileRowBytes;        // tile A's row, then tile B's row
constexpr int kPairSlots = kTileRows;                   // ring slots
constexpr int kPairBufBytes = kPairSlots * kPairRowBytes;  // 16 KB
constexpr int kTileWarpSmem0 = kTileBufBytes > kTileWarpSmemRing ? kTileBufBytes : kTileWarpSmemRing;
constexpr int kTileWarpSmem = AM_PAIRS && kPairBufBytes > kTileWarpSmem0 ? kPairBufBytes : kTileWarpSmem0;
constexpr int kTileSmem = kTileThreads / 32 * kTileWarpSmem;  // dynamic shared memory of k_block_tiles

enum { kOutNone = 0, kOutTop = 1, kOutBot = 2, kOutMid = 3 };  // kOutMid: outputs feed acc only

// Steps [s0, s1): the upper half reads staged row s, the lower half row s+16.
// HI: rows between the two u16 streams (16 for tile halves, 8 for quarter items).
template <int OUT, int HI = kHalfRows>
__device__ __forceinline__ void tile_phase(const uint8_t* buf, int s0, int s1, uint32_t lagw, bool lag,
                                           uint32_t (&P0)[kK][4], uint32_t (&P1)[kK][4], uint16_t*& oA,
                                           uint16_t*& oB, size_t pitch, bool st, uint32_t& acc, uint32_t& acc_edge) {
  using C = Cell<16>;
  constexpr int kRow = HI < 0 ? kPairRowBytes : kTileRowBytes;   // HI < 0: pair buffer (see fill_pair)
  constexpr int kB = HI < 0 ? kTileRowBytes : HI * kTileRowBytes;  // the hi stream runs HI rows further down
  auto words = [](uint2 a, uint2 b, uint32_t (&x)[4]) {
    x[0] = __byte_perm(a.x, b.x, 0x5410);
    x[1] = __byte_perm(a.x, b.x, 0x7632);
    x[2] = __byte_perm(a.y, b.y, 0x5410);
    x[3] = __byte_perm(a.y, b.y, 0x7632);
  };
  auto emit = [&](const uint32_t (&x)[4]) {
#if AM_ST128
    // 16 B stores: lane pairs swap halves, the even lane writes both lanes' 8 cells of row A, the odd lane
    // both lanes' cells of row B (halo pairs 0-1 / 30-31 store nothing: `st` is uniform per pair)
    {
      const uint32_t a0 = __byte_perm(x[0], x[1], 0x5410), a1 = __byte_perm(x[2], x[3], 0x5410);
      const uint32_t b0 = __byte_perm(x[0], x[1], 0x7632), b1 = __byte_perm(x[2], x[3], 0x7632);
      const bool odd = threadIdx.x & 1;
      const uint32_t r0 = __shfl_xor_sync(0xffffffffu, odd ? a0 : b0, 1);
      const uint32_t r1 = __shfl_xor_sync(0xffffffffu, odd ? a1 : b1, 1);
      if (st) {
        if (!odd) *reinterpret_cast<uint4*>(oA) = make_uint4(a0, a1, r0, r1);
        else *reinterpret_cast<uint4*>(oB - 4) = make_uint4(r0, r1, b0, b1);
      }
    }
#else
    if (st) {
      *reinterpret_cast<uint2*>(oA) = make_uint2(__byte_perm(x[0], x[1], 0x5410), __byte_perm(x[2], x[3], 0x5410));
      *reinterpret_cast<uint2*>(oB) = make_uint2(__byte_perm(x[0], x[1], 0x7632), __byte_perm(x[2], x[3], 0x7632));
    }
#endif
    oA += pitch;
    oB += pitch;
    uint32_t rm = 0xFFFFFFFFu;
#pragma unroll
    for (int w = 0; w < 4; ++w) rm = C::acc_min(x[w], rm);
    acc = C::vmin(acc, rm);
    if (OUT != kOutMid) acc_edge = C::vmin(acc_edge, rm);
  };
#pragma unroll 1
  for (int s = s0; s < s1; s += 2) {
    const uint8_t* r = buf + (HI < 0 ? s % kPairSlots : s) * kRow;
    uint32_t x0[4], x1[4];
    words(*reinterpret_cast<const uint2*>(r), *reinterpret_cast<const uint2*>(r + kB), x0);
    words(*reinterpret_cast<const uint2*>(r + kRow), *reinterpret_cast<const uint2*>(r + kB + kRow), x1);
    if (lag) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        x0[w] = add_lag<16>(x0[w], lagw);
        x1[w] = add_lag<16>(x1[w], lagw);
      }
    }
#if AM_SKEW
    stream_step2<16, 4>(x0, x1, P0, P1);
#else
    stream_step<16, 0, false, 4>(x0, P0, P1, 0u, nullptr, nullptr, 0, 0);
    stream_step<16, 1, false, 4>(x1, P0, P1, 0u, nullptr, nullptr, 0, 0);
#endif
    if constexpr (OUT != kOutNone) {
      emit(x0);
      emit(x1);
    }
  }
}

// Pipeline fill (steps 0 .. 2K-1) without the work that cannot reach an
// output.  Layer j+1 of row t-j-1 is produced at step t; the K-layer result
// is needed on rows [K, steps) only, so layer j+1 is needed on rows >= j+1,
// i.e. from step 2j+2 on.  At steps 2j and 2j+1 layer j's input rows only
// have to enter the window (P0 / P1 slot of the step's parity); before that
// the iteration does nothing.  Step pair m (steps 2m, 2m+1) therefore runs
// iterations j < m, stores j == m and skips the rest: 56 of the 128 layer
// updates of the fill (a tile item: 184 instead of 256 per u16 stream).
#ifndef AM_TRIM
#define AM_TRIM 1
#endif
#ifndef AM_SPEC_LIST
#define AM_SPEC_LIST 1
#endif
#ifndef AM_FIN_BATCH
#define AM_FIN_BATCH 1
#endif
#ifndef AM_STATIC_FIRST
#define AM_STATIC_FIRST 1
#endif
// HI: rows between the lo and hi streams of a staged buffer of kTileRowBytes rows; or HI < 0: pair
// buffers (rows of kPairRowBytes, the hi stream's row right after the lo stream's)
template <int M, int HI>
__device__ __forceinline__ void fill_pair(const uint8_t* buf, uint32_t lagw, bool lag, uint32_t (&P0)[kK][4],
                                          uint32_t (&P1)[kK][4]) {
  constexpr int kRow = HI < 0 ? kPairRowBytes : kTileRowBytes;
  constexpr int kB = HI < 0 ? kTileRowBytes : HI * kTileRowBytes;
  const uint8_t* r = buf + 2 * M * kRow;
  const uint2 a0 = *reinterpret_cast<const uint2*>(r), b0 = *reinterpret_cast<const uint2*>(r + kB);
  const uint2 a1 = *reinterpret_cast<const uint2*>(r + kRow), b1 = *reinterpret_cast<const uint2*>(r + kB + kRow);
  uint32_t x0[4] = {__byte_perm(a0.x, b0.x, 0x5410), __byte_perm(a0.x, b0.x, 0x7632),
                    __byte_perm(a0.y, b0.y, 0x5410), __byte_perm(a0.y, b0.y, 0x7632)};
  uint32_t x1[4] = {__byte_perm(a1.x, b1.x, 0x5410), __byte_perm(a1.x, b1.x, 0x7632),
                    __byte_perm(a1.y, b1.y, 0x5410), __byte_perm(a1.y, b1.y, 0x7632)};
  if (lag) {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      x0[w] = add_lag<16>(x0[w], lagw);
      x1[w] = add_lag<16>(x1[w], lagw);
    }
  }
#pragma unroll
  for (int j = 0; j <= M + 1; ++j) {  // skewed as in stream_step2
    if (j < M) {
      stream_layer<16, 0, 4>(j, x0, P0, P1);
    } else if (j == M) {
#pragma unroll
      for (int w = 0; w < 4; ++w) P0[M][w] = x0[w];
    }
    if (j >= 1 && j - 1 < M) {
      stream_layer<16, 1, 4>(j - 1, x1, P0, P1);
    } else if (j >= 1 && j - 1 == M) {
#pragma unroll
      for (int w = 0; w < 4; ++w) P1[M][w] = x1[w];
    }
  }
}

// steps [0, K) read with lag a, [K, 2K) with lag b
template <int HI>
__device__ __forceinline__ void tile_fill(const uint8_t* buf, uint32_t lag_a, bool la, uint32_t lag_b, bool lb,
                                          uint32_t (&P0)[kK][4], uint32_t (&P1)[kK][4]) {
  static_assert(kK == 8, "fill schedule written for K = 8");
  fill_pair<0, HI>(buf, lag_a, la, P0, P1);
  fill_pair<1, HI>(buf, lag_a, la, P0, P1);
  fill_pair<2, HI>(buf, lag_a, la, P0, P1);
  fill_pair<3, HI>(buf, lag_a, la, P0, P1);
  fill_pair<4, HI>(buf, lag_b, lb, P0, P1);
  fill_pair<5, HI>(buf, lag_b, lb, P0, P1);
  fill_pair<6, HI>(buf, lag_b, lb, P0, P1);
  fill_pair<7, HI>(buf, lag_b, lb, P0, P1);
}

// Tile (band b, chunk c) without source rows; lw / homes: this lane's lag and
// home field of the regions above / inside / below the tile (bits 0-2), bit
// 6 = output field.  Returns the min over covered output cells of a-1 (lo =
// upper half, hi = lower half); edge[0] / edge[1]: the same over the first /
// last kK rows of each half (use lo of [0] and hi of [1]).
// Issues the copies of the tile's rows into buf (two commit groups); the
// caller may still decide not to run the staged path (then waits them out).
__device__ __forceinline__ void tile_stage16(const Geo& g, const uint16_t* __restrict__ f0, ptrdiff_t delta,
                                             uint32_t b, uint32_t c, uint32_t homes, uint8_t* buf,
                                             const TmaStage& ts) {
  const int lane = threadIdx.x & 31;
  const size_t pitch = g.pitch;
  __syncwarp();  // every lane is done reading the previous item's rows
  uint32_t tmask = 0;
#if AM_TMA
  // slots: staged rows 0-7 above the tile, 8-39 inside, 40-47 below
  tmask = tma_stage(ts, homes, buf, b * kTileCols, c * kTileRows, kStageRows / kSlotRows,
                    [](int sl) { return sl == 0 ? 0 : (sl == kStageRows / kSlotRows - 1 ? 2 : 1); });
#else
  (void)ts;
#endif
  {
    // the 8 cells this lane copies belong to compute lanes 2*(lane&15) and +1: their band's homes
    const uint32_t ch = __shfl_sync(0xffffffffu, homes, (2 * lane) & 31);
    const int half = lane >> 4;
    const uint32_t col = b * kTileCols + (lane & 15) * 8;
    const uint16_t* base[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) base[r] = f0 + (((ch >> r) & 1u) ? delta : 0) + (size_t)c * kTileRows * pitch + col;
    uint8_t* dst = buf + (lane & 15) * 16;
#pragma unroll
    for (int k = 0; k < kStageRows / 2; ++k) {
      const int row = 2 * k + half;  // staged row = tile row + kK
      const int reg = row < kK ? 0 : (row < kK + kTileRows ? 1 : 2);
      if (!((tmask >> reg) & 1u)) cp_async16(dst + row * kTileRowBytes, base[reg] + (size_t)row * pitch);
      if (k == kHalfRows - 1) asm volatile("cp.async.commit_group;" ::: "memory");  // rows 0..31: phases 0-1
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
}

__device__ __forceinline__ uint32_t tile_item16(const Geo& g, uint16_t* __restrict__ f0, ptrdiff_t delta, uint32_t b,
                                                uint32_t c, const uint32_t (&lw)[3], uint32_t homes,
                                                uint32_t* edge, const uint8_t* buf, const TmaStage& ts) {
  const int lane = threadIdx.x & 31;
  const size_t pitch = g.pitch;
  uint32_t P0[kK][4], P1[kK][4];
#if !AM_TRIM
#pragma unroll
  for (int j = 0; j < kK; ++j)
#pragma unroll
    for (int w = 0; w < 4; ++w) P0[j][w] = P1[j][w] = 0u;
#endif
  uint32_t acc = 0xFFFFFFFFu, accTop = 0xFFFFFFFFu, accBot = 0xFFFFFFFFu;
  const ptrdiff_t od = ((homes >> 6) & 1u) ? delta : 0;
  uint16_t* oA = f0 + od + (size_t)(c * kTileRows + kK) * pitch + b * kTileCols + lane * kTileWPL;  // tile row 0
  uint16_t* oB = oA + (size_t)kHalfRows * pitch;                                                 // tile row 16
  const bool st = lane >= kK / kTileWPL && lane < 32 - kK / kTileWPL;
  const uint8_t* rb = buf + lane * 8;
  const uint32_t lag_up = lw[0] | lw[1] << 16, lag_in = lw[1] | lw[1] << 16, lag_dn = lw[1] | lw[2] << 16;
  const bool l_up = __any_sync(0xffffffffu, lag_up != 0u), l_in = __any_sync(0xffffffffu, lag_in != 0u),
             l_dn = __any_sync(0xffffffffu, lag_dn != 0u);
  asm volatile("cp.async.wait_group 1;" ::: "memory");
#if AM_TMA
  mbar_wait(ts.mbA, ts.parity);
#else
  (void)ts;
#endif
  __syncwarp();
#if AM_TRIM
  tile_fill<kHalfRows>(rb, lag_up, l_up, lag_in, l_in, P0, P1);
#else
  tile_phase<kOutNone>(rb, 0, kK, lag_up, l_up, P0, P1, oA, oB, pitch, st, acc, accTop);
  tile_phase<kOutNone>(rb, kK, 2 * kK, lag_in, l_in, P0, P1, oA, oB, pitch, st, acc, accTop);
#endif
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#if AM_TMA
  mbar_wait(ts.mbB, ts.parity);
#endif
  __syncwarp();
  tile_phase<kOutTop>(rb, 2 * kK, 3 * kK, lag_in, l_in, P0, P1, oA, oB, pitch, st, acc, accTop);
  tile_phase<kOutBot>(rb, 3 * kK, kTileSteps, lag_dn, l_dn, P0, P1, oA, oB, pitch, st, acc, accBot);
  if (!st) acc = accTop = accBot = 0xFFFFFFFFu;  // halo lanes hold no output
  edge[0] = accTop;
  edge[1] = accBot;
  return acc;
}

// ---- heavy blocks: pairs of tiles (lo = tile A, hi = tile B) ----------------
//
// With more active tiles than warps the kernel is throughput bound, and the
// halves layout pays 2 x 2K halo rows per 32-row tile.  A pair item streams
// two whole tiles side by side instead (any two listed tiles: the u16 streams
// are independent): 32 + 2K = 48 steps for 64 tile rows, 156 instead of 184
// layer updates per tile after the trimmed fill.  Staged rows live in a
// 32-slot ring (16 KB per warp): rows 0-31 up front, rows 32-47 into the slots
// of rows 0-15 once the fill has consumed them.
// copies staged rows [r0, r1) (staged row = tile row + kK) into ring slot row % kPairSlots;
// lanes 0-15 copy tile A's 256 B of the row, lanes 16-31 tile B's
__device__ __forceinline__ void pair_stage(const Geo& g, const uint16_t* __restrict__ f0, ptrdiff_t delta,
                                           const uint16_t* baseA, const uint16_t* baseB, uint32_t homesA,
                                           uint32_t homesB, uint8_t* buf, int r0, int r1) {
  const int lane = threadIdx.x & 31;
  const size_t pitch = g.pitch;
  const uint32_t hA = __shfl_sync(0xffffffffu, homesA, (2 * lane) & 31);
  const uint32_t hB = __shfl_sync(0xffffffffu, homesB, (2 * lane) & 31);
  const uint32_t ch = lane < 16 ? hA : hB;
  const uint16_t* base = (lane < 16 ? baseA : baseB) + (lane & 15) * 8;  // tile row -kK, this lane's 8 cells
  uint8_t* dst = buf + (lane >> 4) * kTileRowBytes + (lane & 15) * 16;
  for (int row = r0; row < r1; ++row) {
    const int reg = row < kK ? 0 : (row < kK + kTileRows ? 1 : 2);
    cp_async16(dst + (row % kPairSlots) * kPairRowBytes, base + (((ch >> reg) & 1u) ? delta : 0) + (size_t)row * pitch);
  }
}

// lwA / lwB: this lane's lag of the regions above / inside / below tile A / B; homes bit 6: output field.
// Returns the min over covered output cells of a-1 (lo = A, hi = B); edge[0] / edge[1]: the same over the
// tiles' first / last kK rows.  The caller has issued pair_stage of rows [0, 16) and [16, 32) (two groups).
__device__ __forceinline__ uint32_t tile_pair16(const Geo& g, uint16_t* __restrict__ f0, ptrdiff_t delta,
                                                const uint16_t* baseA, const uint16_t* baseB, const uint32_t (&lwA)[3],
                                                const uint32_t (&lwB)[3], uint32_t homesA, uint32_t homesB,
                                                uint16_t* oA, uint16_t* oB, uint32_t* edge, uint8_t* buf) {
  const int lane = threadIdx.x & 31;
  const size_t pitch = g.pitch;
  uint32_t P0[kK][4], P1[kK][4];
  uint32_t acc = 0xFFFFFFFFu, accTop = 0xFFFFFFFFu, accBot = 0xFFFFFFFFu, dummy = 0u;
  const bool st = lane >= kK / kTileWPL && lane < 32 - kK / kTileWPL;
  const uint8_t* rb = buf + lane * 8;
  const uint32_t lag_up = lwA[0] | lwB[0] << 16, lag_in = lwA[1] | lwB[1] << 16, lag_dn = lwA[2] | lwB[2] << 16;
  const bool l_up = __any_sync(0xffffffffu, lag_up != 0u), l_in = __any_sync(0xffffffffu, lag_in != 0u),
             l_dn = __any_sync(0xffffffffu, lag_dn != 0u);
  asm volatile("cp.async.wait_group 1;" ::: "memory");
  __syncwarp();
  tile_fill<-1>(rb, lag_up, l_up, lag_in, l_in, P0, P1);  // steps 0-15: staged rows 0-15
  __syncwarp();                                            // every lane is done with slots 0-15
  pair_stage(g, f0, delta, baseA, baseB, homesA, homesB, buf, kPairSlots, kPairSteps);
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 1;" ::: "memory");  // rows 16-31
  __syncwarp();
  tile_phase<kOutTop, -1>(rb, 2 * kK, 3 * kK, lag_in, l_in, P0, P1, oA, oB, pitch, st, acc, accTop);
  tile_phase<kOutMid, -1>(rb, 3 * kK, 4 * kK, lag_in, l_in, P0, P1, oA, oB, pitch, st, acc, dummy);
  asm volatile("cp.async.wait_group 0;" ::: "memory");  // rows 32-47
  __syncwarp();
  tile_phase<kOutMid, -1>(rb, 4 * kK, 5 * kK, lag_in, l_in, P0, P1, oA, oB, pitch, st, acc, dummy);
  tile_phase<kOutBot, -1>(rb, 5 * kK, kPairSteps, lag_dn, l_dn, P0, P1, oA, oB, pitch, st, acc, accBot);
  if (!st) acc = accTop = accBot = 0xFFFFFFFFu;  // halo lanes hold no output
  edge[0] = accTop;
  edge[1] = accBot;
  return acc;
}

// ---- light blocks: quarter items (two warps per tile) ---------------------
//
// When a block has fewer tiles than half the warp slots it is bound by one
// item's latency, not by throughput.  Each tile then runs as two items of 16
// rows (half = 0: rows 0-15, 1: rows 16-31), whose u16 streams carry 8 rows
// each: 8 + 2K = 24 steps instead of 32.  Both items of a tile do the tile's
// bookkeeping (state, pushes: idempotent), each with the edge regions it
// holds.  Staged rows: the 32 rows -8 .. 23 around the item (8 KB).
constexpr int kQuarterRows = kHalfRows / 2;             // rows per u16 stream
constexpr int kQuarterSteps = kQuarterRows + 2 * kK;    // 24
constexpr int kQuarterStage = kHalfRows + 2 * kK;       // 32 rows staged
static_assert(kQuarterRows == kK, "quarter phase layout assumes 8-row streams with K = 8");

__device__ __forceinline__ uint32_t tile_quarter16(const Geo& g, uint16_t* __restrict__ f0, ptrdiff_t delta,
                                                   uint32_t b, uint32_t c, uint32_t half, const uint32_t (&lw)[3],
                                                   uint32_t homes, uint32_t* edge, uint8_t* buf, TmaStage& ts) {
  const int lane = threadIdx.x & 31;
  const size_t pitch = g.pitch;
  const uint32_t r0 = half * kHalfRows;  // first tile row of the item
  __syncwarp();  // every lane is done reading the previous item's rows
  uint32_t tmask = 0;
#if AM_TMA
  // slots (staged rows 8s..8s+7 = tile rows r0-8+8s..): half 0: above, inside x 3; half 1: inside x 3, below
  tmask = tma_stage(ts, homes, buf, b * kTileCols, c * kTileRows + r0, kQuarterStage / kSlotRows,
                    [half](int sl) { return half ? (sl == 3 ? 2 : 1) : (sl == 0 ? 0 : 1); });
#endif
  {
    const uint32_t ch = __shfl_sync(0xffffffffu, homes, (2 * lane) & 31);
    const uint32_t col = b * kTileCols + (lane & 15) * 8;
    const uint16_t* base[3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
      base[r] = f0 + (((ch >> r) & 1u) ? delta : 0) + ((size_t)c * kTileRows + r0) * pitch + col;
    uint8_t* dst = buf + (lane & 15) * 16;
#pragma unroll
    for (int k = 0; k < kQuarterStage / 2; ++k) {
      const int row = 2 * k + (lane >> 4);  // staged row = item row + kK
      const int trow = (int)r0 + row - kK;  // tile row
      const int reg = trow < 0 ? 0 : (trow < kTileRows ? 1 : 2);
      if (!((tmask >> reg) & 1u)) cp_async16(dst + row * kTileRowBytes, base[reg] + (size_t)row * pitch);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  uint32_t P0[kK][4], P1[kK][4];
#if !AM_TRIM
#pragma unroll
  for (int j = 0; j < kK; ++j)
#pragma unroll
    for (int w = 0; w < 4; ++w) P0[j][w] = P1[j][w] = 0u;
#endif
  uint32_t acc = 0xFFFFFFFFu, accE = 0xFFFFFFFFu;
  const ptrdiff_t od = ((homes >> 6) & 1u) ? delta : 0;
  uint16_t* oA = f0 + od + ((size_t)c * kTileRows + r0 + kK) * pitch + b * kTileCols + lane * kTileWPL;
  uint16_t* oB = oA + (size_t)kQuarterRows * pitch;
  const bool st = lane >= kK / kTileWPL && lane < 32 - kK / kTileWPL;
  const uint8_t* rb = buf + lane * 8;
  // phase lags: [0,8) lo reads rows r0-8.. (above the tile for half 0), hi rows r0..; [8,16) own;
  // [16,24) hi reads rows r0+16.. (below the tile for half 1)
  const uint32_t lag0 = (half ? lw[1] : lw[0]) | lw[1] << 16, lag1 = lw[1] | lw[1] << 16,
                 lag2 = lw[1] | (half ? lw[2] : lw[1]) << 16;
  const bool l0 = __any_sync(0xffffffffu, lag0 != 0u), l1 = __any_sync(0xffffffffu, lag1 != 0u),
             l2 = __any_sync(0xffffffffu, lag2 != 0u);
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#if AM_TMA
  mbar_wait(ts.mbA, ts.parity);  // (mbB completed on its zero-byte arrive)
  ts.parity ^= 1u;
#else
  (void)ts;
#endif
  __syncwarp();
#if AM_TRIM
  tile_fill<kQuarterRows>(rb, lag0, l0, lag1, l1, P0, P1);
#else
  tile_phase<kOutNone, kQuarterRows>(rb, 0, kK, lag0, l0, P0, P1, oA, oB, pitch, st, acc, accE);
  tile_phase<kOutNone, kQuarterRows>(rb, kK, 2 * kK, lag1, l1, P0, P1, oA, oB, pitch, st, acc, accE);
#endif
  tile_phase<kOutTop, kQuarterRows>(rb, 2 * kK, kQuarterSteps, lag2, l2, P0, P1, oA, oB, pitch, st, acc, accE);
  if (!st) acc = accE = 0xFFFFFFFFu;  // halo lanes hold no output
  edge[0] = edge[1] = accE;  // every output row of a quarter stream is within kK of its item's edge
  return acc;
}

// ---- very light blocks: eighth items (four warps per tile) ------------------
//
// When a block has at most a quarter warp slot per tile, each tile runs as
// four items of 8 rows (part p: tile rows 8p .. 8p+7) whose u16 streams carry
// 4 rows each: 4 + 2K = 20 steps.  Staged: the 24 rows 8p-8 .. 8p+15.  The lo
// stream reads staged row s, the hi stream row s+4; every 4-step phase reads
// one region (above / inside / below the tile) per stream, so a phase has one
// lag word.  Items of tiles with a source in reach run as quarter items (parts
// 0 and 2; parts 1 and 3 then do nothing).
#ifndef AM_EIGHTHS
#define AM_EIGHTHS 0  // 1: C2 -2%, C4 +0.9% (code growth in the heavy path)
#endif
constexpr int kEighthRows = 4;                          // rows per u16 stream
constexpr int kEighthSteps = kEighthRows + 2 * kK;      // 20
constexpr int kEighthStage = 2 * kEighthRows + 2 * kK;  // 24 rows staged
static_assert(kEighthStage % 2 == 0 && kTileRows == 4 * 2 * kEighthRows, "eighth layout");

__device__ __forceinline__ uint32_t tile_eighth16(const Geo& g, uint16_t* __restrict__ f0, ptrdiff_t delta,
                                                  uint32_t b, uint32_t c, uint32_t part, const uint32_t (&lw)[3],
                                                  uint32_t homes, uint32_t* edge, uint8_t* buf) {
  const int lane = threadIdx.x & 31;
  const size_t pitch = g.pitch;
  const int r0 = (int)part * 2 * kEighthRows;  // first tile row of the item
  auto region = [](int trow) { return trow < 0 ? 0 : (trow < kTileRows ? 1 : 2); };
  __syncwarp();  // every lane is done reading the previous item's rows
  {
    const uint32_t ch = __shfl_sync(0xffffffffu, homes, (2 * lane) & 31);
    const uint32_t col = b * kTileCols + (lane & 15) * 8;
    const uint16_t* base[3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
      base[r] = f0 + (((ch >> r) & 1u) ? delta : 0) + ((size_t)c * kTileRows + r0) * pitch + col;
    uint8_t* dst = buf + (lane & 15) * 16;
#pragma unroll
    for (int k = 0; k < kEighthStage / 2; ++k) {
      const int row = 2 * k + (lane >> 4);  // staged row = item row + kK
      cp_async16(dst + row * kTileRowBytes, base[region(r0 + row - kK)] + (size_t)row * pitch);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  uint32_t P0[kK][4], P1[kK][4];
  uint32_t acc = 0xFFFFFFFFu, accE = 0xFFFFFFFFu;
  const ptrdiff_t od = ((homes >> 6) & 1u) ? delta : 0;
  uint16_t* oA = f0 + od + ((size_t)c * kTileRows + r0 + kK) * pitch + b * kTileCols + lane * kTileWPL;
  uint16_t* oB = oA + (size_t)kEighthRows * pitch;
  const bool st = lane >= kK / kTileWPL && lane < 32 - kK / kTileWPL;
  const uint8_t* rb = buf + lane * 8;
  // phase q (steps 4q .. 4q+3): lo reads tile rows r0-8+4q.., hi rows r0-4+4q..
  uint32_t lag[5];
  bool lg[5];
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    lag[q] = lw[region(r0 - kK + 4 * q)] | lw[region(r0 - kK + kEighthRows + 4 * q)] << 16;
    lg[q] = __any_sync(0xffffffffu, lag[q] != 0u);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
  fill_pair<0, kEighthRows>(rb, lag[0], lg[0], P0, P1);
  fill_pair<1, kEighthRows>(rb, lag[0], lg[0], P0, P1);
  fill_pair<2, kEighthRows>(rb, lag[1], lg[1], P0, P1);
  fill_pair<3, kEighthRows>(rb, lag[1], lg[1], P0, P1);
  fill_pair<4, kEighthRows>(rb, lag[2], lg[2], P0, P1);
  fill_pair<5, kEighthRows>(rb, lag[2], lg[2], P0, P1);
  fill_pair<6, kEighthRows>(rb, lag[3], lg[3], P0, P1);
  fill_pair<7, kEighthRows>(rb, lag[3], lg[3], P0, P1);
  tile_phase<kOutTop, kEighthRows>(rb, 2 * kK, kEighthSteps, lag[4], lg[4], P0, P1, oA, oB, pitch, st, acc, accE);
  if (!st) acc = accE = 0xFFFFFFFFu;  // halo lanes hold no output
  edge[0] = edge[1] = accE;
  return acc;
}

// Quarter items next to a source: the general path on two 8-row streams (rows r0.. and r0+8..).
__device__ __noinline__ uint32_t tile_item16_sources8(const Geo& g, uint16_t* f0, const uint8_t* srcmask,
                                                      const uint8_t* rf, uint32_t b, uint32_t r0, uint32_t lag0,
                                                      uint32_t lag1, uint32_t lag2, ptrdiff_t delta, uint32_t homes,
                                                      uint32_t* edge) {
  return stream_item<16, false, true, kTileStages, kTileWPL, kTileWarpSmem>(
      g, f0, f0, srcmask, rf, rf, b, r0, b, r0 + kQuarterRows, kQuarterRows, true, lag0, lag1, lag2, delta, homes,
      edge);
}

// The rare items whose rows hold a source (the +1 path): kept out of line so
// the hot loop of k_block_tiles stays small in the instruction cache.
__device__ __noinline__ uint32_t tile_item16_sources(const Geo& g, uint16_t* f0, const uint8_t* srcmask,
                                                     const uint8_t* rf, uint32_t b, uint32_t ra, uint32_t lag0,
                                                     uint32_t lag1, uint32_t lag2, ptrdiff_t delta, uint32_t homes,
                                                     uint32_t* edge) {
  return stream_item<16, false, true, kTileStages, kTileWPL, kTileWarpSmem>(g, f0, f0, srcmask, rf, rf, b, ra, b,
                                                                            ra + kHalfRows, kHalfRows, true, lag0,
                                                                            lag1, lag2, delta, homes, edge);
}

// Dense mode: every (band, segment pair) of the grid, one warp each.
template <int CB, bool SLAB>
__global__ void __launch_bounds__(kBlockThreads, AM_BLOCK_MINB) k_block(Geo g, const typename Cell<CB>::T* __restrict__ in,
                                                         typename Cell<CB>::T* __restrict__ out,
                                                         const uint8_t* __restrict__ srcmask,
                                                         const uint8_t* __restrict__ rowsrc,
                                                         FlagSink flag) {
  const uint32_t warp = blockIdx.x * (kBlockThreads / 32) + (threadIdx.x >> 5);
  const uint32_t ntiles = CB == 16 ? g.nseg / 2 : g.nseg;
  if (warp >= g.nbands * ntiles) return;
  const uint32_t band = warp % g.nbands, tile = warp / g.nbands;
  const uint32_t rA = tile * g.seg_len;  // allocated row of step 0
  const uint32_t rB = (CB == 16 ? tile + ntiles : tile) * g.seg_len;
  const uint8_t* rf = rowsrc + g.dense_rowsrc(band);
  const uint32_t acc = stream_item<CB, SLAB>(g, in, out, srcmask, rf, rf, band, rA, band, rB, g.seg_len, true);
  publish_flag<false>(flag, __reduce_min_sync(0xffffffffu, Cell<CB>::fold(acc)), g.nbands * ntiles);
}

// Frontier-region bit a neighbour N at (dr, dc) from tile T must have for T
// to become active: a frontier cell within kK of T lies in N's region facing
// T (bits: 0 any, 1 top, 2 bottom, 3 left, 4 right, 5 tl, 6 tr, 7 bl, 8 br).
__constant__ uint8_t kFacing[3][3] = {{8, 2, 7}, {4, 0, 3}, {6, 1, 5}};

// Lists tile (c, b) for block blk + 1 unless it is already listed (one
// lane per candidate; the appends are warp-aggregated).
__device__ __forceinline__ void push_tiles(const Geo& g, TileBook& book, uint32_t blk, bool want, int c, int b) {
  const bool in = want && c >= 0 && b >= 0 && c < (int)g.nchunks && b < (int)g.tbands;
  bool add = false;
  uint32_t src = 0;
  if (in) {
    const uint32_t t = (uint32_t)c * g.tbands + (uint32_t)b;
    src = book.tsrc[t];  // independent of the atomic: no added latency
    add = atomicMax(&book.sched[t], blk + 2) < blk + 2;
  }
  const uint32_t m = __ballot_sync(0xffffffffu, add);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(&book.count[(blk + 1) % 3], (uint32_t)__popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (add)
    book.list[(blk + 1) & 1][base + __popc(m & ((1u << lane) - 1u))] =
        (uint32_t)b << 16 | (uint32_t)c | (src ? kListSrc : 0u);
}

// Active-tile mode: the warps walk the block's work list (items = band << 16
// | chunk), two tiles per warp in 16-bit mode.  Every tile has a home field
// (the ping-pong field holding its latest values) and the layer of those
// values (TileBook state).  The item reads each region it touches from that
// region's home with the region's lag added to covered cells, and writes its
// own rows to the other field, so quiet tiles are never copied or
// rewritten.  Each processed tile then lists, for the next block, itself
// and the neighbours its frontier (cells covered in the block's last layer)
// can reach within kK cells.
template <int CB>
__global__ void __launch_bounds__(kTileThreads, kTileCtasPerSm)
    k_block_tiles(Geo g, typename Cell<CB>::T* __restrict__ f0, ptrdiff_t delta, const uint8_t* __restrict__ srcmask,
                  const uint8_t* __restrict__ rowsrc, TileBook book, uint32_t blk, uint32_t l0, FlagSink flag,
                  FlagSink prev, const __grid_constant__ TileMaps tmaps) {
  extern __shared__ __align__(128) uint8_t smem_tiles[];
  // this warp's two staging mbarriers live after the per-warp buffers
  TmaStage ts{&tmaps, smem_u32(smem_tiles + kTileSmem + (threadIdx.x >> 5) * 16),
              smem_u32(smem_tiles + kTileSmem + (threadIdx.x >> 5) * 16 + 8), 0u};
#if AM_TMA
  if (CB == 16 && (threadIdx.x & 31) == 0) {
    mbar_init(ts.mbA, 4);  // slot lanes 0-3
    mbar_init(ts.mbB, 2);  // slot lanes 4-5
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
#endif
  // programmatic dependent launch: this grid may start while the previous
  // block's grid drains; wait for it (memory visible) before touching state,
  // and let the next block's grid get scheduled right away
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  // the previous block's fixed-point word is complete now: publish it here
  // (no arrival counter or fence at the end of every block)
  if (prev.host && blockIdx.x == 0 && threadIdx.x == 0)
    *reinterpret_cast<volatile uint32_t*>(prev.host) = atomicExch(prev.word, 0xFFFFFFFFu);
  const uint32_t n = book.count[blk % 3];
  const uint32_t* __restrict__ list = book.list[blk & 1];
#if AM_SPEC_LIST
  // Light blocks take static quarter items (w -> tile w / 2): the list entry of this warp's first
  // item is loaded alongside the list length instead of after it (one L2 round trip less per block)
  const uint32_t w_static = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  const uint32_t spec_entry = (w_static >> 1) < g.ntiles() ? list[w_static >> 1] : 0u;
#endif
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    book.count[(blk + 2) % 3] = 0;
    book.count[3 + (blk + 2) % 3] = 0;
    atomicAdd(book.processed, (unsigned long long)n);
  }
  const uint32_t l1 = l0 + kK;  // layer after this block
  const int lane = threadIdx.x & 31;
  constexpr int kHaloLanes = kK / kTileWPL;  // lanes holding the left / right halo columns
  const int brel = lane < kHaloLanes ? -1 : (lane >= 32 - kHaloLanes ? 1 : 0);  // band of this lane's cells
  // state at l0 of tile t (cur, or old if t was already processed in this block)
  auto state_at_l0 = [&](uint32_t t) -> uint32_t {
    const unsigned long long w = *reinterpret_cast<const volatile unsigned long long*>(book.state + t);
    const uint32_t cur = (uint32_t)w;
    return (cur >> 1) == l1 ? (uint32_t)(w >> 32) : cur;
  };
  // (lag, home) of the tile this lane reads at chunk c0+dr
  auto region = [&](uint32_t c0, uint32_t b0, int dr, uint32_t& home) -> uint32_t {
    const int c = (int)c0 + dr, b = (int)b0 + brel;
    home = 0;
    if (c < 0 || b < 0 || c >= (int)g.nchunks || b >= (int)g.tbands) return 0u;  // padding: zero in both fields
    const uint32_t s = state_at_l0((uint32_t)c * g.tbands + (uint32_t)b);
    home = s & 1u;
    const uint32_t e = s >> 1;
    return e < l0 ? l0 - e : 0u;
  };
  uint32_t gmin = 0xFFFFFFFFu;
  constexpr int kL = kHaloLanes, kR = 32 - 2 * kHaloLanes;  // first lane of the left / right edge columns
  auto lanes_min = [&](uint32_t v, int first) {
    uint32_t m = __shfl_sync(0xffffffffu, v, first);
#pragma unroll
    for (int k = 1; k < kHaloLanes; ++k) m = Cell<CB>::vmin(m, __shfl_sync(0xffffffffu, v, first + k));
    return m;
  };
  // 9 region bits of the stream in half h (lo 0, hi 1) of a quarter item: every output row of the
  // stream is within kK of both its top and bottom, so e serves both edges
  auto regions16q = [&](uint32_t acc, uint32_t e, int h) -> uint32_t {
    auto part = [h](uint32_t v) { return h ? v >> 16 : v & 0xFFFFu; };
    const uint32_t a = __reduce_min_sync(0xffffffffu, part(acc)), ee = __reduce_min_sync(0xffffffffu, part(e));
    const uint32_t l = part(lanes_min(acc, kL)), r = part(lanes_min(acc, kR));
    const uint32_t el = part(lanes_min(e, kL)), er = part(lanes_min(e, kR));
    return (a == 0u ? 1u : 0u) | (ee == 0u ? 6u : 0u) | (l == 0u ? 8u : 0u) | (r == 0u ? 16u : 0u) |
           (el == 0u ? 0xA0u : 0u) | (er == 0u ? 0x140u : 0u);
  };
  // light blocks (at most half a warp slot per tile): two quarter items per tile, shorter latency
  const uint32_t nwarps = gridDim.x * (kTileThreads / 32);
  const bool quarters = CB == 16 && AM_QUARTERS && 2u * n <= (uint32_t)AM_QUARTER_SLOTS * nwarps;
  const bool eighths = quarters && AM_EIGHTHS && 4u * n <= nwarps;  // four items per tile (tile_eighth16)
  // heavy blocks (more tiles than warps): two whole tiles per item (tile_pair16)
  const bool pairs = CB == 16 && AM_PAIRS && !quarters && 4u * n > (uint32_t)AM_PAIR_MIN4 * nwarps;
  const uint32_t nitems = eighths ? 4u * n : quarters ? 2u * n : (pairs ? (n + 1) / 2 : n);
#if AM_STATIC_FIRST
  // Every warp's first item is static, spread over the CTAs (item i -> CTA i mod grid, so consecutive items
  // land on different SMs); only items past the warp count are fetched dynamically (a warp that finishes
  // early takes the next one).  A light block then runs without a single fetch atomic, and a heavy block
  // saves one same-address atomic per warp.
  const bool light = nitems <= nwarps;
  auto fetch = [&]() {
    if (AM_STATIC_FIRST == 2 ? light : AM_STATIC_FIRST == 1 && light) return 0xFFFFFFFFu;
    uint32_t v = 0;
    if (lane == 0) v = atomicAdd(&book.count[3 + blk % 3], 1u) + (AM_STATIC_FIRST == 2 ? nwarps : 0u);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  // 1: static items in light blocks only (heavy blocks fetch every item); 2: static first item everywhere
  uint32_t w = (AM_STATIC_FIRST == 2 || light) ? (threadIdx.x >> 5) * gridDim.x + blockIdx.x : fetch();
#else
  // items are fetched dynamically: a warp that finishes early takes the next one
  auto fetch = [&]() {
    uint32_t v = 0;
    if (lane == 0) v = atomicAdd(&book.count[3 + blk % 3], 1u);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  uint32_t w = fetch();
#endif
  constexpr uint32_t kNone = 0xFFFFFFFFu;
  uint32_t solo = kNone;  // the second tile of a pair item that takes the single-tile path
  while (w < nitems || solo != kNone) {
    uint32_t it, half = 0;
    bool fetch_next = true;
    if (solo != kNone) {
      it = solo;
      solo = kNone;
    } else if (CB == 16 && pairs) {
      const uint32_t itA = list[2 * w], itB = 2 * w + 1 < n ? list[2 * w + 1] : kNone;
      if constexpr (CB == 16) {
        if (itB != kNone) {
          const uint32_t bA = (itA >> 16) & kListBand, cA = itA & 0xFFFFu, bB = (itB >> 16) & kListBand,
                         cB = itB & 0xFFFFu;
          if (!((itA | itB) & kListSrc)) {  // no source in reach of either tile
            const uint32_t tA = cA * g.tbands + bA, tB = cB * g.tbands + bB;
            const uint32_t sA = state_at_l0(tA), sB = state_at_l0(tB);
            uint32_t lwA[3], hmA[3], lwB[3], hmB[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              lwA[d] = region(cA, bA, d - 1, hmA[d]);
              lwB[d] = region(cB, bB, d - 1, hmB[d]);
            }
            const uint32_t ohA = (sA & 1u) ^ 1u, ohB = (sB & 1u) ^ 1u;
            const uint32_t homesA = hmA[0] | hmA[1] << 1 | hmA[2] << 2, homesB = hmB[0] | hmB[1] << 1 | hmB[2] << 2;
            uint16_t* f16 = reinterpret_cast<uint16_t*>(f0);
            const size_t pitch = g.pitch;
            const uint16_t* baseA = f16 + (size_t)cA * kTileRows * pitch + bA * kTileCols;
            const uint16_t* baseB = f16 + (size_t)cB * kTileRows * pitch + bB * kTileCols;
            uint8_t* buf = smem_tiles + (threadIdx.x >> 5) * kTileWarpSmem;
            __syncwarp();  // every lane is done reading the previous item's rows
            pair_stage(g, f16, delta, baseA, baseB, homesA, homesB, buf, 0, kHalfRows);
            asm volatile("cp.async.commit_group;" ::: "memory");
            pair_stage(g, f16, delta, baseA, baseB, homesA, homesB, buf, kHalfRows, kTileRows);
            asm volatile("cp.async.commit_group;" ::: "memory");
            uint16_t* oA = f16 + (ohA ? delta : 0) + (size_t)(cA * kTileRows + kK) * pitch + bA * kTileCols + lane * kTileWPL;
            uint16_t* oB = f16 + (ohB ? delta : 0) + (size_t)(cB * kTileRows + kK) * pitch + bB * kTileCols + lane * kTileWPL;
            uint32_t edge[2];
            const uint32_t acc = tile_pair16(g, f16, delta, baseA, baseB, lwA, lwB, homesA, homesB, oA, oB, edge, buf);
            const uint32_t next = fetch();
            // frontier regions of A (lo) and B (hi)
            auto m9_of = [&](int h) -> uint32_t {
              auto part = [h](uint32_t v) { return h ? v >> 16 : v & 0xFFFFu; };
              const uint32_t vals[9] = {__reduce_min_sync(0xffffffffu, part(acc)),
                                        __reduce_min_sync(0xffffffffu, part(edge[0])),
                                        __reduce_min_sync(0xffffffffu, part(edge[1])),
                                        part(lanes_min(acc, kL)),
                                        part(lanes_min(acc, kR)),
                                        part(lanes_min(edge[0], kL)),
                                        part(lanes_min(edge[0], kR)),
                                        part(lanes_min(edge[1], kL)),
                                        part(lanes_min(edge[1], kR))};
              uint32_t m = 0;
#pragma unroll
              for (int k = 0; k < 9; ++k) m |= (vals[k] == 0u ? 1u : 0u) << k;
              gmin = min(gmin, vals[0]);
              return m;
            };
            const uint32_t mA = m9_of(0), mB = m9_of(1);
            if (lane == 0) {
              book.state[tA] = (unsigned long long)sA << 32 | (l1 << 1 | ohA);
              book.state[tB] = (unsigned long long)sB << 32 | (l1 << 1 | ohB);
            }
            const int dr = lane / 3 - 1, dc = lane % 3 - 1;
            const int fk = kFacing[(lane / 3) % 3][lane % 3];
            push_tiles(g, book, blk, lane < 9 && ((mA >> fk) & 1u), (int)cA - dr, (int)bA - dc);
            push_tiles(g, book, blk, lane < 9 && ((mB >> fk) & 1u), (int)cB - dr, (int)bB - dc);
            w = next;
            continue;
          }
        }
      }
      it = itA;  // a source in reach or no partner: the single-tile path, one tile after the other
      solo = itB;
      fetch_next = itB == kNone;
    } else {
#if AM_SPEC_LIST
      it = (quarters && !eighths && w == w_static) ? spec_entry : list[eighths ? w >> 2 : (quarters ? w >> 1 : w)];
#else
      it = list[eighths ? w >> 2 : (quarters ? w >> 1 : w)];
#endif
      half = eighths ? (w & 3u) : (quarters ? w & 1u : 0u);  // eighths: the part (0-3)
    }
    const uint32_t bA = (it >> 16) & kListBand, cA = it & 0xFFFFu;
    const uint32_t tA = cA * g.tbands + bA;
    const uint8_t* rf = rowsrc + g.tile_rowsrc(bA);
    const uint32_t ra = cA * kTileRows;
    uint32_t f = 0;  // source rows in reach (read only for tiles listed with kListSrc)
    if constexpr (CB == 16) {
      if (!(it & kListSrc) || eighths) {  // (eighths: the quarter fallback below reads its own rows)
      } else if (quarters) {
        f = rf[ra + half * kHalfRows + lane];  // the item's 32 staged rows
      } else {
        f = rf[ra + lane];
        if (lane < kStageRows - 32) f |= rf[ra + 32 + lane];
      }
    }
    const uint32_t sa = state_at_l0(tA);  // own state before the neighbours' (rewritten below)
    uint32_t lw[3], hm[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) lw[d] = region(cA, bA, d - 1, hm[d]);
    const uint32_t out_home = (sa & 1u) ^ 1u;  // own rows go to the field that is not the tile's home
    uint32_t edge[2], acc;
    uint32_t m9;  // frontier regions (bits: any, top, bottom, left, right, tl, tr, bl, br)
    if (CB == 16 && eighths && !(it & kListSrc)) {
      uint8_t* buf = smem_tiles + (threadIdx.x >> 5) * kTileWarpSmem;
      acc = tile_eighth16(g, reinterpret_cast<uint16_t*>(f0), delta, bA, cA, half, lw,
                          hm[0] | hm[1] << 1 | hm[2] << 2 | out_home << 6, edge, buf);
      // any / left / right from both streams; top (bottom) edge bits when the item holds tile rows 0-7 (24-31)
      const uint32_t m2 = regions16q(acc, edge[0], 0) | regions16q(acc, edge[0], 1);
      m9 = (m2 & 0x19u) | (half == 0 ? (m2 & 0x62u) : 0u) | (half == 3 ? (m2 & 0x184u) : 0u);
      gmin = min(gmin, min(__reduce_min_sync(0xffffffffu, acc & 0xFFFFu), __reduce_min_sync(0xffffffffu, acc >> 16)));
    } else if (CB == 16 && quarters) {
      if (eighths) {  // a tile with a source in reach: quarter items (parts 0 and 2), parts 1 and 3 idle
        if (half & 1u) {
          w = fetch_next ? fetch() : w;
          continue;
        }
        half >>= 1;
        f = rf[ra + half * kHalfRows + lane];  // the quarter's 32 staged rows (the eighth read no flags)
      }
      uint8_t* buf = smem_tiles + (threadIdx.x >> 5) * kTileWarpSmem;
      const uint32_t r0 = ra + half * kHalfRows;
      if (!__any_sync(0xffffffffu, f != 0u)) {
        acc = tile_quarter16(g, reinterpret_cast<uint16_t*>(f0), delta, bA, cA, half, lw,
                             hm[0] | hm[1] << 1 | hm[2] << 2 | out_home << 6, edge, buf, ts);
      } else {  // a source in reach: the general path on the same two 8-row streams
        const uint32_t up = half ? hm[1] : hm[0], dn = half ? hm[2] : hm[1];
        const uint32_t homes = up | hm[1] << 1 | hm[1] << 2 | hm[1] << 3 | hm[1] << 4 | dn << 5 | out_home << 6 |
                               out_home << 7;
        acc = tile_item16_sources8(g, reinterpret_cast<uint16_t*>(f0), srcmask, rf, bA, r0, (half ? lw[1] : lw[0]) | lw[1] << 16,
                                   lw[1] | lw[1] << 16, lw[1] | (half ? lw[2] : lw[1]) << 16, delta, homes, edge);
      }
      // regions: any / left / right from both streams; the top edge (tl, tr) is the lo stream of half 0,
      // the bottom edge (bl, br) the hi stream of half 1
      const uint32_t mlo = regions16q(acc, edge[0], 0), mhi = regions16q(acc, edge[0], 1);
      m9 = ((mlo | mhi) & 0x19u) | (half == 0 ? (mlo & 0x62u) : 0u) | (half == 1 ? (mhi & 0x184u) : 0u);
      gmin = min(gmin, min(__reduce_min_sync(0xffffffffu, acc & 0xFFFFu), __reduce_min_sync(0xffffffffu, acc >> 16)));
    } else if constexpr (CB == 16) {
      // upper half (lo): tile rows 0-15, lower half (hi): rows 16-31
      uint8_t* buf = smem_tiles + (threadIdx.x >> 5) * kTileWarpSmem;
      const uint32_t homes16 = hm[0] | hm[1] << 1 | hm[2] << 2 | out_home << 6;
      tile_stage16(g, f0, delta, bA, cA, homes16, buf, ts);  // copies in flight during the source vote
      if (!__any_sync(0xffffffffu, f != 0u)) {
        acc = tile_item16(g, f0, delta, bA, cA, lw, homes16, edge, buf, ts);
#if AM_TMA
        ts.parity ^= 1u;
#endif
      } else {  // a source in reach: the general path, same halves (its ring reuses buf)
        asm volatile("cp.async.wait_group 0;" ::: "memory");
#if AM_TMA
        mbar_wait(ts.mbA, ts.parity);
        mbar_wait(ts.mbB, ts.parity);
        ts.parity ^= 1u;
#endif
        __syncwarp();
        const uint32_t homes = hm[0] | hm[1] << 1 | hm[1] << 2 | hm[1] << 3 | hm[1] << 4 | hm[2] << 5 |
                               out_home << 6 | out_home << 7;
        acc = tile_item16_sources(g, f0, srcmask, rf, bA, ra, lw[0] | lw[1] << 16, lw[1] | lw[1] << 16,
                                  lw[1] | lw[2] << 16, delta, homes, edge);
      }
      auto lo = [](uint32_t v) { return v & 0xFFFFu; };
      auto hi = [](uint32_t v) { return v >> 16; };
      auto both = [&](uint32_t v) { return min(lo(v), hi(v)); };
      const uint32_t vals[9] = {both(__reduce_min_sync(0xffffffffu, lo(acc)) | __reduce_min_sync(0xffffffffu, hi(acc)) << 16),
                                __reduce_min_sync(0xffffffffu, lo(edge[0])),
                                __reduce_min_sync(0xffffffffu, hi(edge[1])),
                                both(lanes_min(acc, kL)),
                                both(lanes_min(acc, kR)),
                                lo(lanes_min(edge[0], kL)),
                                lo(lanes_min(edge[0], kR)),
                                hi(lanes_min(edge[1], kL)),
                                hi(lanes_min(edge[1], kR))};
      m9 = 0;
#pragma unroll
      for (int k = 0; k < 9; ++k) m9 |= (vals[k] == 0u ? 1u : 0u) << k;
      gmin = min(gmin, vals[0]);
    } else {
      const uint32_t homes = hm[0] | hm[1] << 1 | hm[2] << 2 | out_home << 6;
      acc = stream_item<CB, false, true, kTileStages, kTileWPL, kTileWarpSmem>(
          g, f0, f0, srcmask, rf, rf, bA, cA * kTileRows, bA, cA * kTileRows, kTileRows, false, lw[0], lw[1], lw[2],
          delta, homes, edge);
      const uint32_t vals[9] = {__reduce_min_sync(0xffffffffu, acc), __reduce_min_sync(0xffffffffu, edge[0]),
                                __reduce_min_sync(0xffffffffu, edge[1]), lanes_min(acc, kL), lanes_min(acc, kR),
                                lanes_min(edge[0], kL), lanes_min(edge[0], kR), lanes_min(edge[1], kL),
                                lanes_min(edge[1], kR)};
      m9 = 0;
#pragma unroll
      for (int k = 0; k < 9; ++k) m9 |= (vals[k] == 0u ? 1u : 0u) << k;
      gmin = min(gmin, vals[0]);
    }
    const uint32_t next = fetch_next ? fetch() : w;  // the next item's index travels while the bookkeeping runs
    // new state (old kept in the high word for this block's readers)
    if (lane == 0) book.state[tA] = (unsigned long long)sa << 32 | (l1 << 1 | out_home);
    // list the next block's candidates: lane k < 9 for the neighbour at (dr, dc) = (k/3-1, k%3-1)
    {
      const int dr = lane / 3 - 1, dc = lane % 3 - 1;  // T = N - (dr, dc) is activated by N's facing region
      const bool want = lane < 9 && ((m9 >> kFacing[(lane / 3) % 3][lane % 3]) & 1u);
      push_tiles(g, book, blk, want, (int)cA - dr, (int)bA - dc);
    }
    w = next;
  }
  publish_flag<true>(flag, gmin, gridDim.x);
}

// ------------------------------------------------- active-tile bookkeeping
//
// Exact skipping.  A cell covered during block b+1 is at
// most kK hops from a cell covered in the last layer of block b, and tiles
// are at least kK cells in both directions, so only tiles whose 3x3 tile
// neighbourhood holds a frontier cell (covered during block b) can change
// coverage in block b+1.  Every other tile is quiet: its covered cells just
// gain +1 per layer, applied lazily through its state (layer of the stored
// values + home field).

// Covered cells (flag set, a > 0) are exactly the halves above the bare flag:
// adds `lagw` (per-half lag) to them, leaving uncovered and obstacle cells.
// Obstacle and padding cells are unflagged but keep junk low bits (the layer
// step only clears their flag), so the test must include the flag: lag added
// to junk would grow it across layers and runs until it carried into the flag
// bit and turned a wall or padding cell into a covered one.
template <int CB>
__device__ __forceinline__ uint32_t add_lag(uint32_t w, uint32_t lagw) {
  if constexpr (CB == 16) {
    // covered <=> half > 0x8000: after a per-half max with 0x8000 every half is >= 0x8000, so
    // subtracting 1 per half cannot borrow across halves and leaves bit 15 set exactly for
    // covered halves; PRMT replicates bit 15 (VIMNMX + IADD + PRMT)
    uint32_t cov;  // prmt's sign-replicate selectors (__byte_perm drops the selector msb)
    asm("prmt.b32 %0, %1, 0, 0xbb99;" : "=r"(cov) : "r"(__vmaxu2(w, 0x80008000u) - 0x00010001u));
    return w + (cov & lagw);
  } else return w + (w > kFlag32 ? lagw : 0u);
}

// 16 B per lane-row: 8 cells (u16) or 4 cells (u32)
template <int CB, typename F>
__device__ __forceinline__ void tile_rows_foreach(const Geo& g, uint32_t band, uint32_t chunk, F f) {
  const int lane = threadIdx.x & 31;
  constexpr int kVecCells = 16 / sizeof(typename Cell<CB>::T);
  constexpr int kVecs = kTileCols / kVecCells;  // vectors per tile row
  for (int v = lane; v < kVecs * kTileRows; v += 32) {
    const uint32_t r = v / kVecs, k = v % kVecs;
    f((size_t)(chunk * kTileRows + r + g.pad) * g.pitch + g.pad + band * kTileCols + k * kVecCells);
  }
}

// Gathers every tile at layer l into field `dst` (f0 or f0+delta): values from
// the tile's home plus its lag.  One warp per tile.  Afterwards all tiles are
// current in dst (state = l << 1 | dst).
template <int CB>
__global__ void k_tiles_finalize(Geo g, unsigned long long* __restrict__ state, typename Cell<CB>::T* __restrict__ f0,
                                 ptrdiff_t delta, uint32_t dst, uint32_t l, uint32_t* __restrict__ zero) {
  const uint32_t t = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (t >= g.ntiles()) return;
  const uint32_t s = (uint32_t)state[t], home = s & 1u, e = s >> 1;
  const bool move = e != l || home != dst;
  if (move || zero) {
    const uint32_t lag = l - e;
    const uint32_t lagw = CB == 16 ? (lag | lag << 16) : lag;
    const typename Cell<CB>::T* src = f0 + (home ? delta : 0);
    typename Cell<CB>::T* out = f0 + (dst ? delta : 0);
    // fused fixed-point zero check (k_zero_check): a free cell still at a = 0 is the bare flag
    const uint32_t bare = CB == 16 ? 0x80008000u : kFlag32;
    bool z = false;
#if AM_FIN_BATCH
    // all of this lane's vectors in flight at once (memory-level parallelism), then processed
    constexpr int kVecCells = 16 / sizeof(typename Cell<CB>::T);
    constexpr int kVecs = kTileCols / kVecCells;
    constexpr int kPer = kVecs * kTileRows / 32;
    static_assert(kVecs * kTileRows % 32 == 0, "vectors per lane");
    const int lane = threadIdx.x & 31;
    const uint32_t band = t % g.tbands, chunk = t / g.tbands;
    size_t at[kPer];
    uint4 vv[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int v = lane + 32 * k;
      const uint32_t r = v / kVecs, q = v % kVecs;
      at[k] = (size_t)(chunk * kTileRows + r + g.pad) * g.pitch + g.pad + band * kTileCols + q * kVecCells;
      vv[k] = *reinterpret_cast<const uint4*>(src + at[k]);
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      uint4 v = vv[k];
      const size_t i = at[k];
#else
    tile_rows_foreach<CB>(g, t % g.tbands, t / g.tbands, [&](size_t i) {
      uint4 v = *reinterpret_cast<const uint4*>(src + i);
#endif
      if (lag) {
        v.x = add_lag<CB>(v.x, lagw);
        v.y = add_lag<CB>(v.y, lagw);
        v.z = add_lag<CB>(v.z, lagw);
        v.w = add_lag<CB>(v.w, lagw);
      }
      if (zero) {
        const uint32_t w[4] = {v.x ^ bare, v.y ^ bare, v.z ^ bare, v.w ^ bare};
#pragma unroll
        for (int k = 0; k < 4; ++k) z |= CB == 16 ? ((w[k] & 0xFFFFu) == 0u || (w[k] >> 16) == 0u) : w[k] == 0u;
      }
      if (move) *reinterpret_cast<uint4*>(out + i) = v;
#if AM_FIN_BATCH
    }
#else
    });
#endif
    if (zero && __any_sync(0xffffffffu, z) && (threadIdx.x & 31) == 0) atomicOr(zero, 1u);
  }
  __syncwarp();
  if ((threadIdx.x & 31) == 0) state[t] = (unsigned long long)(l << 1 | dst) << 32 | (l << 1 | dst);
}

// Row slabs: the slab's first (side 0) and last (side 1) kK rows at layer l,
// gathered from each tile's home field with its lag, into bnd[side] (pitched
// rows, padding columns left as allocated).  One warp per (side, tile band).
template <int CB>
__global__ void k_tiles_boundary(Geo g, const unsigned long long* __restrict__ state,
                                 const typename Cell<CB>::T* __restrict__ f0, ptrdiff_t delta, uint32_t l,
                                 typename Cell<CB>::T* __restrict__ dst0, typename Cell<CB>::T* __restrict__ dst1) {
  const uint32_t w = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (w >= 2 * g.tbands) return;
  const int lane = threadIdx.x & 31;
  const uint32_t side = w / g.tbands, b = w % g.tbands;
  constexpr int kVecCells = 16 / sizeof(typename Cell<CB>::T);
  constexpr int kVecs = kTileCols / kVecCells;  // vectors per tile row
  for (int v = lane; v < kVecs * kK; v += 32) {
    const uint32_t k = v / kVecs, q = v % kVecs;
    const uint32_t r = side ? g.H - kK + k : k;  // slab row
    const uint32_t s = (uint32_t)state[(r / kTileRows) * g.tbands + b], home = s & 1u, e = s >> 1;
    const uint32_t lag = l - e, lagw = CB == 16 ? (lag | lag << 16) : lag;
    const size_t col = g.pad + b * kTileCols + q * kVecCells;
    uint4 x = *reinterpret_cast<const uint4*>(f0 + (home ? delta : 0) + (size_t)(r + g.pad) * g.pitch + col);
    if (lag) {
      x.x = add_lag<CB>(x.x, lagw);
      x.y = add_lag<CB>(x.y, lagw);
      x.z = add_lag<CB>(x.z, lagw);
      x.w = add_lag<CB>(x.w, lagw);
    }
    *reinterpret_cast<uint4*>((side ? dst1 : dst0) + (size_t)k * g.pitch + col) = x;  // (peer memory: P2P store)
  }
}

// Row slabs: lists for block blk every boundary tile (first / last chunk) that
// a frontier cell (a == 1) of the received halo rows lies within kK of.
template <int CB>
__global__ void k_tiles_halo_scan(Geo g, const typename Cell<CB>::T* __restrict__ f0, TileBook book, uint32_t blk) {
  const uint32_t w = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (w >= 2 * g.tbands) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const uint32_t side = w / g.tbands, b = w % g.tbands;
  constexpr int kVecCells = 16 / sizeof(typename Cell<CB>::T);
  constexpr int kVecs = (kTileCols + 2 * kK) / kVecCells;  // the band's columns plus kK each side
  const uint32_t frontier = CB == 16 ? (kFlag16 | 1u) : (kFlag32 | 1u);
  const uint32_t row0 = side ? g.H + kK : 0u;  // allocated halo rows
  bool any = false;
  for (int v = lane; v < kVecs * kK; v += 32) {
    const uint32_t k = v / kVecs, q = v % kVecs;
    const uint4 x = *reinterpret_cast<const uint4*>(f0 + (size_t)(row0 + k) * g.pitch + b * kTileCols + q * kVecCells);
    const uint32_t ws[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      any |= CB == 16 ? ((ws[i] & 0xFFFFu) == frontier || (ws[i] >> 16) == frontier) : ws[i] == frontier;
  }
  any = __any_sync(0xffffffffu, any);
  push_tiles(g, book, blk - 1u, any && lane == 0, side ? (int)g.nchunks - 1 : 0, (int)b);
}

// Block 0's work list: the 3x3 neighbourhood of every tile with a source in
// reach (the layer-0 frontier, a = 1; TileBook::tsrc, a superset of the tiles
// holding one -- listing a tile that cannot change is harmless); pushed as
// block "-1" (lists 0, sched 1).
__global__ void k_tiles_init(Geo g, const uint8_t* __restrict__ srcmask, TileBook book) {
  (void)srcmask;
  const uint32_t t = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (t >= g.ntiles()) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const uint32_t chunk = t / g.tbands, band = t % g.tbands;
  if (!book.tsrc[t]) return;  // warp-uniform
  const int dr = lane / 3 - 1, dc = lane % 3 - 1;
  push_tiles(g, book, 0xFFFFFFFFu, lane < 9, (int)chunk + dr, (int)band + dc);
}

// Every tile current at `layer` in field `home` and listed for block blk
// (after dense single layers or the 32-bit promotion).
__global__ void k_tiles_all(Geo g, TileBook book, uint32_t blk, uint32_t layer, uint32_t home) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0) {
    book.count[blk % 3] = g.ntiles();
    book.count[(blk + 1) % 3] = 0;
    book.count[3 + blk % 3] = 0;
    book.count[3 + (blk + 1) % 3] = 0;
  }
  if (t >= g.ntiles()) return;
  const uint32_t cur = layer << 1 | home;
  book.state[t] = (unsigned long long)cur << 32 | cur;
  book.sched[t] = blk + 1;
  book.list[blk & 1][t] = (t % g.tbands) << 16 | (t / g.tbands) | (book.tsrc[t] ? kListSrc : 0u);
}

// -------------------------------------------------------- single layer
// One layer over the grid region (remainder layers, Mode::kIterative).
template <int CB>
__global__ void k_layer(Geo g, const typename Cell<CB>::T* __restrict__ in, typename Cell<CB>::T* __restrict__ out,
                        const uint8_t* __restrict__ srcmask, uint32_t* __restrict__ flag) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t r = blockIdx.y;
  uint32_t m = 0xFFFFFFFFu;
  if (c < g.W) {
    const size_t i = g.idx(r, c);
    const size_t p = g.pitch;
    uint32_t v = 0;
#pragma unroll
    for (int dr = -1; dr <= 1; ++dr)
#pragma unroll
      for (int dc = -1; dc <= 1; ++dc) {
        uint32_t u = in[i + dr * (long)p + dc];
        v = u > v ? u : v;
      }
    const uint32_t low = CB == 16 ? 0x7FFFu : kLow32;
    const uint32_t y = (v & ((uint32_t)in[i] | low)) + srcmask[i];
    out[i] = (typename Cell<CB>::T)y;
    m = Cell<CB>::fold(Cell<CB>::acc_min(CB == 16 ? (y | (y << 16)) : y, 0xFFFFFFFFu));
  }
  m = __reduce_min_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMin(flag, m);
}

// ------------------------------------------------------- promote / decode
__global__ void k_promote(Geo g, const uint16_t* __restrict__ in, uint32_t* __restrict__ out) {
  const size_t n = (size_t)g.rows * g.pitch;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t v = in[i];
    out[i] = (v & kFlag16) ? (kFlag32 | (v & 0x7FFFu)) : 0u;
  }
}

template <int CB>
__global__ void k_zero_check(Geo g, const typename Cell<CB>::T* __restrict__ val, uint32_t* __restrict__ flag) {
  const uint32_t c0 = 8 * (blockIdx.x * blockDim.x + threadIdx.x);  // 8 cells per thread, one vector load
  const uint32_t r = blockIdx.y;
  bool z = false;
  if (c0 < g.W) {  // cells past the edge are padding (never equal to the bare flag)
    const size_t i = g.idx(r, c0);
    if constexpr (CB == 16) {
      const uint4 q = *reinterpret_cast<const uint4*>(val + i);
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) z |= (w[k] & 0xFFFFu) == kFlag16 || (w[k] >> 16) == kFlag16;  // free, a == 0
    } else {
      const uint4 a = reinterpret_cast<const uint4*>(val + i)[0], b = reinterpret_cast<const uint4*>(val + i)[1];
      z = a.x == kFlag32 || a.y == kFlag32 || a.z == kFlag32 || a.w == kFlag32 || b.x == kFlag32 || b.y == kFlag32 ||
          b.z == kFlag32 || b.w == kFlag32;
    }
  }
  if (__any_sync(0xffffffffu, z) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

template <int CB>
__global__ void k_decode(Geo g, const typename Cell<CB>::T* __restrict__ val, uint32_t rollback, uint32_t r0,
                         uint32_t* __restrict__ dense) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t r = blockIdx.y + r0;
  if (c >= g.W) return;
  const uint32_t v = val[g.idx(r, c)];
  const uint32_t flagbit = CB == 16 ? kFlag16 : kFlag32;
  const uint32_t low = CB == 16 ? 0x7FFFu : kLow32;
  const uint32_t a = v & low;
  dense[(size_t)(r - r0) * g.W + c] = ((v & flagbit) && a) ? a - rollback : 0u;
}

// user-supplied dense map -> encoded 32-bit field (reconstruct on foreign maps)
__global__ void k_encode_dense(Geo g, const uint32_t* __restrict__ dense, const uint8_t* __restrict__ occ,
                               uint32_t* __restrict__ val) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t r = blockIdx.y;
  if (c >= g.W) return;
  const size_t d = (size_t)r * g.W + c;
  val[g.idx(r, c)] = occ[d] ? 0u : (kFlag32 | (dense[d] & kLow32));
}

// ------------------------------------------ plain / sentinel single layers
// propagate_layer on an arbitrary uint32 input (propagate.hpp:37-38): dense
// layout, explicit occupancy, wrap-around uint32 arithmetic like the host API.
__global__ void k_plain_layer(uint32_t W, uint32_t H, const uint8_t* __restrict__ occ,
                              const uint8_t* __restrict__ src, const uint32_t* __restrict__ in,
                              uint32_t* __restrict__ out) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t r = blockIdx.y;
  if (c >= W) return;
  uint32_t m = 0;
  for (int dr = -1; dr <= 1; ++dr) {
    const long rr = (long)r + dr;
    if (rr < 0 || rr >= (long)H) continue;
    for (int dc = -1; dc <= 1; ++dc) {
      const long cc = (long)c + dc;
      if (cc < 0 || cc >= (long)W) continue;
      const uint32_t u = in[(size_t)rr * W + cc];
      m = u > m ? u : m;
    }
  }
  const size_t i = (size_t)r * W + c;
  out[i] = occ[i] ? 0u : m + (uint32_t)(src[i] != 0);
}

// propagate_reference (propagate.hpp:63-68): literal signed formulation with
// the INT32_MIN obstacle sentinel re-added every layer, then ReLU.
__global__ void k_sentinel_layer(uint32_t W, uint32_t H, const uint8_t* __restrict__ occ,
                                 const uint8_t* __restrict__ src, const int32_t* __restrict__ in,
                                 int32_t* __restrict__ out) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t r = blockIdx.y;
  if (c >= W) return;
  int32_t m = 0;  // zero padding
  for (int dr = -1; dr <= 1; ++dr) {
    const long rr = (long)r + dr;
    if (rr < 0 || rr >= (long)H) continue;
    for (int dc = -1; dc <= 1; ++dc) {
      const long cc = (long)c + dc;
      if (cc < 0 || cc >= (long)W) continue;
      const int32_t u = in[(size_t)rr * W + cc];
      m = u > m ? u : m;
    }
  }
  const size_t i = (size_t)r * W + c;
  const long long t = (long long)m + (occ[i] ? INT32_MIN : 0) + (src[i] ? 1 : 0);
  out[i] = t > 0 ? (int32_t)t : 0;
}

__global__ void k_srcmask_dense(uint32_t W, uint32_t H, const uint32_t* __restrict__ rc, uint64_t n,
                                uint8_t* __restrict__ m, const uint8_t* __restrict__ occ, int* __restrict__ err) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t r = rc[2 * i], c = rc[2 * i + 1];
  if (r >= H || c >= W || occ[(size_t)r * W + c]) {
    atomicOr(err, 1);
    return;
  }
  m[(size_t)r * W + c] = 1;
}

// ------------------------------------------------------------- launchers
static dim3 grid2d(uint32_t W, uint32_t H, int bx) { return dim3((W + bx - 1) / bx, H); }

void launch_srcmask_rows(const Geo& g, uint32_t total_h, uint32_t row0, const uint32_t* d_src_rc, uint64_t n,
                         uint8_t* d_dense, const uint8_t* d_occ, uint8_t* d_srcmask, uint8_t* d_rowsrc, int* d_err,
                         cudaStream_t s) {
  if (!n) return;
  k_srcmask_rows<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, total_h, row0, d_src_rc, n, d_dense, d_occ,
                                                             d_srcmask, d_rowsrc, d_err);
}

void launch_init(const Geo& g, const uint8_t* d_occ, void* d_val, int cb, cudaStream_t s) {
  const dim3 grid((g.W + 8 * 128 - 1) / (8 * 128), g.H);
  if (cb == 16)
    k_init<16><<<grid, 128, 0, s>>>(g, d_occ, (uint16_t*)d_val);
  else
    k_init<32><<<grid, 128, 0, s>>>(g, d_occ, (uint32_t*)d_val);
}

void launch_src_init(const Geo& g, const uint32_t* rc, uint64_t n, uint32_t row0, void* d_val, int cb,
                     cudaStream_t s) {
  if (!n) return;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  if (cb == 16)
    k_src_init<16><<<blocks, 256, 0, s>>>(g, rc, n, row0, (uint16_t*)d_val);
  else
    k_src_init<32><<<blocks, 256, 0, s>>>(g, rc, n, row0, (uint32_t*)d_val);
}

void launch_block(const Geo& g, int cb, bool slab, const void* in, void* out, const uint8_t* srcmask,
                  const uint8_t* rowsrc, FlagSink flag, cudaStream_t s) {
  const uint32_t ntiles = cb == 16 ? g.nseg / 2 : g.nseg;
  const uint32_t warps = g.nbands * ntiles;
  const uint32_t blocks = (warps + kBlockThreads / 32 - 1) / (kBlockThreads / 32);
  const auto* i16 = (const uint16_t*)in;
  const auto* i32 = (const uint32_t*)in;
  if (cb == 16 && !slab)
    k_block<16, false><<<blocks, kBlockThreads, kBlockSmem, s>>>(g, i16, (uint16_t*)out, srcmask, rowsrc, flag);
  else if (cb == 16)
    k_block<16, true><<<blocks, kBlockThreads, kBlockSmem, s>>>(g, i16, (uint16_t*)out, srcmask, rowsrc, flag);
  else if (!slab)
    k_block<32, false><<<blocks, kBlockThreads, kBlockSmem, s>>>(g, i32, (uint32_t*)out, srcmask, rowsrc, flag);
  else
    k_block<32, true><<<blocks, kBlockThreads, kBlockSmem, s>>>(g, i32, (uint32_t*)out, srcmask, rowsrc, flag);
}

// TileBook::tsrc: one thread per tile, OR of its band's source-row flags over the rows its items stage
__global__ void k_tile_src(Geo g, const uint8_t* __restrict__ rowsrc, uint8_t* __restrict__ tsrc) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.ntiles()) return;
  const uint32_t b = t % g.tbands, c = t / g.tbands;
  const uint8_t* rf = rowsrc + g.tile_rowsrc(b);
  uint32_t any = 0;
  for (uint32_t r = c * kTileRows; r < c * kTileRows + kTileRows + 2 * kK && r < g.rows; ++r) any |= rf[r];
  tsrc[t] = any ? 1 : 0;
}

__global__ void k_flags_merge(uint32_t* __restrict__ f) {
  const int k = threadIdx.x;
  if (k < kFlagSlots) f[k] = min(f[k], min(f[kFlagRecvUp + k], f[kFlagRecvDn + k]));
}

void launch_flags_merge(uint32_t* d_flags, cudaStream_t s) { k_flags_merge<<<1, kFlagSlots, 0, s>>>(d_flags); }

void launch_tile_src(const Geo& g, const uint8_t* rowsrc, uint8_t* tsrc, cudaStream_t s) {
  const uint32_t n = g.ntiles();
  if (n) k_tile_src<<<(n + 255) / 256, 256, 0, s>>>(g, rowsrc, tsrc);
}

void launch_tiles_init(const Geo& g, const uint8_t* srcmask, TileBook book, cudaStream_t s) {
  const uint32_t n = g.ntiles();
  k_tiles_init<<<(n + 3) / 4, 128, 0, s>>>(g, srcmask, book);
}

__global__ void k_publish_flag(FlagSink f) {
  *reinterpret_cast<volatile uint32_t*>(f.host) = atomicExch(f.word, 0xFFFFFFFFu);
}

void launch_publish_flag(FlagSink f, cudaStream_t s) { k_publish_flag<<<1, 1, 0, s>>>(f); }

void launch_tiles_boundary(const Geo& g, int cb, const unsigned long long* state, void* f0, void* f1, uint32_t l,
                           void* dst_top, void* dst_bottom, cudaStream_t s) {
  const uint32_t warps = 2 * g.tbands;
  if (cb == 16) {
    auto* a = (const uint16_t*)f0;
    k_tiles_boundary<16><<<(warps + 3) / 4, 128, 0, s>>>(g, state, a, (const uint16_t*)f1 - a, l, (uint16_t*)dst_top,
                                                         (uint16_t*)dst_bottom);
  } else {
    auto* a = (const uint32_t*)f0;
    k_tiles_boundary<32><<<(warps + 3) / 4, 128, 0, s>>>(g, state, a, (const uint32_t*)f1 - a, l, (uint32_t*)dst_top,
                                                         (uint32_t*)dst_bottom);
  }
}

__global__ void k_peer_reduce(const uint32_t* __restrict__ vals, uint32_t n, int take_max, uint32_t* out) {
  uint32_t m = take_max ? 0u : 0xFFFFFFFFu;
  for (uint32_t i = threadIdx.x; i < n; i += 32) m = take_max ? max(m, vals[i]) : min(m, vals[i]);
  m = take_max ? __reduce_max_sync(0xffffffffu, m) : __reduce_min_sync(0xffffffffu, m);
  if (threadIdx.x == 0) *out = m;
}

void launch_peer_reduce(const uint32_t* vals, uint32_t n, int take_max, uint32_t* out, cudaStream_t s) {
  k_peer_reduce<<<1, 32, 0, s>>>(vals, n, take_max, out);
}

void launch_tiles_halo_scan(const Geo& g, int cb, const void* f0, TileBook book, uint32_t blk, cudaStream_t s) {
  const uint32_t warps = 2 * g.tbands;
  if (cb == 16)
    k_tiles_halo_scan<16><<<(warps + 3) / 4, 128, 0, s>>>(g, (const uint16_t*)f0, book, blk);
  else
    k_tiles_halo_scan<32><<<(warps + 3) / 4, 128, 0, s>>>(g, (const uint32_t*)f0, book, blk);
}

void launch_tiles_all(const Geo& g, TileBook book, uint32_t blk, uint32_t layer, int home, cudaStream_t s) {
  const uint32_t n = g.ntiles();
  k_tiles_all<<<(n + 255) / 256, 256, 0, s>>>(g, book, blk, layer, (uint32_t)home);
}

// f0/f1: the two fields; book: tile states / lists (block blk reads list[blk & 1])
#if AM_TMA
// TMA descriptors of the two 16-bit fields (box: one 8-row slot of a 128-column tile band), encoded
// through the driver entry point the runtime exposes; cached for the last (f0, f1, geometry).
static bool tile_maps(const Geo& g, void* f0, void* f1, TileMaps* out) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<Encode>(fn);
  }();
  static TileMaps cached{};
  static const void* key[2] = {nullptr, nullptr};
  static uint32_t key_pitch = 0, key_rows = 0;
  if (!encode) return false;
  if (key[0] != f0 || key[1] != f1 || key_pitch != g.pitch || key_rows != g.rows) {
    void* f[2] = {f0, f1};
    for (int i = 0; i < 2; ++i) {
      const cuuint64_t dims[2] = {g.pitch, g.rows};
      const cuuint64_t strides[1] = {(cuuint64_t)g.pitch * 2};
      const cuuint32_t box[2] = {32 * kTileWPL, kSlotRows};
      const cuuint32_t estr[2] = {1, 1};
      if (encode(&cached.box8[i], CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, f[i], dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        key[0] = key[1] = nullptr;
        return false;
      }
    }
    key[0] = f0;
    key[1] = f1;
    key_pitch = g.pitch;
    key_rows = g.rows;
  }
  *out = cached;
  return true;
}
#endif  // AM_TMA

constexpr int kTileSmemTotal = kTileSmem + kTileThreads / 32 * 16;  // + two mbarriers per warp

void launch_block_tiles(const Geo& g, int cb, int ctas, void* f0, void* f1, const uint8_t* srcmask,
                        const uint8_t* rowsrc, TileBook book, uint32_t blk, uint32_t l0, FlagSink flag,
                        FlagSink prev, bool pdl, cudaStream_t s) {
  static bool attr = [] {
    cudaFuncSetAttribute(k_block_tiles<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmemTotal);
    cudaFuncSetAttribute(k_block_tiles<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmemTotal);
    return true;
  }();
  (void)attr;
  TileMaps maps{};
  if (cb == 16) {
#if AM_TMA
    if (!tile_maps(g, f0, f1, &maps)) {
      fprintf(stderr, "actmap: cuTensorMapEncodeTiled unavailable (driver too old for TMA staging)\n");
      abort();
    }
#endif
    auto* a = (uint16_t*)f0;
    // programmatic stream serialization: the launch overlaps the previous block's tail (griddepcontrol.wait)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(kTileThreads);
    cfg.dynamicSmemBytes = kTileSmemTotal;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_block_tiles<16>, g, a, (ptrdiff_t)((uint16_t*)f1 - a), srcmask, rowsrc, book, blk, l0,
                       flag, prev, maps);
  } else {
    auto* a = (uint32_t*)f0;
    k_block_tiles<32><<<ctas, kTileThreads, kTileSmemTotal, s>>>(g, a, (uint32_t*)f1 - a, srcmask, rowsrc, book, blk,
                                                                   l0, flag, prev, maps);
  }
}

// every tile to layer l in field dst (0 = f0, 1 = f1)
void launch_tiles_finalize(const Geo& g, int cb, unsigned long long* state, void* f0, void* f1, int dst, uint32_t l,
                           uint32_t* zero, cudaStream_t s) {
  const uint32_t n = g.ntiles();
  if (cb == 16) {
    auto* a = (uint16_t*)f0;
    k_tiles_finalize<16><<<(n + 3) / 4, 128, 0, s>>>(g, state, a, (uint16_t*)f1 - a, (uint32_t)dst, l, zero);
  } else {
    auto* a = (uint32_t*)f0;
    k_tiles_finalize<32><<<(n + 3) / 4, 128, 0, s>>>(g, state, a, (uint32_t*)f1 - a, (uint32_t)dst, l, zero);
  }
}

int block_kernel_blocks_per_sm(int cb) {
  int n = 0;
  if (cb == 16)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_block<16, false>, kBlockThreads, kBlockSmem);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_block<32, false>, kBlockThreads, kBlockSmem);
  return n;
}

void launch_layer(const Geo& g, int cb, const void* in, void* out, const uint8_t* srcmask, uint32_t* flag,
                  cudaStream_t s) {
  if (cb == 16)
    k_layer<16><<<grid2d(g.W, g.H, 256), 256, 0, s>>>(g, (const uint16_t*)in, (uint16_t*)out, srcmask, flag);
  else
    k_layer<32><<<grid2d(g.W, g.H, 256), 256, 0, s>>>(g, (const uint32_t*)in, (uint32_t*)out, srcmask, flag);
}

void launch_promote(const Geo& g, const uint16_t* in, uint32_t* out, cudaStream_t s) {
  k_promote<<<148 * 8, 256, 0, s>>>(g, in, out);
}

void launch_zero_check(const Geo& g, int cb, const void* val, uint32_t* flag, cudaStream_t s) {
  const dim3 grid((g.W + 8 * 128 - 1) / (8 * 128), g.H);
  if (cb == 16)
    k_zero_check<16><<<grid, 128, 0, s>>>(g, (const uint16_t*)val, flag);
  else
    k_zero_check<32><<<grid, 128, 0, s>>>(g, (const uint32_t*)val, flag);
}

void launch_decode(const Geo& g, int cb, const void* val, uint32_t rollback, uint32_t r0, uint32_t r1,
                   uint32_t* dense, cudaStream_t s) {
  if (r1 <= r0) return;
  if (cb == 16)
    k_decode<16><<<grid2d(g.W, r1 - r0, 256), 256, 0, s>>>(g, (const uint16_t*)val, rollback, r0, dense);
  else
    k_decode<32><<<grid2d(g.W, r1 - r0, 256), 256, 0, s>>>(g, (const uint32_t*)val, rollback, r0, dense);
}

void launch_encode_dense(const Geo& g, const uint32_t* dense, const uint8_t* occ, uint32_t* val32,
                         cudaStream_t s) {
  k_encode_dense<<<grid2d(g.W, g.H, 256), 256, 0, s>>>(g, dense, occ, val32);
}

void launch_plain_layer(uint32_t W, uint32_t H, const uint8_t* occ, const uint8_t* src, const uint32_t* in,
                        uint32_t* out, cudaStream_t s) {
  k_plain_layer<<<grid2d(W, H, 256), 256, 0, s>>>(W, H, occ, src, in, out);
}

void launch_sentinel_layer(uint32_t W, uint32_t H, const uint8_t* occ, const uint8_t* src, const int32_t* in,
                           int32_t* out, cudaStream_t s) {
  k_sentinel_layer<<<grid2d(W, H, 256), 256, 0, s>>>(W, H, occ, src, in, out);
}

void launch_srcmask_dense(uint32_t W, uint32_t H, const uint32_t* rc, uint64_t n, uint8_t* m, const uint8_t* occ,
                          int* err, cudaStream_t s) {
  if (!n) return;
  k_srcmask_dense<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(W, H, rc, n, m, occ, err);
}

}  // namespace am
