// trace.cu -- K3: batched gradient-ascent path extraction, one warp per target
// (reconstruct.hpp:34-47, pins P1/P2/P5).
//
// Lanes 0..7 each fetch one of the 8 neighbours (row-major order, the order
// the tie-break enumerates) and the warp reduces them with a vote, so each
// path step costs one dependent L2/L1 round trip.  Encoded maps (produced by
// the device propagate) have a closed-form point count L_used+2-A(t), so the
// output offsets are an exclusive scan with no atomics.
#include "am_internal.cuh"

namespace am {

__constant__ int kDR[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
__constant__ int kDC[8] = {-1, 0, 1, -1, 1, -1, 0, 1};

enum : int32_t { ST_OK = 0, ST_EINVAL = 1, ST_EUNCOVERED = 2, ST_EINTERNAL = 6 };

struct Reader {
  MapView m;
  uint32_t or0 = 0, oc0 = 0;  // subtracted from every written point (a batch maze's origin: maze-local paths)
  // raw encoded cell at grid (r, c); (r, c) may lie up to the padding width outside the grid
  __device__ __forceinline__ uint32_t raw(int r, int c) const {
    const int ac = c + (int)m.g.pad;
    if (m.cell_bits == 16) return m.row<uint16_t>(r + (int)m.g.pad)[ac];
    return m.row<uint32_t>(r + (int)m.g.pad)[ac];
  }
  __device__ __forceinline__ uint32_t value(uint32_t r, uint32_t c) const {
    if (m.bt) {  // bit-plane map: covered cells hold (lref - u) mod 2^14 (lref + 1 at sources)
      uint32_t f;
      if (!m.bword(r, c, &f)) return 0u;
      return (m.layers - m.bu(r, c)) & kBTSrcU;
    }
    if (m.cell_bits == 16) {
      const uint32_t v = raw((int)r, (int)c);
      return (v & kFlag16) ? (v & 0x7FFFu) : 0u;
    }
    if (m.cell_bits == 32) {
      const uint32_t v = raw((int)r, (int)c);
      return (v & kFlag32) ? (v & kLow32) : 0u;
    }
    return static_cast<const uint32_t*>(m.val)[(size_t)r * m.g.W + c];
  }
  // encoded fields only: (r, c) may lie up to the padding width outside the grid
  __device__ __forceinline__ uint32_t value_pad(int r, int c) const {
    const uint32_t v = raw(r, c);
    if (m.cell_bits == 16) return (v & kFlag16) ? (v & 0x7FFFu) : 0u;
    return (v & kFlag32) ? (v & kLow32) : 0u;
  }
  __device__ __forceinline__ bool source(uint32_t r, uint32_t c) const {
    // a distributed map has no source mask here: on a propagated (law-abiding) map the sources are
    // exactly the cells at L+1
    if (m.dir) return value(r, c) == m.layers + 1;
    if (m.cell_bits) return m.srcmask[m.g.idx(r, c)] != 0;
    return m.srcmask[(size_t)r * m.g.W + c] != 0;
  }
  __device__ __forceinline__ bool obstacle(uint32_t r, uint32_t c) const {
    if (m.bt) {
      uint32_t f;
      (void)m.bword(r, c, &f);
      return !f;
    }
    if (m.cell_bits == 16) return !(raw((int)r, (int)c) & kFlag16);
    if (m.cell_bits == 32) return !(raw((int)r, (int)c) & kFlag32);
    return m.occ[(size_t)r * m.g.W + c] != 0;
  }
};

__device__ __forceinline__ uint64_t splitmix64(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ int32_t target_status(const Reader& rd, uint32_t r, uint32_t c) {
  if (r >= rd.m.g.H || c >= rd.m.g.W) return ST_EINVAL;  // pin P8
  if (rd.obstacle(r, c)) return ST_EINVAL;               // reconstruct.hpp:36
  if (rd.value(r, c) == 0) return ST_EUNCOVERED;         // reconstruct.hpp:37
  return ST_OK;
}

// Walks one path with a full warp.  WRITE=false only counts points.
// Returns the point count (>= 1) or 0 with *st set on failure.
template <bool WRITE>
__device__ uint64_t walk(const Reader& rd, uint32_t r, uint32_t c, int method, uint64_t seed, uint64_t limit,
                         uint32_t* out, int32_t* st) {
  const int lane = threadIdx.x & 31;
  const uint32_t W = rd.m.g.W, H = rd.m.g.H;
  uint64_t rng = seed;
  uint32_t cur = rd.value(r, c);
  uint64_t n = 1;
  if (WRITE && lane == 0) {
    out[0] = r - rd.or0;
    out[1] = c - rd.oc0;
  }
  while (!rd.source(r, c)) {
    if (n >= limit) {
      *st = ST_EINTERNAL;
      return 0;
    }
    uint32_t v = 0;
    if (lane < 8) {
      const long rr = (long)r + kDR[lane], cc = (long)c + kDC[lane];
      if (rr >= 0 && cc >= 0 && rr < (long)H && cc < (long)W) v = rd.value((uint32_t)rr, (uint32_t)cc);
    }
    int sel = -1;
    uint32_t best;
    if (method == 0) {  // simple: 8-neighbour argmax, seeded tie-break (pin P2)
      best = __reduce_max_sync(0xffffffffu, v);
      const uint32_t mask = __ballot_sync(0xffffffffu, lane < 8 && v == best);
      if (best > cur) {
        const int cnt = __popc(mask);
        int pick = 0;
        if (cnt >= 2) pick = (int)__umul64hi(splitmix64(rng), (uint64_t)cnt);
        uint32_t mm = mask;
        for (int k = 0; k < pick; ++k) mm &= mm - 1;
        sel = __ffs(mm) - 1;
      }
    } else {  // Euclidean: axis order L,R,U,D then diagonals (pin P1)
      uint32_t nb[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) nb[k] = __shfl_sync(0xffffffffu, v, k);
      const int axis[4] = {3, 4, 1, 6}, dg[4] = {0, 2, 5, 7};
      int ba = axis[0];
      uint32_t bv = nb[axis[0]];
#pragma unroll
      for (int k = 1; k < 4; ++k)
        if (nb[axis[k]] > bv) {
          bv = nb[axis[k]];
          ba = axis[k];
        }
      if (bv > cur) {
        sel = ba;
      } else {
        ba = dg[0];
        bv = nb[dg[0]];
#pragma unroll
        for (int k = 1; k < 4; ++k)
          if (nb[dg[k]] > bv) {
            bv = nb[dg[k]];
            ba = dg[k];
          }
        if (bv > cur) sel = ba;
      }
      best = bv;
    }
    if (sel < 0) {
      *st = ST_EINTERNAL;  // no ascending neighbour
      return 0;
    }
    r = (uint32_t)((long)r + kDR[sel]);
    c = (uint32_t)((long)c + kDC[sel]);
    cur = best;
    if (WRITE && lane == 0) {
      out[2 * n] = r - rd.or0;
      out[2 * n + 1] = c - rd.oc0;
    }
    ++n;
  }
  return n;
}

// Windowed walk for maps produced by the device propagation (encoded
// fields).  The warp stages a window of RAW cells around the current cell in
// shared memory (32x32 cells; 16 B vector
// loads), then takes steps inside it with one shared-memory read per
// candidate lane and two votes per step; it re-stages when the current
// cell's 3x3 neighbourhood reaches the window border (~15-31 steps per load).
// Raw cells compare like decoded activities: every free cell has the flag
// bit, so it beats any obstacle or padding cell (flag clear), and free cells
// order by activity; a cell is a source exactly when its activity is L+1
// (d = 0), so no source-mask load is needed.  Candidate lanes follow the
// reference enumerations: row-major for the simple rule (pin P2), axis order
// L,R,U,D then the diagonals for the Euclidean rule (pin P1).  Points are
// gathered 32 at a time and written by the whole warp.
#ifndef AM_TRACE_LAW
#define AM_TRACE_LAW 1
#endif
#ifndef AM_TWR
#define AM_TWR 32  // 16-bit window rows
#endif
#ifndef AM_TWC
#define AM_TWC 32  // 16-bit window columns (smaller windows stage faster; tools/ab_trace.sh)
#endif
constexpr int kWinBytes = 4096;  // shared memory per warp: a window (<= 4 KB)
#ifndef AM_TRACE_FAST
#define AM_TRACE_FAST 1  // Euclidean plane walk: linear window index, flush outside the step loop
#endif
#ifndef AM_TRACE_PLANES
#define AM_TRACE_PLANES 1  // bit-plane runs: walk on the coverage / time planes (walk_planes)
#endif

template <typename T, int WR, int WC>
__device__ uint64_t walk_smem(const Reader& rd, uint32_t r, uint32_t c, int method, uint64_t seed, uint64_t limit,
                              uint32_t* out, int32_t* st, T* win) {
  static_assert(WR * WC * sizeof(T) <= kWinBytes && WR % 32 == 0, "window");
  constexpr int kVec = 16 / sizeof(T);  // cells per 16 B vector
  const int lane = threadIdx.x & 31;
  const MapView& m = rd.m;
  const int pad = (int)m.g.pad, pitch = (int)m.g.pitch;
  const int rmax = (int)m.g.rows - pad - WR;  // window origin limits (grid coordinates)
  const uint32_t flag = sizeof(T) == 2 ? kFlag16 : kFlag32;
  const uint32_t top = flag | (m.layers + 1);  // raw value of a source
  uint64_t rng = seed;
  // candidate k (lane k < 8): 2-bit packed (d + 1) offsets, k-th pair
  const uint32_t pr_ = method == 0 ? 0xA940u : 0xA085u;  // dr: simple -1,-1,-1,0,0,1,1,1 / eucl 0,0,-1,1,-1,-1,1,1
  const uint32_t pc_ = method == 0 ? 0x9224u : 0x8858u;  // dc: simple -1,0,1,-1,1,-1,0,1 / eucl -1,1,0,0,-1,1,-1,1
  auto off = [](uint32_t pack, int k) { return (int)((pack >> (2 * k)) & 3u) - 1; };
  const int dr = off(pr_, lane & 7), dc = off(pc_, lane & 7);
  int wr = 0, wc = 0;
  bool loaded = false;
  auto stage = [&]() {
    wr = min(max((int)r - WR / 2, -pad), rmax);
    const int ac = min(max(((int)c + pad - WC / 2) & ~(kVec - 1), 0), pitch - WC);  // allocated column, 16 B aligned
    wc = ac - pad;
    __syncwarp();  // previous window fully read
#pragma unroll
    for (int h = 0; h < WR / 32; ++h) {
      const int row = lane + 32 * h;
      const uint4* p = reinterpret_cast<const uint4*>(m.row<T>(wr + row + pad) + ac);
      uint4* o = reinterpret_cast<uint4*>(win + row * WC);
#pragma unroll
      for (int q = 0; q < WC / kVec; ++q) o[q] = p[q];
    }
    __syncwarp();
    loaded = true;
  };
  uint32_t cur = m.row<T>((int)r + pad)[(int)c + pad];
  uint64_t n = 0;
  uint32_t keep_r = 0, keep_c = 0;  // point n of this lane's slot (n % 32 == lane)
  auto record = [&]() {
    if ((int)(n & 31) == lane) keep_r = r, keep_c = c;
    if ((n & 31) == 31) reinterpret_cast<uint2*>(out)[n - 31 + lane] = make_uint2(keep_r - rd.or0, keep_c - rd.oc0);
    ++n;
  };
  record();
  while (cur != top) {
    if (n >= limit) {
      *st = ST_EINTERNAL;
      return 0;
    }
    const int pr = (int)r - wr, pc = (int)c - wc;
    if (!loaded || pr < 1 || pr > WR - 2 || pc < 1 || pc > WC - 2) stage();
    const uint32_t v = lane < 8 ? (uint32_t)win[((int)r - wr + dr) * WC + ((int)c - wc + dc)] : 0u;
    int sel = -1;
    uint32_t best;
#if AM_TRACE_LAW
    // Maps from the device propagation obey the law (8-adjacent free cells differ by <= 1, every
    // ascent is exactly +1), so the maxima the rules look for are exactly the cells at cur + 1:
    // one vote per step, no max-reduction on the dependent chain.
    best = cur + 1u;
    if (method == 0) {  // simple: the row-major candidates at cur + 1, seeded tie-break (pin P2)
      uint32_t mask = __ballot_sync(0xffffffffu, lane < 8 && v == best);
      if (mask) {
        const int cnt = __popc(mask);
        int pick = 0;
        if (cnt >= 2) pick = (int)__umul64hi(splitmix64(rng), (uint64_t)cnt);
        for (int k = 0; k < pick; ++k) mask &= mask - 1;
        sel = __ffs(mask) - 1;
      }
    } else {  // Euclidean: first of L,R,U,D at cur + 1, else the first diagonal (pin P1)
      const uint32_t mask = __ballot_sync(0xffffffffu, lane < 8 && v == best);
      sel = (mask & 0xFu) ? __ffs(mask & 0xFu) - 1 : (mask ? __ffs(mask) - 1 : -1);
    }
#else
    if (method == 0) {  // simple: 8-neighbour argmax, seeded tie-break (pin P2)
      best = __reduce_max_sync(0xffffffffu, v);
      uint32_t mask = __ballot_sync(0xffffffffu, lane < 8 && v == best);
      if (best > cur) {
        const int cnt = __popc(mask);
        int pick = 0;
        if (cnt >= 2) pick = (int)__umul64hi(splitmix64(rng), (uint64_t)cnt);
        for (int k = 0; k < pick; ++k) mask &= mask - 1;
        sel = __ffs(mask) - 1;
      }
    } else {  // Euclidean: first maximum of L,R,U,D, else of the diagonals (pin P1)
      best = __reduce_max_sync(0xffffffffu, lane < 4 ? v : 0u);
      if (best > cur) {
        sel = __ffs(__ballot_sync(0xffffffffu, lane < 4 && v == best)) - 1;
      } else {
        best = __reduce_max_sync(0xffffffffu, lane >= 4 && lane < 8 ? v : 0u);
        if (best > cur) sel = __ffs(__ballot_sync(0xffffffffu, lane >= 4 && lane < 8 && v == best)) - 1;
      }
    }
#endif
    if (sel < 0) {
      *st = ST_EINTERNAL;  // no ascending neighbour
      return 0;
    }
    r = (uint32_t)((int)r + off(pr_, sel));
    c = (uint32_t)((int)c + off(pc_, sel));
    cur = best;
    record();
  }
  // flush the partial group of points
  const uint64_t base = n & ~(uint64_t)31;
  if (base + lane < n) reinterpret_cast<uint2*>(out)[base + lane] = make_uint2(keep_r - rd.or0, keep_c - rd.oc0);
  if (!rd.source(r, c)) *st = ST_EINTERNAL;  // a non-source at the top value would violate the law
  return n;
}

// Euclidean walk, two steps per iteration (law-abiding device maps, see walk_smem):
// lanes 0-24 read the 5x5 cells around the current cell, one ballot marks the
// cells at cur + 1 and one the cells at cur + 2; the first step is the first
// of L, R, U, D (else of the diagonals) at cur + 1, the second the same rule
// among the chosen cell's neighbours at cur + 2 -- both decided from the two
// masks, so two steps cost one shared-memory read and two votes.
#ifndef AM_TRACE_2STEP
#define AM_TRACE_2STEP 1
#endif
// first set bit of m among lanes base + {-1, +1, -5, +5} (L, R, U, D), else base + {-6, -4, +4, +6}
__device__ __forceinline__ int eucl_pick5(uint32_t m, int base) {
  const int ax[4] = {-1, 1, -5, 5}, dg[4] = {-6, -4, 4, 6};
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if ((m >> (base + ax[k])) & 1u) return base + ax[k];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if ((m >> (base + dg[k])) & 1u) return base + dg[k];
  return -1;
}

template <typename T, int WR, int WC>
__device__ uint64_t walk_eucl2(const Reader& rd, uint32_t r, uint32_t c, uint64_t limit, uint32_t* out, int32_t* st,
                               T* win) {
  static_assert(WR * WC * sizeof(T) <= kWinBytes && WR % 32 == 0, "window");
  constexpr int kVec = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const MapView& m = rd.m;
  const int pad = (int)m.g.pad, pitch = (int)m.g.pitch;
  const int rmax = (int)m.g.rows - pad - WR;
  const uint32_t flag = sizeof(T) == 2 ? kFlag16 : kFlag32;
  const uint32_t top = flag | (m.layers + 1);  // raw value of a source
  const int dr = lane / 5 - 2, dc = lane % 5 - 2;  // this lane's cell of the 5x5 (lanes < 25)
  int wr = 0, wc = 0;
  bool loaded = false;
  auto stage = [&]() {
    wr = min(max((int)r - WR / 2, -pad), rmax);
    const int ac = min(max(((int)c + pad - WC / 2) & ~(kVec - 1), 0), pitch - WC);
    wc = ac - pad;
    __syncwarp();
#pragma unroll
    for (int h = 0; h < WR / 32; ++h) {
      const int row = lane + 32 * h;
      const uint4* p = reinterpret_cast<const uint4*>(m.row<T>(wr + row + pad) + ac);
      uint4* o = reinterpret_cast<uint4*>(win + row * WC);
#pragma unroll
      for (int q = 0; q < WC / kVec; ++q) o[q] = p[q];
    }
    __syncwarp();
    loaded = true;
  };
  uint32_t cur = m.row<T>((int)r + pad)[(int)c + pad];
  uint64_t n = 0;
  uint32_t keep_r = 0, keep_c = 0;
  auto record = [&]() {
    if ((int)(n & 31) == lane) keep_r = r, keep_c = c;
    if ((n & 31) == 31) reinterpret_cast<uint2*>(out)[n - 31 + lane] = make_uint2(keep_r - rd.or0, keep_c - rd.oc0);
    ++n;
  };
  record();
  while (cur != top) {
    if (n >= limit) {
      *st = ST_EINTERNAL;
      return 0;
    }
    const int pr = (int)r - wr, pc = (int)c - wc;
    if (!loaded || pr < 2 || pr > WR - 3 || pc < 2 || pc > WC - 3) stage();
    const uint32_t v = lane < 25 ? (uint32_t)win[((int)r - wr + dr) * WC + ((int)c - wc + dc)] : 0u;
    const uint32_t m1 = __ballot_sync(0xffffffffu, lane < 25 && v == cur + 1u);
    const uint32_t m2 = __ballot_sync(0xffffffffu, lane < 25 && v == cur + 2u);
    const int s1 = eucl_pick5(m1, 12);
    if (s1 < 0) {
      *st = ST_EINTERNAL;  // no ascending neighbour
      return 0;
    }
    r = (uint32_t)((int)r + s1 / 5 - 2);
    c = (uint32_t)((int)c + s1 % 5 - 2);
    cur += 1u;
    record();
    if (cur == top || n >= limit) continue;  // reached a source (or the count says so: checked above)
    const int s2 = eucl_pick5(m2, s1);
    if (s2 < 0) {
      *st = ST_EINTERNAL;
      return 0;
    }
    r = (uint32_t)((int)r + s2 / 5 - s1 / 5);
    c = (uint32_t)((int)c + s2 % 5 - s1 % 5);
    cur += 1u;
    record();
  }
  const uint64_t base = n & ~(uint64_t)31;
  if (base + lane < n) reinterpret_cast<uint2*>(out)[base + lane] = make_uint2(keep_r - rd.or0, keep_c - rd.oc0);
  if (!rd.source(r, c)) *st = ST_EINTERNAL;
  return n;
}

// Walk on the planes of a bit-plane run (bits.cu): coverage C and the two low bits of u = t - 1 (the
// layer a cell was covered at, minus one; sources kBTSrcU == -1 mod 4).  On a propagated map an
// 8-neighbour n is an ascent candidate of c (activity + 1) exactly when both are covered and
// u_c - u_n == 1 (activities of covered 8-neighbours differ by <= 1, activity = lref - u), and mod 4 that
// is two LOP3s per 32 cells: (a0 ^ b0) & ~(a1 ^ b1 ^ b0) with a = u_c, b = u_n.  A warp stages a 64 x 64
// window (two rows of two words per lane: per word the covered word of the tile's home plane, by its state,
// and time planes 0 and 1 -- the propagation's own planes, read while k_bits_finalize encodes the field),
// builds every cell's candidates for all 8 directions with shifts and shuffles of whole words and stores
// one 16 B record per word in shared memory.  Euclidean rule (pin P1): the first candidate of L, R, U, D,
// UL, UR, DL, DR, kept as four move planes (row +1, row -1, column +1, column -1), so a step is one
// broadcast 16 B shared-memory read, four shifts and two subtractions; the window's border cells get no
// move, so "no move" means re-stage (8 cells behind the cell in its direction of travel) or, right after a
// re-stage, a map without an ascending neighbour.  Simple rule (pin P2): the 8 candidate words (two
// records), the seeded tie-break per step.  Points are held in registers (lane k: point k mod 32), written by the
// whole warp every 32 points.
constexpr int kPR = 64, kPW = 2;  // plane window: rows, 32-cell words per row (two rows per lane)
constexpr int kPTab = kPR * kPW * 2 * 16;  // window records (simple rule: two per word)
static_assert(kPTab <= kWinBytes, "plane window records");

// Stages the plane window around (r, c), 8 cells behind it in its direction of travel (ldr, ldc), and
// builds the window records (out of line: the step loop stays short).
template <int METHOD>
__device__ __noinline__ int2 stage_planes(const uint4* __restrict__ bp, const uint32_t* __restrict__ bt,
                                          const unsigned long long* __restrict__ bstate, uint32_t H, uint32_t wpr,
                                          uint32_t tbands, uint32_t prows, uint32_t r, uint32_t c, int ldr, int ldc,
                                          uint4* tab) {
  // scalars by value and the origin returned in registers: a reference to the MapView would put the
  // whole view in local memory for this out-of-line call
  const int lane = threadIdx.x & 31;
  const int orr = ldr < 0 ? kPR - 8 : (ldr > 0 ? 8 : kPR / 2);
  // columns: the origin is floored to a word, so the cell lands in [orc, orc + 31]
  const int orc = ldc < 0 ? 32 * kPW - 33 : (ldc > 0 ? 1 : 16 * kPW - 16);
  const int wr = (int)r - orr;
  const int wc = (((int)c - orc) >> 5) * 32;  // arithmetic shift: floor
  uint32_t X[2][kPW], A0[2][kPW], A1[2][kPW];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int x = 0; x < kPW; ++x) {
      const int gr = wr + 2 * lane + i, gw = (wc >> 5) + x;
      X[i][x] = A0[i][x] = A1[i][x] = 0u;
      if (gr >= 0 && gr < (int)H && gw >= 0 && gw < (int)wpr) {  // planes are read-only here: L1
        const size_t pw = (size_t)gr * wpr + gw;  // time planes: row-major
        const uint4 p = __ldg(bp + (AM_BITS_PCM ? (size_t)gw * prows + gr : pw));  // {cov 0, cov 1, free, -}
        const uint2 u01 = __ldg(reinterpret_cast<const uint2*>(bt + pw * 16));  // t - 1, bits 0 and 1
        const uint32_t st = (uint32_t)__ldg(bstate + ((uint32_t)gr / kBTR) * tbands + (uint32_t)gw / kBTW);
        X[i][x] = st == 0u ? 0u : (st & 1u) ? p.y : p.x;
        A0[i][x] = u01.x;
        A1[i][x] = u01.y;
      }
    }
  // rows above / below each of the lane's two rows
  uint32_t UX[2][kPW], U0[2][kPW], U1[2][kPW], DX[2][kPW], D0[2][kPW], D1[2][kPW];
#pragma unroll
  for (int x = 0; x < kPW; ++x) {
    UX[0][x] = __shfl_up_sync(0xffffffffu, X[1][x], 1);
    U0[0][x] = __shfl_up_sync(0xffffffffu, A0[1][x], 1);
    U1[0][x] = __shfl_up_sync(0xffffffffu, A1[1][x], 1);
    DX[1][x] = __shfl_down_sync(0xffffffffu, X[0][x], 1);
    D0[1][x] = __shfl_down_sync(0xffffffffu, A0[0][x], 1);
    D1[1][x] = __shfl_down_sync(0xffffffffu, A1[0][x], 1);
    UX[1][x] = X[0][x], U0[1][x] = A0[0][x], U1[1][x] = A1[0][x];
    DX[0][x] = X[1][x], D0[0][x] = A0[1][x], D1[0][x] = A1[1][x];
  }
  __syncwarp();  // the previous window's records are no longer read
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int x = 0; x < kPW; ++x) {
      // neighbour planes of word x of a row (dc = -1: bit j from column j - 1; +1: from j + 1)
      auto shl = [&](const uint32_t(&w)[kPW]) { return x > 0 ? __funnelshift_l(w[x - 1], w[x], 1) : w[x] << 1; };
      auto shr = [&](const uint32_t(&w)[kPW]) {
        return x < kPW - 1 ? __funnelshift_r(w[x], w[x + 1], 1) : w[x] >> 1;
      };
      const uint32_t a0 = A0[i][x], a1 = A1[i][x];
      auto cand = [&](uint32_t nc, uint32_t n0, uint32_t n1) { return nc & (a0 ^ n0) & ~(a1 ^ n1 ^ n0); };
      const uint32_t cL = cand(shl(X[i]), shl(A0[i]), shl(A1[i]));
      const uint32_t cR = cand(shr(X[i]), shr(A0[i]), shr(A1[i]));
      const uint32_t cU = cand(UX[i][x], U0[i][x], U1[i][x]);
      const uint32_t cD = cand(DX[i][x], D0[i][x], D1[i][x]);
      const uint32_t cUL = cand(shl(UX[i]), shl(U0[i]), shl(U1[i]));
      const uint32_t cUR = cand(shr(UX[i]), shr(U0[i]), shr(U1[i]));
      const uint32_t cDL = cand(shl(DX[i]), shl(D0[i]), shl(D1[i]));
      const uint32_t cDR = cand(shr(DX[i]), shr(D0[i]), shr(D1[i]));
      // the window's border cells get no move (their neighbourhoods are not all staged)
      const int wrow = 2 * lane + i;
      const uint32_t inner = (wrow == 0 || wrow == kPR - 1) ? 0u
                             : (x == 0 ? 0xFFFFFFFEu : 0xFFFFFFFFu) & (x == kPW - 1 ? 0x7FFFFFFFu : 0xFFFFFFFFu);
      const int e = wrow * kPW + x;
      if (METHOD == 1) {  // first of L, R, U, D, UL, UR, DL, DR
        uint32_t taken = cL;
        const uint32_t sR = cR & ~taken;
        taken |= cR;
        const uint32_t sU = cU & ~taken;
        taken |= cU;
        const uint32_t sD = cD & ~taken;
        taken |= cD;
        const uint32_t sUL = cUL & ~taken;
        taken |= cUL;
        const uint32_t sUR = cUR & ~taken;
        taken |= cUR;
        const uint32_t sDL = cDL & ~taken;
        taken |= cDL;
        const uint32_t sDR = cDR & ~taken;
        tab[e] = make_uint4((sD | sDL | sDR) & inner, (sU | sUL | sUR) & inner, (sR | sUR | sDR) & inner,
                            (cL | sUL | sDL) & inner);  // row +1, row -1, column +1, column -1
      } else {  // simple: row-major candidate words (-1,-1) (-1,0) (-1,1) (0,-1) | (0,1) (1,-1) (1,0) (1,1)
        tab[2 * e] = make_uint4(cUL & inner, cU & inner, cUR & inner, cL & inner);
        tab[2 * e + 1] = make_uint4(cR & inner, cDL & inner, cD & inner, cDR & inner);
      }
    }
  __syncwarp();
  return make_int2(wr, wc);
}

template <int METHOD>
__device__ uint64_t walk_planes(const Reader& rd, uint32_t r, uint32_t c, uint64_t seed, uint32_t limit,
                                uint32_t* out, int32_t* st, uint4* tab) {
  const int lane = threadIdx.x & 31;
  const MapView& m = rd.m;
  // simple rule: direction k (row-major) -> (dr, dc), 2-bit packed (d + 1)
  constexpr uint32_t PR = 0xA940u, PC = 0x9224u;
  uint64_t rng = seed;
  int wr = 0, wc = 0, ldr = 0, ldc = 0;
  const uint4* const bp = m.bp;
  const uint32_t* const bt = m.bt;
  const unsigned long long* const bs = m.bstate;
  const uint32_t bh = m.bg.H, bw = m.bg.wpr, btb = m.bg.tbands, brows = m.bg.rows;
  auto stage = [&]() {
    const int2 o = stage_planes<METHOD>(bp, bt, bs, bh, bw, btb, brows, r, c, ldr, ldc, tab);
    wr = o.x;
    wc = o.y;
  };
  // points in registers: lane k holds point k mod 32 of the current group of 32 (a predicated move per
  // step, no branch), and the warp writes a group at once
  uint2 pt = make_uint2(r, c);
  auto flush = [&](uint32_t upto) {  // points [(upto - 1) & ~31, upto) are held by the lanes
    const uint32_t base = (upto - 1) & ~31u;
    if (base + lane < upto) reinterpret_cast<uint2*>(out)[base + lane] = make_uint2(pt.x - rd.or0, pt.y - rd.oc0);
  };
  int lr = 0, lc = 0;
  bool fresh = false;  // the window was staged for the current cell
  stage();
  lr = (int)r - wr;
  lc = (int)c - wc;
  fresh = true;
  uint32_t n = 1;
  if (METHOD == 1 && AM_TRACE_FAST) {
    // Euclidean rule, tight loop: the cell as one window index pos = row * 64 + column (its record is word
    // pos >> 5, bit pos & 31), one index update per step, and the 32-point flush out of the step loop (the
    // inner loop runs to the next multiple of 32 or the end of the path)
    static_assert(kPW == 2, "window rows of 64 cells");
    int pos = lr * 64 + lc;
    while (n < limit) {
      const uint32_t stop = min(limit, (n | 31u) + 1u);
      bool leave = false;
      while (n < stop) {
        const uint4 q = tab[pos >> 5];
        const uint32_t b = (uint32_t)pos & 31u;
        const uint32_t dp = (q.x >> b) & 1u, dm = (q.y >> b) & 1u, cp = (q.z >> b) & 1u, cm = (q.w >> b) & 1u;
        if (!(dp | dm | cp | cm)) {
          leave = true;
          break;
        }
        const int dr = (int)dp - (int)dm, dc = (int)cp - (int)cm;
        pos += dr * 64 + dc;
        r = (uint32_t)((int)r + dr);
        c = (uint32_t)((int)c + dc);
        ldr = dr;
        ldc = dc;
        pt = lane == (int)(n & 31) ? make_uint2(r, c) : pt;
        ++n;
        fresh = false;
      }
      if (leave) {  // no move inside this window: re-stage (SPEC.md:205 if it was just staged)
        if (fresh) {
          *st = ST_EINTERNAL;
          return 0;
        }
        stage();
        pos = ((int)r - wr) * 64 + ((int)c - wc);
        fresh = true;
        continue;
      }
      if ((n & 31) == 0) flush(n);
    }
  }
  if (METHOD == 0 && AM_TRACE_FAST) {
    // simple rule (pin P2), the same tight loop: the 8 candidate bits of the cell from its two records,
    // the seeded draw only when >= 2 candidates tie
    static_assert(kPW == 2, "window rows of 64 cells");
    int pos = lr * 64 + lc;
    while (n < limit) {
      const uint32_t stop = min(limit, (n | 31u) + 1u);
      bool leave = false;
      while (n < stop) {
        const uint4 q0 = tab[2 * (pos >> 5)], q1 = tab[2 * (pos >> 5) + 1];
        const uint32_t b = (uint32_t)pos & 31u;
        uint32_t mask = ((q0.x >> b) & 1u) | ((q0.y >> b) & 1u) << 1 | ((q0.z >> b) & 1u) << 2 |
                        ((q0.w >> b) & 1u) << 3 | ((q1.x >> b) & 1u) << 4 | ((q1.y >> b) & 1u) << 5 |
                        ((q1.z >> b) & 1u) << 6 | ((q1.w >> b) & 1u) << 7;
        if (!mask) {
          leave = true;
          break;
        }
        const int cnt = __popc(mask);
        if (cnt >= 2) {
          const int pick = (int)__umul64hi(splitmix64(rng), (uint64_t)cnt);
          for (int j = 0; j < pick; ++j) mask &= mask - 1;
        }
        const int k = __ffs(mask) - 1;
        const int dr = (int)((PR >> (2 * k)) & 3u) - 1, dc = (int)((PC >> (2 * k)) & 3u) - 1;
        pos += dr * 64 + dc;
        r = (uint32_t)((int)r + dr);
        c = (uint32_t)((int)c + dc);
        ldr = dr;
        ldc = dc;
        pt = lane == (int)(n & 31) ? make_uint2(r, c) : pt;
        ++n;
        fresh = false;
      }
      if (leave) {
        if (fresh) {
          *st = ST_EINTERNAL;
          return 0;
        }
        stage();
        pos = ((int)r - wr) * 64 + ((int)c - wc);
        fresh = true;
        continue;
      }
      if ((n & 31) == 0) flush(n);
    }
  }
  while (n < limit) {
    int dr, dc;
    for (;;) {
      const int e = lr * kPW + (lc >> 5), b = lc & 31;
      if (METHOD == 1) {
        const uint4 q = tab[e];
        const uint32_t dp = q.x >> b, dm = q.y >> b, cp = q.z >> b, cm = q.w >> b;
        dr = (int)(dp & 1u) - (int)(dm & 1u);
        dc = (int)(cp & 1u) - (int)(cm & 1u);
        if ((dp | dm | cp | cm) & 1u) break;
      } else {
        const uint4 q0 = tab[2 * e], q1 = tab[2 * e + 1];
        uint32_t mask = ((q0.x >> b) & 1u) | ((q0.y >> b) & 1u) << 1 | ((q0.z >> b) & 1u) << 2 |
                        ((q0.w >> b) & 1u) << 3 | ((q1.x >> b) & 1u) << 4 | ((q1.y >> b) & 1u) << 5 |
                        ((q1.z >> b) & 1u) << 6 | ((q1.w >> b) & 1u) << 7;
        if (mask) {
          const int cnt = __popc(mask);
          int pick = 0;
          if (cnt >= 2) pick = (int)__umul64hi(splitmix64(rng), (uint64_t)cnt);
          for (int j = 0; j < pick; ++j) mask &= mask - 1;
          const int k = __ffs(mask) - 1;
          dr = (int)((PR >> (2 * k)) & 3u) - 1;
          dc = (int)((PC >> (2 * k)) & 3u) - 1;
          break;
        }
      }
      if (fresh) {  // staged around this cell and still no move: no ascending neighbour
        *st = ST_EINTERNAL;
        return 0;
      }
      stage();
      lr = (int)r - wr;
      lc = (int)c - wc;
      fresh = true;
    }
    fresh = false;
    ldr = dr;
    ldc = dc;
    r = (uint32_t)((int)r + dr);
    c = (uint32_t)((int)c + dc);
    lr += dr;
    lc += dc;
    pt = lane == (int)(n & 31) ? make_uint2(r, c) : pt;
    ++n;
    if ((n & 31) == 0) flush(n);
  }
  if (n & 31) flush(n);
  if (!rd.source(r, c)) *st = ST_EINTERNAL;  // the point count is exact on a law-abiding map
  return n;
}

// Encoded maps: closed-form count L+2-A(t).  Plain maps: a counting walk.
__global__ void k_path_counts(MapView m, const uint32_t* __restrict__ tgt, uint64_t n, int method,
                              uint64_t seed, uint64_t* __restrict__ counts, int32_t* __restrict__ status) {
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= n) return;
  const int lane = threadIdx.x & 31;
  Reader rd{m};
  const uint32_t r = tgt[2 * w], c = tgt[2 * w + 1];
  int32_t st = target_status(rd, r, c);
  uint64_t cnt = 0;
  if (st == ST_OK) {
    if (m.cell_bits) {
      cnt = (uint64_t)m.layers + 2 - rd.value(r, c);
    } else {
      cnt = walk<false>(rd, r, c, method, seed, 0xFFFFFFFFFFFFull, nullptr, &st);
    }
  }
  if (lane == 0) {
    counts[w] = st == ST_OK ? cnt : 0;
    status[w] = st;
  }
}

// One target's path, by one warp.
__device__ __forceinline__ void trace_one(const MapView& m, const uint32_t* __restrict__ tgt, uint64_t w, int method,
                                          uint64_t seed, const uint64_t* __restrict__ offsets, uint32_t* __restrict__ pts,
                                          int32_t* __restrict__ status, uint64_t cap, uint8_t* win) {
  if (status[w] != ST_OK) return;
  Reader rd{m};
  const uint64_t off = offsets[w], limit = offsets[w + 1] - off;
  if (offsets[w + 1] > cap) {  // the caller's point buffer ends before this path: report, never write past it
    if ((threadIdx.x & 31) == 0) status[w] = ST_EINVAL;
    return;
  }
  int32_t st = ST_OK;
  if (m.cell_h) {  // mazes packed on a lattice: points in the coordinates of the target's maze
    rd.or0 = tgt[2 * w] / m.cell_h * m.cell_h;
    rd.oc0 = tgt[2 * w + 1] / m.cell_w * m.cell_w;
  }
  const bool planes = AM_TRACE_PLANES && m.bt && m.cell_bits == 16 && !m.dir;
  const uint64_t got = planes ? (method == 1 ? walk_planes<1>(rd, tgt[2 * w], tgt[2 * w + 1], seed, (uint32_t)limit,
                                                              pts + 2 * off, &st, reinterpret_cast<uint4*>(win))
                                             : walk_planes<0>(rd, tgt[2 * w], tgt[2 * w + 1], seed, (uint32_t)limit,
                                                              pts + 2 * off, &st, reinterpret_cast<uint4*>(win)))
                       : AM_TRACE_2STEP && method == 1 && m.cell_bits == 16
                           ? walk_eucl2<uint16_t, AM_TWR, AM_TWC>(rd, tgt[2 * w], tgt[2 * w + 1], limit, pts + 2 * off,
                                                                  &st, (uint16_t*)win)
                       : m.cell_bits == 16 ? walk_smem<uint16_t, AM_TWR, AM_TWC>(rd, tgt[2 * w], tgt[2 * w + 1], method, seed,
                                                                       limit, pts + 2 * off, &st, (uint16_t*)win)
                       : m.cell_bits == 32
                           ? walk_smem<uint32_t, 32, 32>(rd, tgt[2 * w], tgt[2 * w + 1], method, seed, limit,
                                                         pts + 2 * off, &st, (uint32_t*)win)
                           : walk<true>(rd, tgt[2 * w], tgt[2 * w + 1], method, seed, limit, pts + 2 * off, &st);
  if ((threadIdx.x & 31) == 0) {
    if (st != ST_OK) status[w] = st;
    else if (got != limit) status[w] = ST_EINTERNAL;
  }
}

// order == nullptr: warp w traces target w.  Otherwise the warps take targets from order[] (longest paths
// first, k_trace_order) through the counter *next: the walk time is set by the longest path, and every
// warp sharing its SM sub-partition slows it down, so few warps per sub-partition with the longest paths
// started first finish soonest (greedy longest-processing-time scheduling).
// sched (when order is set): [0] the counter, [1] whether k_trace_order chose the ordered mode; in that mode
// only the first `workers` warps run.
__global__ void k_trace(MapView m, const uint32_t* __restrict__ tgt, uint64_t n, int method, uint64_t seed,
                        const uint64_t* __restrict__ offsets, uint32_t* __restrict__ pts,
                        int32_t* __restrict__ status, uint64_t cap, const uint32_t* __restrict__ order,
                        uint32_t* sched, uint32_t workers) {
  __shared__ __align__(16) uint8_t wins[4][kWinBytes];  // one window per warp (128-thread CTAs)
  uint8_t* win = wins[(threadIdx.x >> 5) & 3];
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  if (!order || !__ldcg(sched + 1)) {
    if (gw < n) trace_one(m, tgt, gw, method, seed, offsets, pts, status, cap, win);
    return;
  }
  if (gw >= workers) return;
  uint32_t* next = sched;
  const int lane = threadIdx.x & 31;
  for (;;) {
    uint32_t i = 0;
    if (lane == 0) i = atomicAdd(next, 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= n) return;
    trace_one(m, tgt, order[i], method, seed, offsets, pts, status, cap, win);
    __syncwarp();
  }
}

// Targets in order of decreasing path length (offsets[i + 1] - offsets[i], exact from the closed-form
// counts), bucketed into kOrderBuckets length classes: a histogram, an exclusive scan and a scatter in one
// CTA.  sched: kOrderBuckets + 1 words (the bucket cursors, then the trace counter, reset here).
constexpr int kOrderBuckets = 1024;
// The ordered mode pays only when the longest path is long against the mean work of a worker warp
// (total points / workers): many short paths (C5) run faster one warp per target.
__global__ void __launch_bounds__(1024) k_trace_order(const uint64_t* __restrict__ offsets, uint64_t n,
                                                      uint32_t* __restrict__ order, uint32_t* __restrict__ sched,
                                                      uint32_t workers) {
  __shared__ uint32_t hist[kOrderBuckets];
  __shared__ uint64_t maxlen_s;
  const int t = threadIdx.x;
  for (int b = t; b < kOrderBuckets; b += blockDim.x) hist[b] = 0;
  if (t == 0) maxlen_s = 0;
  __syncthreads();
  unsigned long long mx = 0;
  for (uint64_t i = t; i < n; i += blockDim.x) mx = max(mx, (unsigned long long)(offsets[i + 1] - offsets[i]));
  atomicMax(reinterpret_cast<unsigned long long*>(&maxlen_s), mx);
  __syncthreads();
  const bool ordered = 2 * maxlen_s * workers >= offsets[n];
  if (t == 0) {
    sched[kOrderBuckets] = 0;
    sched[kOrderBuckets + 1] = ordered ? 1u : 0u;
  }
  if (!ordered) return;
  const uint64_t span = maxlen_s + 1;
  auto bucket = [&](uint64_t i) {  // longest first
    const uint64_t len = offsets[i + 1] - offsets[i];
    return kOrderBuckets - 1 - (int)(len * kOrderBuckets / span);
  };
  for (uint64_t i = t; i < n; i += blockDim.x) atomicAdd(&hist[bucket(i)], 1u);
  __syncthreads();
  if (t == 0) {  // 1024 buckets: a serial scan is a few microseconds
    uint32_t acc = 0;
    for (int b = 0; b < kOrderBuckets; ++b) {
      const uint32_t v = hist[b];
      hist[b] = acc;
      acc += v;
    }
  }
  __syncthreads();
  for (uint64_t i = t; i < n; i += blockDim.x) order[atomicAdd(&hist[bucket(i)], 1u)] = (uint32_t)i;
}

void launch_path_counts(const MapView& m, const uint32_t* tgt, uint64_t n, int method, uint64_t seed,
                        uint64_t* counts, int32_t* status, cudaStream_t s) {
  if (!n) return;
  const unsigned blocks = (unsigned)((n * 32 + 127) / 128);
  k_path_counts<<<blocks, 128, 0, s>>>(m, tgt, n, method, seed, counts, status);
}



#ifndef AM_TRACE_SCHED
#define AM_TRACE_SCHED 1  // longest-first scheduling of the targets (k_trace_order)
#endif
#ifndef AM_TRACE_WPS
#define AM_TRACE_WPS 2  // warps per SM sub-partition when the targets are scheduled longest-first
#endif
void launch_trace(const MapView& m, const uint32_t* tgt, uint64_t n, int method, uint64_t seed,
                  const uint64_t* offsets, uint32_t* pts, int32_t* status, cudaStream_t s, uint64_t cap,
                  uint32_t* order, uint32_t* sched, int sms) {
  if (!n) return;
  const uint64_t blocks = (n * 32 + 127) / 128;
  const uint64_t sched_blocks = (uint64_t)sms * AM_TRACE_WPS;  // 4 warps per CTA, one CTA per sub-partition
  if (AM_TRACE_SCHED && order && sched && sms > 0 && blocks > sched_blocks && n < (1ull << 32)) {
    const uint32_t workers = (uint32_t)sched_blocks * 4;
    k_trace_order<<<1, 1024, 0, s>>>(offsets, n, order, sched, workers);
    k_trace<<<(unsigned)blocks, 128, 0, s>>>(m, tgt, n, method, seed, offsets, pts, status, cap, order,
                                             sched + kOrderBuckets, workers);
    return;
  }
  k_trace<<<(unsigned)blocks, 128, 0, s>>>(m, tgt, n, method, seed, offsets, pts, status, cap, nullptr, nullptr, 0);
}

}  // namespace am

namespace am {
// Exclusive scan of n counts into offsets[0..n] (single CTA; n is the target
// count, a few thousand), so offsets never leave the device.
__global__ void k_scan(const uint64_t* __restrict__ counts, uint64_t n, uint64_t* __restrict__ offsets) {
  __shared__ uint64_t part[1024];
  const uint64_t per = (n + blockDim.x - 1) / blockDim.x;
  const uint64_t b = threadIdx.x * per, e = b + per < n ? b + per : n;
  uint64_t s = 0;
  for (uint64_t i = b; i < e; ++i) s += counts[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (unsigned d = 1; d < blockDim.x; d <<= 1) {
    uint64_t v = threadIdx.x >= d ? part[threadIdx.x - d] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  uint64_t run = part[threadIdx.x] - s;
  for (uint64_t i = b; i < e; ++i) {
    offsets[i] = run;
    run += counts[i];
  }
  if (threadIdx.x == blockDim.x - 1) offsets[n] = part[threadIdx.x];
}

void launch_scan(const uint64_t* counts, uint64_t n, uint64_t* offsets, cudaStream_t s) {
  k_scan<<<1, 1024, 0, s>>>(counts, n, offsets);
}
}  // namespace am
