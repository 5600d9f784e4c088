// bits.cu -- bit-plane active-tile propagation.
//
// The layer stack of propagate.hpp:34-38, started from the initial map
// (activity.hpp:20-21), obeys the closed form A_L(c) = max(0, L+1-d(c)) with
// d the 8-connected multi-source hop distance through free cells
// (activity.hpp:12-14; pinned against a BFS by the oracle
// tests).  A layer therefore changes coverage only: the set of covered cells
// grows by one 3x3 dilation restricted to free cells, and every covered cell
// gains exactly +1.  So the propagation runs on two 1-bit planes -- free (F,
// static) and covered (C) -- 32 cells per 32-bit word: one layer is
//   C' = (v | v<<1 | v>>1) & F,  v = C[r-1] | C[r] | C[r+1]
// i.e. one LOP3, two funnel shifts and two logic ops per 32 cells.  The only
// per-cell state besides the planes is the layer t at which a cell became
// covered; it is written exactly once, straight into the encoded 16-bit field
// the rest of the library reads (flag | activity relative to a reference layer
// count lref: a = lref + 1 - t), so no decode pass follows the run.
//
// Work is organised like the 16-bit tile kernel: temporally blocked (kBK
// layers per launch, tile + kBK-deep halo in registers), exact active-tile
// skipping (a tile is processed in block b+1 only if a cell covered in the last
// layer of block b lies within kBK of it), self-listing tiles, programmatic
// dependent launches and one fixed-point word per block.  A warp holds a
// 32*kBRPL-row x (kBTW+2)-word region: lane i owns rows i*kBRPL .. +kBRPL-1,
// vertical neighbours come from the adjacent lanes (two shuffles per word
// column and layer), horizontal ones from the lane's own words.
#include <cstdlib>

#include "am_internal.cuh"

namespace am {

BitGeo make_bit_geo(uint32_t W, uint32_t H) {
  BitGeo b{};
  b.W = W;
  b.H = H;
  b.nchunks = (H + kBTR - 1) / kBTR;
  b.tbands = (W + 32 * kBTW - 1) / (32 * kBTW);
  b.wpr = b.tbands * kBTW;
  b.rows = b.nchunks * kBTR;
  return b;
}

namespace {

#ifndef AM_BITS_PACKH
#define AM_BITS_PACKH 1
#endif
// words per region row: the tile's kBTW words and the horizontal halo.  Packed (default): one word, bits
// 16-31 = the kBK cells left of the tile, bits 0-15 = the kBK cells right of it, index 0, and the row is a
// ring (word 0's left neighbour is word kBTW, word kBTW's right neighbour is word 0).  The two halves meet
// at the outermost halo cells, whose errors travel one cell per layer and reach the tile after kBK + 1
// layers, never within a block.  Unpacked: one full word each side (index 0 and kBTW + 1).
static_assert(!AM_BITS_PACKH || kBK == 16, "packed halo: 16 cells each side");
constexpr int kBNW = AM_BITS_PACKH ? kBTW + 1 : kBTW + 2;
__device__ __forceinline__ constexpr int bleft(int x) { return AM_BITS_PACKH && x == 0 ? kBNW - 1 : x - 1; }
__device__ __forceinline__ constexpr int bright(int x) { return AM_BITS_PACKH && x == kBNW - 1 ? 0 : x + 1; }
constexpr int kBNJ = kBK == 8 ? 3 : kBK == 16 ? 4 : 5;  // bit planes of the in-block layer index
static_assert(kBK == 8 || kBK == 16 || kBK == 32, "layers per bit block");
static_assert(kBTR >= kBK && kBTR > 0, "tiles at least kBK rows");
#ifndef AM_BITS_THREADS
#define AM_BITS_THREADS 128
#endif
constexpr int kBThreads = AM_BITS_THREADS;
constexpr int kBTsmBytes = kBThreads / 32 * kBTR * kBTW * 4 * 16;  // time-plane staging (dynamic smem)
#ifndef AM_BITS_RUN_THREADS
#define AM_BITS_RUN_THREADS 256
#endif
constexpr int kBRunThreads = AM_BITS_RUN_THREADS;                    // k_bits_run: one CTA per SM
constexpr int kBRunSmem = kBRunThreads / 32 * kBTR * kBTW * 4 * 16;
#ifndef AM_BITS_PREF
#define AM_BITS_PREF 0  // the next item's states and region load during the current item's bookkeeping
                        // (measured: C4 +3.5%, the longer live ranges spill)
#endif
#ifndef AM_BITS_DONE
#define AM_BITS_DONE 1  // tiles whose free cells are all covered are never listed again
#endif
#ifndef AM_BITS_STATS
#define AM_BITS_STATS 0  // experiment: item counters in stat[3..5]
#endif
#ifndef AM_BITS_FRJ
#define AM_BITS_FRJ 1  // the last layer's new cells from the in-block index bits (no register set in the loop)
#endif
#ifndef AM_BITS_TPRED
#define AM_BITS_TPRED 1  // stage only the time-plane words a merge needs (see the staging after the region load)
#endif
#ifndef AM_BITS_HFIRST
#define AM_BITS_HFIRST 0  // experiment: horizontal dilation per row first, then the vertical OR (one op fewer
                          // per column; measured C4 +2.4%: the extra live registers spill at 128)
#endif
#ifndef AM_BITS_HMASK_ASM
#define AM_BITS_HMASK_ASM 1
#endif
#ifndef AM_BITS_PF2
#define AM_BITS_PF2 0  // experiment: L2 prefetch of the next item's region after the layers
#endif
#ifndef AM_BITS_NOT
#define AM_BITS_NOT 0  // experiment only (wrong maps): no time-plane staging / updates
#endif

__constant__ uint8_t kBFacing[3][3] = {{8, 2, 7}, {4, 0, 3}, {6, 1, 5}};


// Lists tile (c, b) for block blk + 1 unless already listed (warp-aggregated), in two halves so the
// dedup atomic's round trip overlaps other work: bit_push_begin issues it, bit_push_end appends.
struct PushTicket {
  uint32_t old;  // previous sched value (lanes with a candidate)
  int c, b;
  bool in;
};
__device__ __forceinline__ PushTicket bit_push_begin(const BitGeo& bg, const BitBook& bk, uint32_t blk, bool want,
                                                     int c, int b) {
  PushTicket t{0xFFFFFFFFu, c, b, want && c >= 0 && b >= 0 && c < (int)bg.nchunks && b < (int)bg.tbands};
  if (t.in) t.old = atomicMax(&bk.sched[(uint32_t)c * bg.tbands + (uint32_t)b], blk + 2);
  return t;
}
__device__ __forceinline__ void bit_push_end(const BitBook& bk, uint32_t blk, const PushTicket& t) {
  const bool add = t.in && t.old < blk + 2;
  const uint32_t m = __ballot_sync(0xffffffffu, add);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(&bk.count[(blk + 1) % 3], (uint32_t)__popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (add)
    ((blk + 1) & 1 ? bk.list[1] : bk.list[0])[base + __popc(m & ((1u << lane) - 1u))] =
        (uint32_t)t.b << 16 | (uint32_t)t.c;
}
__device__ __forceinline__ void bit_push(const BitGeo& bg, const BitBook& bk, uint32_t blk, bool want, int c, int b) {
  bit_push_end(bk, blk, bit_push_begin(bg, bk, blk, want, c, b));
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// One kBK-layer block over the listed tiles.  nl (<= kBK) layers are applied
// (the last block of a fixed-L or capped run may be partial).
#ifndef AM_BITS_MINB
#define AM_BITS_MINB 4
#endif
// The items of block blk for the warp whose first item is list entry w (nwarps warps share the list,
// round-robin); leader: the one thread that resets the counters two blocks ahead and counts the items.
// wmin / covered accumulate the warp's fixed-point word and covered cells (k_bits_tiles, k_bits_run).
__device__ __forceinline__ uint32_t bits_first_item(const BitGeo& bg, const BitBook& bk, uint32_t blk, uint32_t w) {
  const uint32_t* __restrict__ list = (blk & 1) ? bk.list[1] : bk.list[0];
  return w < bg.ntiles() ? __ldcg(list + w) : 0u;
}
// n: the block's list length, it: the warp's first list entry (bits_first_item), loaded by the caller
// so they travel together with its other loads
template <bool PART>
__device__ __forceinline__ void bits_block(const BitGeo& bg, const BitBook& bk, uint32_t blk, uint32_t nl, uint32_t w,
                                           uint32_t nwarps, bool leader, uint4* tsm, uint32_t n, uint32_t it,
                                           uint32_t& wmin, uint32_t& covered) {
  const uint32_t* __restrict__ list = (blk & 1) ? bk.list[1] : bk.list[0];
  if (leader) {
    bk.count[(blk + 2) % 3] = 0;
    bk.count[3 + (blk + 2) % 3] = 0;
    atomicAdd(&bk.stat[0], (unsigned long long)n);
    if (bk.hcount) reinterpret_cast<volatile uint32_t*>(bk.hcount)[blk % kFlagSlots] = n;  // host policy (drive_bits)
  }
  const int lane = threadIdx.x & 31;
#ifndef AM_BITS_STATIC
#define AM_BITS_STATIC 1  // items dealt round-robin (measured: the fetch atomic costs more than the imbalance)
#endif
  static_assert(!AM_BITS_PREF || AM_BITS_STATIC, "prefetching needs the static item order");
  const bool light = AM_BITS_STATIC || n <= nwarps;  // one item per warp at most: no fetch atomics
  const uint32_t mark = blk + 1;
  uint32_t hmask[kBTPlanes - kBNJ];  // all-ones where bit k of blk is set: the time planes above the J bits
#pragma unroll
  for (int k = 0; k < kBTPlanes - kBNJ; ++k) hmask[k] = 0u - ((blk >> k) & 1u);
  // wmin: fixed-point word, min over new cells of (nl - 1 - in-block index); covered: cells the warp covered.
  // tsm, per warp: the time-plane words of the item's own rows (32 rows x kBTW row words x 16 words),
  // staged with cp.async at item start so the read-modify-write after the layers finds them on chip
  // An item's inputs: the states of its 3x3 tile neighbourhood (lane k < 9: (tc + k/3 - 1, tb + k%3 - 1),
  // the pre-block state whether or not that tile was processed in this block yet) and its region (rows
  // tc*TR - K .. tc*TR + TR + K, memory words tb*TW - 1 .. tb*TW + TW; each plane word is {coverage plane
  // 0, coverage plane 1, free, -}, so both coverage planes come with one 16 B load and the homes pick one
  // afterwards).  Neither changes during the block (a tile processed in it writes its other plane), so
  // with AM_BITS_PREF the next item's inputs load while the current item finishes.
  uint32_t R0[kBRPL][kBTW + 2], R1[kBRPL][kBTW + 2], RF[kBRPL][kBTW + 2], rs9 = 0;
  auto load_item = [&](uint32_t item) {
    const uint32_t ib = item >> 16, ic = item & 0xFFFFu;
    rs9 = 0;
    if (lane < 9) {
      const int c = (int)ic + lane / 3 - 1, b = (int)ib + lane % 3 - 1;
      if (c >= 0 && b >= 0 && c < (int)bg.nchunks && b < (int)bg.tbands) {
        const unsigned long long sw = __ldcg(bk.state + (uint32_t)c * bg.tbands + (uint32_t)b);
        const uint32_t cur = (uint32_t)sw;
        rs9 = (cur >> 1) == mark ? (uint32_t)(sw >> 32) : cur;
      }
    }
    const bool exl = ib > 0, exr = ib + 1 < bg.tbands;
#pragma unroll
    for (int i = 0; i < kBRPL; ++i) {
      const int tr = lane * kBRPL + i - kBK;  // tile-relative row
      const int prow = (int)ic * kBTR + tr;
      const bool er = prow >= 0 && prow < (int)bg.rows;
      const uint32_t prw = er ? (uint32_t)prow : 0u;
#pragma unroll
      for (int x = 0; x < kBTW + 2; ++x) {
        const bool e = er && (x == 0 ? exl : (x == kBTW + 1 ? exr : true));
        const uint4 v = e ? __ldcg(bk.P + bg.pidx(prw, ib * kBTW + x - 1)) : make_uint4(0u, 0u, 0u, 0u);
        R0[i][x] = v.x, R1[i][x] = v.y, RF[i][x] = v.z;
      }
    }
  };
  if (AM_BITS_PREF && w < n) load_item(it);
  while (w < n) {
    const uint32_t tb = it >> 16, tc = it & 0xFFFFu;
    uint32_t fa = 0;  // the next item's index (heavy blocks), in flight during this item
    if (!light && lane == 0)  // inline PTX: the compiler's warp aggregation would consume the result here
      asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(fa) : "l"(bk.count + 3 + blk % 3) : "memory");
    __syncwarp();  // the previous item's reads of tsm are done
    if (!AM_BITS_NOT && !AM_BITS_TPRED) {
      const uint4* tg = reinterpret_cast<const uint4*>(bk.T) + ((size_t)tc * kBTR * bg.wpr + (size_t)tb * kBTW) * 4;
#pragma unroll
      for (int q = 0; q < kBTR * kBTW * 4 / 32; ++q) {
        const int ch = lane + 32 * q, r = ch / (kBTW * 4), o = ch % (kBTW * 4);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(tsm + ch)),
                     "l"(tg + (size_t)r * bg.wpr * 4 + o)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    if (!AM_BITS_PREF) load_item(it);
    const uint32_t it_next =
        (AM_BITS_PREF || AM_BITS_PF2) && w + nwarps < n ? __ldcg(list + w + nwarps) : 0xFFFFFFFFu;
    const uint32_t s9 = rs9;
    uint32_t C[kBRPL][kBNW], C1[kBRPL][kBNW], F[kBRPL][kBNW];
    uint32_t HR0[kBRPL], HR1[kBRPL], HRF[kBRPL];  // packed halo: the right neighbour's word until the select
#pragma unroll
    for (int i = 0; i < kBRPL; ++i)
#pragma unroll
      for (int x = 0; x < kBTW + 2; ++x) {
        if (AM_BITS_PACKH && x == kBTW + 1) {
          HR0[i] = R0[i][x], HR1[i] = R1[i][x], HRF[i] = RF[i][x];
        } else {
          C[i][x] = R0[i][x], C1[i][x] = R1[i][x], F[i][x] = RF[i][x];
        }
      }
    // a state of 0 is a tile no block of this run has processed (and no source tile): its coverage words
    // are stale (a previous run's, or the walkers' layout) and read as empty
    const uint32_t hom = __ballot_sync(0xffffffffu, s9 & 1u);
    const uint32_t vld = __ballot_sync(0xffffffffu, s9 != 0u);
    const uint32_t sown = __shfl_sync(0xffffffffu, s9, 4);
#pragma unroll
    for (int i = 0; i < kBRPL; ++i) {
      const int tr = lane * kBRPL + i - kBK;
      const int d = tr < 0 ? 0 : (tr >= kBTR ? 2 : 1);
#pragma unroll
      for (int x = 0; x < kBNW; ++x) {
        const int q = x == 0 ? 0 : (x == kBTW + 1 ? 2 : 1);
        const uint32_t b = d * 3 + q;
        C[i][x] = !((vld >> b) & 1u) ? 0u : ((hom >> b) & 1u) ? C1[i][x] : C[i][x];
      }
      if (AM_BITS_PACKH) {  // halo word: left neighbour's high half | right neighbour's low half
        const uint32_t b = d * 3 + 2;
        const uint32_t cr = !((vld >> b) & 1u) ? 0u : ((hom >> b) & 1u) ? HR1[i] : HR0[i];
        C[i][0] = __byte_perm(C[i][0], cr, 0x3254);  // bytes: cr.0 cr.1 C.2 C.3
        F[i][0] = __byte_perm(F[i][0], HRF[i], 0x3254);
      }
    }
    // time-plane words of the own rows that a merge after the layers will need: only words already holding
    // covered cells (their bits must survive) and free uncovered ones (which may become new).  A word with
    // no covered cell has no time bits to keep, so new cells are written over it without a read.  Each lane
    // stages its own rows' words into its own slots, so no other lane waits on them.
    uint32_t tneed = 0;  // bit i * kBTW + x
    if (AM_BITS_TPRED && !AM_BITS_NOT) {
#pragma unroll
      for (int i = 0; i < kBRPL; ++i) {
        const int tr = lane * kBRPL + i - kBK;
        if (tr < 0 || tr >= kBTR) continue;
        const uint4* tg = reinterpret_cast<const uint4*>(bk.T) +
                          ((size_t)(tc * kBTR + (uint32_t)tr) * bg.wpr + (size_t)tb * kBTW) * 4;
#pragma unroll
        for (int x = 0; x < kBTW; ++x) {
          const uint32_t cw = C[i][x + 1];
          if (cw == 0u || (F[i][x + 1] & ~cw) == 0u) continue;
          tneed |= 1u << (i * kBTW + x);
#pragma unroll
          for (int qq = 0; qq < 4; ++qq)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(tsm + (tr * kBTW + x) * 4 + qq)),
                         "l"(tg + x * 4 + qq)
                         : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // ---- kBK layers.  J[k]: bit k of the in-block index (layer - 1) of the cells covered in this block,
    // built from snapshots (monotone coverage: the cells new in layers (a, b] are C_b & ~C_a)
    uint32_t C0[kBRPL][kBTW], J[kBNJ][kBRPL][kBTW], S[kBNJ][kBRPL][kBTW], FR[kBRPL][kBTW];
#pragma unroll
    for (int i = 0; i < kBRPL; ++i)
#pragma unroll
      for (int x = 0; x < kBTW; ++x) {
        C0[i][x] = C[i][x + 1];
#pragma unroll
        for (int k = 0; k < kBNJ; ++k) J[k][i][x] = 0u, S[k][i][x] = C[i][x + 1];
      }
#pragma unroll
    for (int j = 1; j <= kBK; ++j) {
      uint32_t N[kBRPL][kBNW];
      if ((!PART || (uint32_t)j <= nl) && AM_BITS_HFIRST) {
        // horizontal dilation of each row first, then the vertical OR: with two rows per lane the
        // rows' OR is shared by both outputs, N0 = (up | h0 | h1) & F0 and N1 = (h0 | h1 | dn) & F1
        uint32_t h[kBRPL][kBNW], up[kBNW], dn[kBNW];
#pragma unroll
        for (int i = 0; i < kBRPL; ++i)
#pragma unroll
          for (int x = 0; x < kBNW; ++x) {
            const uint32_t c = C[i][x];
            const uint32_t l = AM_BITS_PACKH || x > 0 ? __funnelshift_l(C[i][bleft(x)], c, 1) : c << 1;
            const uint32_t r = AM_BITS_PACKH || x < kBNW - 1 ? __funnelshift_r(c, C[i][bright(x)], 1) : c >> 1;
            h[i][x] = c | l | r;
          }
#pragma unroll
        for (int x = 0; x < kBNW; ++x) {
          up[x] = __shfl_up_sync(0xffffffffu, h[kBRPL - 1][x], 1);
          dn[x] = __shfl_down_sync(0xffffffffu, h[0][x], 1);
        }
#pragma unroll
        for (int x = 0; x < kBNW; ++x) {
          if (kBRPL == 2) {
            const uint32_t h01 = h[0][x] | h[kBRPL - 1][x];
            N[0][x] = (up[x] | h01) & F[0][x];
            N[kBRPL - 1][x] = (h01 | dn[x]) & F[kBRPL - 1][x];
          } else {
#pragma unroll
            for (int i = 0; i < kBRPL; ++i) {
              const uint32_t a = i == 0 ? up[x] : h[i - 1][x];
              const uint32_t b = i == kBRPL - 1 ? dn[x] : h[i + 1][x];
              N[i][x] = (a | h[i][x] | b) & F[i][x];
            }
          }
        }
      } else if (!PART || (uint32_t)j <= nl) {
        uint32_t up[kBNW], dn[kBNW];
#pragma unroll
        for (int x = 0; x < kBNW; ++x) {
          up[x] = __shfl_up_sync(0xffffffffu, C[kBRPL - 1][x], 1);
          dn[x] = __shfl_down_sync(0xffffffffu, C[0][x], 1);
        }
#pragma unroll
        for (int i = 0; i < kBRPL; ++i) {
          uint32_t v[kBNW];
#pragma unroll
          for (int x = 0; x < kBNW; ++x) {
            const uint32_t a = i == 0 ? up[x] : C[i - 1][x];
            const uint32_t b = i == kBRPL - 1 ? dn[x] : C[i + 1][x];
            v[x] = a | C[i][x] | b;
          }
#pragma unroll
          for (int x = 0; x < kBNW; ++x) {
            const uint32_t l = AM_BITS_PACKH || x > 0 ? __funnelshift_l(v[bleft(x)], v[x], 1) : v[x] << 1;
            const uint32_t r = AM_BITS_PACKH || x < kBNW - 1 ? __funnelshift_r(v[x], v[bright(x)], 1) : v[x] >> 1;
            N[i][x] = (v[x] | l | r) & F[i][x];
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < kBRPL; ++i)
#pragma unroll
          for (int x = 0; x < kBNW; ++x) N[i][x] = C[i][x];
      }
      // in-block index bits: bit k gains the cells new in layers (j - 2^k, j] when j is a multiple of 2^(k+1)
#pragma unroll
      for (int i = 0; i < kBRPL; ++i)
#pragma unroll
        for (int x = 0; x < kBTW; ++x) {
          const uint32_t nw = N[i][x + 1];
          if (!AM_BITS_FRJ && j == kBK) FR[i][x] = nw & ~C[i][x + 1];
#pragma unroll
          for (int k = 0; k < kBNJ; ++k) {
            const int p = 1 << k;
            if (j % (2 * p) == 0) J[k][i][x] |= nw & ~(k == 0 ? C[i][x + 1] : S[k][i][x]);
            if (k > 0 && j % (2 * p) == p) S[k][i][x] = nw;  // coverage at layer j = (next multiple) - 2^k
          }
        }
#pragma unroll
      for (int i = 0; i < kBRPL; ++i)
#pragma unroll
        for (int x = 0; x < kBNW; ++x) C[i][x] = N[i][x];
    }
    if (AM_BITS_PREF && w + nwarps < n) load_item(it_next);  // lands while this item finishes
    if (AM_BITS_PF2 && it_next != 0xFFFFFFFFu) {  // the next item's region lines into L2 (no registers held)
      const uint32_t nb = it_next >> 16, nc = it_next & 0xFFFFu;
#pragma unroll
      for (int i = 0; i < kBRPL; ++i) {
        const int prow = (int)nc * kBTR + lane * kBRPL + i - kBK;
        if (prow < 0 || prow >= (int)bg.rows) continue;
#pragma unroll
        for (int x = 0; x < kBTW + 2; ++x) {
          const int wd = (int)(nb * kBTW) + x - 1;
          if (wd < 0 || wd >= (int)bg.wpr) continue;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(bk.P + bg.pidx((uint32_t)prow, (uint32_t)wd)));
        }
      }
    }
    // cells new in the last layer: in-block index kBK - 1, all J bits set (none in a partial block)
    if (AM_BITS_FRJ) {
#pragma unroll
      for (int i = 0; i < kBRPL; ++i)
#pragma unroll
        for (int x = 0; x < kBTW; ++x) {
          uint32_t f = C[i][x + 1] & ~C0[i][x];
#pragma unroll
          for (int k = 0; k < kBNJ; ++k) f &= J[k][i][x];
          FR[i][x] = f;
        }
    }
    // ---- own rows: coverage into the other plane; the new cells' layer t into the time planes
    // (T: 16 words per row word, word k = bit k of t-1 for the row word's 32 cells; t - 1 = l0 + in-block
    // index, l0 = kBK * blk, so bits < kBNJ are J and the others the bits of blk; only the new cells' bits
    // change, so T needs no initialisation)
    const uint32_t out_home = (sown & 1u) ^ 1u;
    uint32_t any_new = 0, m9 = 0, fr_all = 0;
    uint32_t NW[kBRPL][kBTW];
#pragma unroll
    for (int i = 0; i < kBRPL; ++i) {
      const int tr = lane * kBRPL + i - kBK;
      const bool own = tr >= 0 && tr < kBTR;
#pragma unroll
      for (int x = 0; x < kBTW; ++x) NW[i][x] = own ? C[i][x + 1] & ~C0[i][x] : 0u;
      if (!own) continue;
      const uint32_t orow = tc * kBTR + (uint32_t)tr;
#pragma unroll
      for (int x = 0; x < kBTW; ++x)
        __stcg(reinterpret_cast<uint32_t*>(bk.P + bg.pidx(orow, tb * kBTW + x)) + out_home, C[i][x + 1]);
      uint32_t fr_any = 0;
#pragma unroll
      for (int x = 0; x < kBTW; ++x) {
        covered += __popc(NW[i][x]);
        any_new |= NW[i][x];
        fr_any |= FR[i][x];
      }
      fr_all |= fr_any;
      // frontier regions (bits: any, top, bottom, left, right, tl, tr, bl, br)
      constexpr uint32_t lowK = kBK >= 32 ? 0xFFFFFFFFu : (1u << kBK) - 1u;
      constexpr uint32_t highK = kBK >= 32 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> kBK);
      const bool left = (FR[i][0] & lowK) != 0, right = (FR[i][kBTW - 1] & highK) != 0;
      const bool top = tr < kBK, bot = tr >= kBTR - kBK;
      if (fr_any) {
        m9 |= 1u | (top ? 2u : 0u) | (bot ? 4u : 0u);
        m9 |= (left ? 8u : 0u) | (right ? 16u : 0u);
        m9 |= (top && left ? 32u : 0u) | (top && right ? 64u : 0u) | (bot && left ? 128u : 0u) |
              (bot && right ? 256u : 0u);
      }
    }
    m9 = __reduce_or_sync(0xffffffffu, m9);
    // list the next block's candidates (lane k < 9: the neighbour at (k/3 - 1, k%3 - 1) facing a frontier
    // region); the dedup atomics travel while the time planes are updated
    PushTicket pt;
    {
      const int dr = lane / 3 - 1, dc = lane % 3 - 1;
      const bool want = lane < 9 && ((m9 >> kBFacing[(lane / 3) % 3][lane % 3]) & 1u);
      pt = bit_push_begin(bg, bk, blk, want, (int)tc - dr, (int)tb - dc);
    }
    uint32_t next = AM_BITS_STATIC ? w + nwarps : nwarps;
    if (AM_BITS_PREF) it = it_next;
    else if (AM_BITS_STATIC && next < n) it = __ldcg(list + next);
    if (!light) {  // dynamic items past the static first one: the list entry loads during the update
      next = __shfl_sync(0xffffffffu, fa, 0) + nwarps;
      if (next < n) it = __ldcg(list + next);
    }
    // ---- time planes (T: 16 words per row word, word k = bit k of t-1 for the row word's 32 cells;
    // t - 1 = l0 + in-block index, l0 = kBK * blk, so bits < kBNJ are J and the others the bits of blk;
    // only the new cells' bits change, so T needs no initialisation)
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kBRPL; ++i) {
      const int tr = lane * kBRPL + i - kBK;
      if (AM_BITS_NOT || tr < 0 || tr >= kBTR) continue;
      const size_t rw = (size_t)(tc * kBTR + (uint32_t)tr) * bg.wpr + (size_t)tb * kBTW;
#pragma unroll
      for (int x = 0; x < kBTW; ++x) {
        const uint32_t nw = NW[i][x];
        if (!nw) continue;
        const uint4* ts = tsm + (tr * kBTW + x) * 4;
        uint32_t v[16];
        if (!AM_BITS_TPRED || ((tneed >> (i * kBTW + x)) & 1u)) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 a4 = ts[q];
            v[4 * q] = a4.x, v[4 * q + 1] = a4.y, v[4 * q + 2] = a4.z, v[4 * q + 3] = a4.w;
          }
        } else {  // no covered cell in the word before this block: nothing to keep
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] = 0u;
        }
#pragma unroll
        for (int k = 0; k < kBTPlanes; ++k) {
          // planes >= kBNJ: bit k - kBNJ of blk for every new cell: one LOP3 (v & ~nw) | (nw & mask) with
          // the block's masks made once per block (the compiler otherwise re-tests each bit per word)
          if (k < kBNJ) {
            v[k] = (v[k] & ~nw) | J[k < kBNJ ? k : 0][i][x];
          } else {
#if AM_BITS_HMASK_ASM
            asm("lop3.b32 %0, %1, %2, %3, 0xB8;" : "=r"(v[k]) : "r"(v[k]), "r"(nw), "r"(hmask[k < kBNJ ? 0 : k - kBNJ]));
#else
            v[k] = (v[k] & ~nw) | (nw & hmask[k < kBNJ ? 0 : k - kBNJ]);
#endif
          }
        }
        uint4* tp = reinterpret_cast<uint4*>(bk.T + (rw + x) * 16);
#pragma unroll
        for (int q = 0; q < 4; ++q) __stcg(tp + q, make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
      }
    }
#if AM_BITS_STATS
    {  // experiment counters: items without new cells, items whose own rows have no free uncovered cell
      uint32_t fu = 0;
#pragma unroll
      for (int i = 0; i < kBRPL; ++i) {
        const int tr = lane * kBRPL + i - kBK;
        if (tr < 0 || tr >= kBTR) continue;
#pragma unroll
        for (int x = 0; x < kBTW; ++x) fu |= F[i][x + 1] & ~C[i][x + 1];
      }
      const bool none_new = !__any_sync(0xffffffffu, any_new != 0);
      const bool full = !__any_sync(0xffffffffu, fu != 0);
      if (lane == 0) {
        if (none_new) atomicAdd(&bk.stat[3], 1ull);
        if (full) atomicAdd(&bk.stat[4], 1ull);
        if (none_new && !full) atomicAdd(&bk.stat[5], 1ull);
      }
    }
#endif
    if (__any_sync(0xffffffffu, any_new != 0)) {
      // in-block index of the warp's last new cell: kBK - 1 if a cell is new in the last layer, else the
      // bit-sliced maximum over the new cells' J
      uint32_t jm = kBK - 1;
      if (!__any_sync(0xffffffffu, fr_all != 0)) {
        jm = 0;
#pragma unroll
        for (int k = kBNJ - 1; k >= 0; --k) {
          uint32_t a = 0;
#pragma unroll
          for (int i = 0; i < kBRPL; ++i)
#pragma unroll
            for (int x = 0; x < kBTW; ++x) a |= NW[i][x] & J[k][i][x];
          const bool set = __any_sync(0xffffffffu, a != 0);
          if (set) jm |= 1u << k;
#pragma unroll
          for (int i = 0; i < kBRPL; ++i)
#pragma unroll
            for (int x = 0; x < kBTW; ++x) NW[i][x] &= set ? J[k][i][x] : ~J[k][i][x];
        }
      }
      const uint32_t v = nl - 1 - jm;
      wmin = v < wmin ? v : wmin;
    }
    if (lane == 0)
      bk.state[tc * bg.tbands + tb] = (unsigned long long)sown << 32 | (mark << 1 | out_home);
    if (AM_BITS_DONE) {
      // every free cell of the tile is covered: its planes are final, so no later block needs it.  A
      // schedule word of ~0 makes every later push of the tile a no-op (the dedup atomicMax sees it as
      // listed); a push racing with this store lists it once more, which is harmless.  (Also counting
      // tiles whose uncovered free cells are closed pockets -- none in the last layer's frontier, none on
      // the border ring -- skipped 2.3% of the C4 items but cost as much per item as it saved.)
      uint32_t fu = 0;
#pragma unroll
      for (int i = 0; i < kBRPL; ++i) {
        const int tr = lane * kBRPL + i - kBK;
        if (tr < 0 || tr >= kBTR) continue;
#pragma unroll
        for (int x = 0; x < kBTW; ++x) fu |= F[i][x + 1] & ~C[i][x + 1];
      }
      if (!__any_sync(0xffffffffu, fu != 0u) && lane == 0) bk.sched[tc * bg.tbands + tb] = 0xFFFFFFFFu;
    }
    bit_push_end(bk, blk, pt);
    w = next;
  }
}

template <bool PART>
__global__ void __launch_bounds__(kBThreads, AM_BITS_MINB) k_bits_tiles(BitGeo bg, BitBook bk, uint32_t blk, uint32_t nl,
                                                          FlagSink flag, FlagSink prev) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  if (prev.host && blockIdx.x == 0 && threadIdx.x == 0)
    *reinterpret_cast<volatile uint32_t*>(prev.host) = atomicExch(prev.word, 0xFFFFFFFFu);
  extern __shared__ uint4 tsm_all[];  // kBTsmBytes: kBThreads / 32 warps x kBTR * kBTW * 4 slots
  uint32_t wmin = 0xFFFFFFFFu, covered = 0;
  // static first item (spread over the SMs): its list entry is loaded alongside the list length
  // item k of the block goes to warp k / gridDim of CTA k % gridDim: the first items spread over every CTA
  // (CTA-major orders measured C4 +7%)
  const uint32_t w = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  const uint32_t n = __ldcg(bk.count + blk % 3);
  bits_block<PART>(bg, bk, blk, nl, w, gridDim.x * (kBThreads / 32), blockIdx.x == 0 && threadIdx.x == 0,
                   tsm_all + (threadIdx.x >> 5) * (kBTR * kBTW * 4), n, bits_first_item(bg, bk, blk, w), wmin,
                   covered);
  covered = __reduce_add_sync(0xffffffffu, covered);
  if ((threadIdx.x & 31) == 0) {
    if (covered) atomicAdd(&bk.stat[1], (unsigned long long)covered);
    if (wmin != 0xFFFFFFFFu) atomicMin(flag.word, wmin);
  }
}

// Light stretches in one thread-block cluster: while a block lists at most nmax tiles, the
// cluster's warps run block after block with a hardware cluster barrier between them instead of a kernel
// boundary (the boundary is ~2.9 us; a light block's own chain ~4 us).  Same items, same bookkeeping as
// k_bits_tiles; the fixed-point word of block b is count[6 + b % 3] (reset one block ahead by the leader)
// and the auto-run termination of drive_bits is evaluated here after each block.  Stops before block
// blk_end, when a block lists more than nmax tiles, or at the fixed point (autom); the outcome goes to
// the mapped record rec: {seq, next block, termination layer or 0, next block's items, blocks run}.
__global__ void __launch_bounds__(kBRunThreads, 1) k_bits_run(BitGeo bg, BitBook bk, uint32_t blk, uint32_t blk_end,
                                                               uint32_t nmax, uint32_t autom, uint32_t seq,
                                                               uint32_t* rec) {
  extern __shared__ uint4 tsm_all[];
  uint4* tsm = tsm_all + (threadIdx.x >> 5) * (kBTR * kBTW * 4);
  uint32_t crank, csize;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  const uint32_t nwarps = csize * (kBRunThreads / 32), w0 = (threadIdx.x >> 5) * csize + crank;
  const bool leader = crank == 0 && threadIdx.x == 0;
  uint32_t lprime = 0, n_next = 0, blocks = 0;
  uint32_t n = __ldcg(bk.count + blk % 3), it = bits_first_item(bg, bk, blk, w0);
  for (;;) {
    if (blk >= blk_end || n > nmax) {
      n_next = n;
      break;
    }
    if (leader) bk.count[6 + (blk + 1) % 3] = 0xFFFFFFFFu;
    uint32_t wmin = 0xFFFFFFFFu, covered = 0;
    bits_block<false>(bg, bk, blk, kBK, w0, nwarps, leader, tsm, n, it, wmin, covered);
    covered = __reduce_add_sync(0xffffffffu, covered);
    if ((threadIdx.x & 31) == 0) {
      if (covered) atomicAdd(&bk.stat[1], (unsigned long long)covered);
      if (wmin != 0xFFFFFFFFu) atomicMin(bk.count + 6 + blk % 3, wmin);
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    // the fixed-point word, the next block's list length and first entries: one round trip
    const uint32_t m = __ldcg(bk.count + 6 + blk % 3);
    n = __ldcg(bk.count + (blk + 1) % 3);
    it = bits_first_item(bg, bk, blk + 1, w0);
    const uint32_t start = kBK * blk;
    ++blk, ++blocks;
    if (autom) {  // drive_bits' block_termination for a full 16-bit block
      const uint32_t t = m >= 0x7FFFu ? start + 1 : m >= 1 ? start + kBK + 1 - m : 0u;
      if (t) {
        lprime = t;
        break;
      }
    }
  }
  if (leader) {
    volatile uint32_t* r = rec;
    r[1] = blk, r[2] = lprime, r[3] = n_next, r[4] = blocks;
    __threadfence_system();
    r[0] = seq;
  }
}

// Plane words {0, 0, free, 0} from the dense occupancy (occ != 0: obstacle).  A warp builds 32 words of
// one plane row: 32 ballots over coalesced byte loads.
__global__ void k_bits_init(BitGeo bg, const uint8_t* __restrict__ occ, uint4* __restrict__ P,
                            unsigned long long* __restrict__ free_cells) {
  const int lane = threadIdx.x & 31;
  const uint32_t row = blockIdx.y * (blockDim.x / 32) + (threadIdx.x >> 5);
  const uint32_t w0 = blockIdx.x * 32;
  if (row >= bg.rows) return;  // warp-uniform
  uint32_t mine = 0;
  const bool in_row = row < bg.H;
  const uint8_t* orow = occ + (size_t)row * bg.W;
  uint8_t o[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) {  // all 32 loads in flight
    const uint32_t col = (w0 + k) * 32 + lane;
    o[k] = in_row && col < bg.W ? orow[col] : (uint8_t)1;
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const uint32_t bits = __ballot_sync(0xffffffffu, o[k] == 0);
    if (lane == k) mine = bits;
  }
  if (w0 + lane < bg.wpr) P[bg.pidx(row, w0 + lane)] = make_uint4(0u, 0u, mine, 0u);  // not covered
  const uint32_t cnt = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(mine));
  if (lane == 0 && cnt) atomicAdd(free_cells, (unsigned long long)cnt);
}

// Plane words {0, 0, free, 0} from packed occupancy rows (bit = obstacle, pw = (W + 31) / 32 words per row).
// A CTA converts 32 rows x 32 words: read along the packed rows, written along P's layout (a shared-memory
// transpose when P is column-major).
__global__ void k_bits_init_packed(BitGeo bg, const uint32_t* __restrict__ packed, uint4* __restrict__ P,
                                   unsigned long long* __restrict__ free_cells) {
  __shared__ uint32_t t[32][33];
  const uint32_t pw = (bg.W + 31) / 32;
  const uint32_t w0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 256 threads: 8 warps
  uint32_t cnt = 0;
  for (uint32_t k = ty; k < 32; k += 8) {  // warp ty: rows r0 + k, lane: word w0 + tx
    const uint32_t row = r0 + k, w = w0 + tx;
    uint32_t f = 0;
    if (row < bg.H && w < pw) {
      const uint32_t valid = bg.W - 32 * w >= 32 ? 0xFFFFFFFFu : (1u << (bg.W - 32 * w)) - 1u;
      f = ~__ldg(packed + (size_t)row * pw + w) & valid;
    }
    t[k][tx] = f;
    cnt += __popc(f);
  }
  __syncthreads();
  for (uint32_t k = ty; k < 32; k += 8) {
    // AM_BITS_PCM: warp ty writes word w0 + k for rows r0 + tx (contiguous); else row r0 + k, words w0 + tx
    const uint32_t row = AM_BITS_PCM ? r0 + tx : r0 + k, w = AM_BITS_PCM ? w0 + k : w0 + tx;
    if (row < bg.rows && w < bg.wpr) P[bg.pidx(row, w)] = make_uint4(0u, 0u, AM_BITS_PCM ? t[tx][k] : t[k][tx], 0u);
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if (tx == 0 && cnt) atomicAdd(free_cells, (unsigned long long)cnt);
}

// The tiles holding a source start the run with valid coverage in home plane 0: their plane-0 words are
// cleared here (before k_bits_sources sets the source bits) and their state set to kBitsSrcState.  One
// warp per source; lane k clears rows k, k + 32, ... of the tile's kBTW words.
constexpr uint32_t kBitsSrcState = 0xFFFFFFFEu;  // home 0, mark 0x7FFFFFFF (no block's mark), nonzero
__global__ void k_bits_src_clear(BitGeo bg, const uint32_t* __restrict__ rc, uint64_t n, BitBook bk) {
  const uint64_t s = blockIdx.x * (uint64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  if (s >= n) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const uint32_t tc = rc[2 * s] / kBTR, tb = rc[2 * s + 1] / (32 * kBTW);
  for (int i = lane; i < kBTR * kBTW; i += 32) {
    const uint32_t row = tc * kBTR + (uint32_t)i / kBTW, wd = tb * kBTW + (uint32_t)i % kBTW;
    if (row < bg.rows) bk.P[bg.pidx(row, wd)].x = 0u;
  }
  if (lane == 0) bk.state[tc * bg.tbands + tb] = kBitsSrcState;
}

// Sources (validated free cells): covered at layer 0, time-plane value kBTSrcU (no covered cell has
// t - 1 = kBTSrcU: t <= lref <= kBitsMaxRef), and block 0's work list (the 3x3 tile neighbourhood of each
// source's tile, pushed as block "-1").  One warp per source.
__global__ void k_bits_sources(BitGeo bg, const uint32_t* __restrict__ rc, uint64_t n, BitBook bk) {
  const uint64_t s = blockIdx.x * (uint64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  if (s >= n) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const uint32_t r = rc[2 * s], c = rc[2 * s + 1];
  const size_t rw = bg.tidx(r, c >> 5);
  const uint32_t bit = 1u << (c & 31);
  if (lane == 0) {
    const uint32_t old = atomicOr(&bk.P[bg.pidx(r, c >> 5)].x, bit);
    if (!(old & bit)) atomicAdd(&bk.stat[1], 1ull);
  }
  if (lane < kBTPlanes) atomicOr(bk.T + rw * 16 + lane, bit);
  const int tc = (int)(r / kBTR), tb = (int)(c / (32 * kBTW));
  bit_push(bg, bk, 0xFFFFFFFFu, lane < 9, tc + lane / 3 - 1, tb + lane % 3 - 1);
}

// The encoded field (am_internal.cuh) from the planes, once per run: free covered cell flag | (lref - u)
// with u = t - 1 from the time planes (lref + 1 at sources: u = kBTSrcU == -1 mod 2^kBTPlanes), free
// uncovered flag | 0, obstacle 0.  It only reads the planes, so it runs on the context's map stream beside
// the path walkers (which read the planes too, never the field).  A warp converts two row words per
// step: lane k of half h (lanes 16h .. 16h+15) holds plane word k of row word wb + 2q + h -- time planes
// 0 .. kBTPlanes-1, then the covered word (the tile's home plane, or 0 in a tile no block processed) and
// the free word -- and a 32 x 32 bit transpose over the lanes (five butterfly shuffles) leaves lane c
// with cell c of both row words as a u16x2 {free, covered, u} pair: the encoding is then a handful of
// word-wide ops, and two coalesced 64 B stores follow.
#ifndef AM_FIN_STEPS
#define AM_FIN_STEPS 2
#endif
constexpr uint32_t kFinalizeSteps = AM_FIN_STEPS;  // warp steps per warp (short-lived CTAs, see the launch)
#ifndef AM_FIN_P
#define AM_FIN_P 8
#endif
constexpr int kFinP = AM_FIN_P;          // row-word pairs per warp step (their loads in flight together)
__global__ void __launch_bounds__(256) k_bits_finalize(BitGeo bg, Geo g, BitBook bk, uint32_t lref,
                                                       uint16_t* __restrict__ field) {
  constexpr int P = kFinP;
  constexpr uint32_t kUMask = (1u << kBTPlanes) - 1u, kU2 = kUMask | kUMask << 16;
  static_assert(kBTPlanes == 14, "planes 14 / 15 of a row word carry covered / free");
  const int lane = threadIdx.x & 31;
  const int k = lane & 15;
  const uint32_t row = blockIdx.y;  // one grid row per plane row: no index division
  const size_t rb = (size_t)row * bg.wpr;
  const uint32_t st_row = (row / kBTR) * bg.tbands;
  // per half: (lref + 2^kBTPlanes) - u >= 0, no borrow across the halves; the low kBTPlanes bits are
  // (lref - u) mod 2^kBTPlanes, which is lref + 1 at sources
  const uint32_t K2 = (lref + (1u << kBTPlanes)) * 0x00010001u;
  uint16_t* const frow = field + (size_t)(row + g.pad) * g.pitch + g.pad + lane;
  uint32_t kp[5];  // the transpose's keep masks, materialised once per thread
#pragma unroll
  for (int jj = 0; jj < 5; ++jj) {
    const int j = 16 >> jj;
    const uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu : j == 2 ? 0x33333333u
                                                                                                  : 0x55555555u;
    kp[jj] = (lane & j) ? ~m : m;
  }
  const uint32_t wb0 = (blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * kFinalizeSteps * 2 * P;
#pragma unroll 1
  for (uint32_t s = 0; s < kFinalizeSteps; ++s) {
    const uint32_t wb = wb0 + s * 2 * P;  // first row word of the step (warp-uniform)
    if (wb >= bg.wpr) break;
    // lanes 0 .. 2P-1: the covered (the tile's home plane; nothing in a tile no block processed) and free
    // words of the step's row words
    uint32_t fv = 0, cv = 0;
    const uint32_t wl = wb + lane;
    if (lane < 2 * P && wl < bg.wpr) {
      const uint4 pv = __ldcg(bk.P + bg.pidx(row, wl));
      const uint32_t st = (uint32_t)__ldcg(bk.state + st_row + wl / kBTW);
      fv = pv.z;
      cv = st == 0u ? 0u : (st & 1u) ? pv.y : pv.x;
    }
    uint32_t x[P];  // lanes 16 .. 31 read the next row word's planes (wpr is even); every lane loads (an
                    // unconditional load: no branch around it for the lanes that take covered / free)
    const uint32_t* tb = bk.T + (rb + wb) * 16 + lane;
#pragma unroll
    for (int q = 0; q < P; ++q) {
      x[q] = 0u;
      if (wb + 2 * q < bg.wpr)  // warp-uniform
        asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(x[q]) : "l"(tb + 32 * q));
    }
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const int from = 2 * q + (lane >> 4);
      const uint32_t c = __shfl_sync(0xffffffffu, cv, from), f = __shfl_sync(0xffffffffu, fv, from);
      x[q] = k == kBTPlanes ? c : k == kBTPlanes + 1 ? f : x[q];
    }
#pragma unroll
    for (int jj = 0; jj < 5; ++jj) {
      const int j = 16 >> jj;
      // lanes with bit j set keep the bits of columns with bit j set and take the partner's, moved down by
      // j; the others keep / take the complementary columns, moved up: the rotated partner word supplies
      // exactly the ~keep columns, so one bit-select (LOP3 0xE4) merges them
      const uint32_t keep = kp[jj];
      const uint32_t rot = (lane & j) ? j : 32 - j;
#pragma unroll
      for (int q = 0; q < P; ++q) {
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x[q], j);
        const uint32_t r = __funnelshift_r(y, y, rot);
        uint32_t o;
        asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(o) : "r"(x[q]), "r"(r), "r"(keep));  // (x & keep) | (r & ~keep)
        x[q] = o;
      }
    }
    uint16_t* dst = frow + (size_t)wb * 32;
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const uint32_t v0 = x[q];                                      // per half: free | covered | u
      const uint32_t a = K2 - (v0 & kU2);                            // per half: low bits (lref - u) mod 2^14
      const uint32_t cm = ((v0 >> kBTPlanes) & 0x00010001u) * kUMask;  // per half: kUMask if covered
      const uint32_t v = (a & cm) | (v0 & 0x80008000u);              // covered implies free
      const uint32_t c0 = (wb + 2 * q) * 32;                         // warp-uniform
      if (c0 + 64 <= bg.W) {  // both row words inside the grid
        dst[64 * q] = (uint16_t)v;
        dst[64 * q + 32] = (uint16_t)(v >> 16);
      } else {
        if (c0 + lane < bg.W) dst[64 * q] = (uint16_t)v;
        if (c0 + 32 + lane < bg.W) dst[64 * q + 32] = (uint16_t)(v >> 16);
      }
    }
  }
}

}  // namespace

static void bits_smem_attr() {
  static const bool done = [] {
    cudaFuncSetAttribute(k_bits_tiles<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBTsmBytes);
    cudaFuncSetAttribute(k_bits_tiles<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBTsmBytes);
    return true;
  }();
  (void)done;
}

int bits_ctas_per_sm() {
  int n = 0;
  bits_smem_attr();
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_bits_tiles<false>, kBThreads, kBTsmBytes) != cudaSuccess)
    n = 1;
  return n < 1 ? 1 : n;
}

void launch_bits_init(const BitGeo& bg, const uint8_t* occ, BitBook bk, cudaStream_t s) {
  const dim3 grid((bg.wpr + 31) / 32, (bg.rows + 7) / 8);
  k_bits_init<<<grid, 256, 0, s>>>(bg, occ, bk.P, bk.stat + 2);
}

void launch_bits_init_packed(const BitGeo& bg, const uint32_t* packed, BitBook bk, cudaStream_t s) {
  const dim3 grid((bg.wpr + 31) / 32, (bg.rows + 31) / 32);
  k_bits_init_packed<<<grid, 256, 0, s>>>(bg, packed, bk.P, bk.stat + 2);
}

void launch_bits_sources(const BitGeo& bg, const uint32_t* rc, uint64_t n, BitBook bk, cudaStream_t s) {
  if (!n) return;
  k_bits_src_clear<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(bg, rc, n, bk);
  k_bits_sources<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(bg, rc, n, bk);
}

void launch_bits_finalize(const BitGeo& bg, const Geo& g, BitBook bk, uint32_t lref, uint16_t* field, int sms,
                          cudaStream_t s) {
  (void)sms;
  const uint32_t words_per_cta = 8 * kFinalizeSteps * 2 * kFinP;  // 8 warps
  const dim3 grid((bg.wpr + words_per_cta - 1) / words_per_cta, bg.H);
  k_bits_finalize<<<grid, 256, 0, s>>>(bg, g, bk, lref, field);
}

void launch_bits_tiles(const BitGeo& bg, int ctas, BitBook bk, uint32_t blk, uint32_t nl, FlagSink flag,
                       FlagSink prev, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(kBThreads);
  cfg.dynamicSmemBytes = kBTsmBytes;
  cfg.stream = s;
  bits_smem_attr();
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // a partial block (the last of a fixed-L or capped run) skips its layers past nl
  if (nl == (uint32_t)kBK)
    cudaLaunchKernelEx(&cfg, k_bits_tiles<false>, bg, bk, blk, nl, flag, prev);
  else
    cudaLaunchKernelEx(&cfg, k_bits_tiles<true>, bg, bk, blk, nl, flag, prev);
}

int bits_run_cluster() {
  static const int size = [] {
    cudaFuncSetAttribute(k_bits_run, cudaFuncAttributeMaxDynamicSharedMemorySize, kBRunSmem);
    cudaFuncSetAttribute(k_bits_run, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c : {16, 8, 4}) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(c);
      cfg.blockDim = dim3(kBRunThreads);
      cfg.dynamicSmemBytes = kBRunSmem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, k_bits_run, &cfg) == cudaSuccess && n >= 1) return c;
      (void)cudaGetLastError();
    }
    return 0;
  }();
  return size;
}

uint32_t bits_run_warps(int cluster) { return (uint32_t)cluster * (kBRunThreads / 32); }

void launch_bits_run(const BitGeo& bg, int cluster, BitBook bk, uint32_t blk, uint32_t blk_end, uint32_t nmax,
                     bool autom, uint32_t seq, uint32_t* rec, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cluster);
  cfg.blockDim = dim3(kBRunThreads);
  cfg.dynamicSmemBytes = kBRunSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_bits_run, bg, bk, blk, blk_end, nmax, (uint32_t)autom, seq, rec);
}

}  // namespace am
