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

constexpr int kBNW = kBTW + 2;   // words per region row (one halo word each side)
constexpr int kBNJ = kBK == 8 ? 3 : kBK == 16 ? 4 : 5;  // bit planes of the in-block layer index
static_assert(kBK == 8 || kBK == 16 || kBK == 32, "layers per bit block");
static_assert(kBTR >= kBK && kBTR > 0, "tiles at least kBK rows");
static_assert(kBK % kBRPL == 0 || kBRPL == 1, "halo rows fill whole lanes");
constexpr int kBThreads = 128;

__constant__ uint8_t kBFacing[3][3] = {{8, 2, 7}, {4, 0, 3}, {6, 1, 5}};

__device__ __forceinline__ uint32_t ldcg(const uint32_t* p) { return __ldcg(p); }

// Lists tile (c, b) for block blk + 1 unless already listed (warp-aggregated).
__device__ __forceinline__ void bit_push(const BitGeo& bg, const BitBook& bk, uint32_t blk, bool want, int c, int b) {
  const bool in = want && c >= 0 && b >= 0 && c < (int)bg.nchunks && b < (int)bg.tbands;
  bool add = false;
  if (in) add = atomicMax(&bk.sched[(uint32_t)c * bg.tbands + (uint32_t)b], blk + 2) < blk + 2;
  const uint32_t m = __ballot_sync(0xffffffffu, add);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(&bk.count[(blk + 1) % 3], (uint32_t)__popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (add) ((blk + 1) & 1 ? bk.list[1] : bk.list[0])[base + __popc(m & ((1u << lane) - 1u))] = (uint32_t)b << 16 | (uint32_t)c;
}

// One kBK-layer block over the listed tiles.  nl (<= kBK) layers are applied
// (the last block of a fixed-L or capped run may be partial).
__global__ void __launch_bounds__(kBThreads) k_bits_tiles(BitGeo bg, Geo g, uint16_t* __restrict__ field, BitBook bk,
                                                          uint32_t blk, uint32_t l0, uint32_t nl, uint32_t lref,
                                                          FlagSink flag, FlagSink prev) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  if (prev.host && blockIdx.x == 0 && threadIdx.x == 0)
    *reinterpret_cast<volatile uint32_t*>(prev.host) = atomicExch(prev.word, 0xFFFFFFFFu);
  const uint32_t n = bk.count[blk % 3];
  const uint32_t* __restrict__ list = (blk & 1) ? bk.list[1] : bk.list[0];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    bk.count[(blk + 2) % 3] = 0;
    bk.count[3 + (blk + 2) % 3] = 0;
    atomicAdd(&bk.stat[0], (unsigned long long)n);
  }
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (kBThreads / 32);
  const uint32_t mark = blk + 1;
  const size_t plane = bg.plane_words();
  uint32_t wmin = 0xFFFFFFFFu;    // fixed-point word: min over new cells of (nl - 1 - in-block index)
  uint32_t covered = 0;           // cells this warp covered
  // static first item (spread over the SMs), then dynamic
  uint32_t w = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  while (w < n) {
    const uint32_t it = list[w];
    const uint32_t tb = it >> 16, tc = it & 0xFFFFu;
    // states of the 3x3 tile neighbourhood: lane k < 9 reads (tc + k/3 - 1, tb + k%3 - 1)
    uint32_t s9 = 0;
    bool ex = false;
    if (lane < 9) {
      const int c = (int)tc + lane / 3 - 1, b = (int)tb + lane % 3 - 1;
      ex = c >= 0 && b >= 0 && c < (int)bg.nchunks && b < (int)bg.tbands;
      if (ex) {
        const unsigned long long sw = __ldcg(bk.state + (uint32_t)c * bg.tbands + (uint32_t)b);
        const uint32_t cur = (uint32_t)sw;
        s9 = (cur >> 1) == mark ? (uint32_t)(sw >> 32) : cur;
      }
    }
    const uint32_t exm = __ballot_sync(0xffffffffu, ex);
    const uint32_t hom = __ballot_sync(0xffffffffu, ex && (s9 & 1u));
    const uint32_t sown = __shfl_sync(0xffffffffu, s9, 4);
    // ---- load the region: rows tc*TR - K .. tc*TR + TR + K, words tb*TW - 1 .. tb*TW + TW
    uint32_t C[kBRPL][kBNW], F[kBRPL][kBNW];
#pragma unroll
    for (int i = 0; i < kBRPL; ++i) {
      const int tr = lane * kBRPL + i - kBK;  // tile-relative row
      const int d = tr < 0 ? 0 : (tr >= kBTR ? 2 : 1);
      const int prow = (int)tc * kBTR + tr;
      const size_t rb = (size_t)(prow < 0 ? 0 : prow) * bg.wpr + (size_t)tb * kBTW;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int k = d * 3 + q;
        const bool e = (exm >> k) & 1u;
        const uint32_t* cp = bk.C + (((hom >> k) & 1u) ? plane : 0);
        if (q == 1) {
          if (e) {
            const uint4 cv = __ldcg(reinterpret_cast<const uint4*>(cp + rb));
            const uint4 fv = __ldg(reinterpret_cast<const uint4*>(bk.F + rb));
            C[i][1] = cv.x, C[i][2] = cv.y, C[i][3] = cv.z, C[i][4] = cv.w;
            F[i][1] = fv.x, F[i][2] = fv.y, F[i][3] = fv.z, F[i][4] = fv.w;
          } else {
#pragma unroll
            for (int x = 1; x <= kBTW; ++x) C[i][x] = F[i][x] = 0u;
          }
        } else {
          const size_t a = q == 0 ? rb - 1 : rb + kBTW;
          C[i][q == 0 ? 0 : kBNW - 1] = e ? ldcg(cp + a) : 0u;
          F[i][q == 0 ? 0 : kBNW - 1] = e ? __ldg(bk.F + a) : 0u;
        }
      }
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
      if ((uint32_t)j <= nl) {
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
            const uint32_t l = x > 0 ? __funnelshift_l(v[x - 1], v[x], 1) : v[x] << 1;
            const uint32_t r = x < kBNW - 1 ? __funnelshift_r(v[x], v[x + 1], 1) : v[x] >> 1;
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
          if (j == kBK) FR[i][x] = nw & ~C[i][x + 1];
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
    // ---- own rows: new cells into the field, coverage into the other plane
    const uint32_t out_home = (sown & 1u) ^ 1u;
    uint32_t jmax = 0, any_new = 0, m9 = 0;
#pragma unroll
    for (int i = 0; i < kBRPL; ++i) {
      const int tr = lane * kBRPL + i - kBK;
      if (tr < 0 || tr >= kBTR) continue;
      const uint32_t row = tc * kBTR + (uint32_t)tr;
      uint32_t* dst = bk.C + (out_home ? plane : 0) + (size_t)row * bg.wpr + (size_t)tb * kBTW;
      __stcg(reinterpret_cast<uint4*>(dst), make_uint4(C[i][1], C[i][2], C[i][3], C[i][4]));
      uint16_t* frow = field + (size_t)(row + g.pad) * g.pitch + g.pad + (size_t)tb * (32 * kBTW);
      uint32_t fr_any = 0;
#pragma unroll
      for (int x = 0; x < kBTW; ++x) {
        uint32_t m = C[i][x + 1] & ~C0[i][x];
        covered += __popc(m);
        any_new |= m;
        fr_any |= FR[i][x];
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          uint32_t jj = 0;
#pragma unroll
          for (int k = 0; k < kBNJ; ++k) jj |= ((J[k][i][x] >> b) & 1u) << k;
          jmax = jj > jmax ? jj : jmax;
          frow[x * 32 + b] = (uint16_t)(kFlag16 | (lref - l0 - jj));
        }
      }
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
    const bool anyw = __any_sync(0xffffffffu, any_new != 0);
    if (anyw) {
      const uint32_t jm = __reduce_max_sync(0xffffffffu, any_new ? jmax : 0u);
      const uint32_t v = nl - 1 - jm;
      wmin = v < wmin ? v : wmin;
    }
    uint32_t next = 0;
    if (lane == 0) next = atomicAdd(&bk.count[3 + blk % 3], 1u) + nwarps;
    next = __shfl_sync(0xffffffffu, next, 0);
    if (lane == 0)
      bk.state[tc * bg.tbands + tb] = (unsigned long long)sown << 32 | (mark << 1 | out_home);
    {
      const int dr = lane / 3 - 1, dc = lane % 3 - 1;
      const bool want = lane < 9 && ((m9 >> kBFacing[(lane / 3) % 3][lane % 3]) & 1u);
      bit_push(bg, bk, blk, want, (int)tc - dr, (int)tb - dc);
    }
    w = next;
  }
  covered = __reduce_add_sync(0xffffffffu, covered);
  if (lane == 0) {
    if (covered) atomicAdd(&bk.stat[1], (unsigned long long)covered);
    if (wmin != 0xFFFFFFFFu) atomicMin(flag.word, wmin);
  }
}

// F plane + layer-0 field from the dense occupancy (occ != 0: obstacle).  A warp
// builds 32 words of one plane row: 32 ballots over coalesced byte loads, the
// field cells (free: flag | 0, obstacle 0) written as it goes.
__global__ void k_bits_init(BitGeo bg, Geo g, const uint8_t* __restrict__ occ, uint32_t* __restrict__ F,
                            uint16_t* __restrict__ field, unsigned long long* __restrict__ free_cells) {
  const int lane = threadIdx.x & 31;
  const uint32_t row = blockIdx.y * (blockDim.x / 32) + (threadIdx.x >> 5);
  const uint32_t w0 = blockIdx.x * 32;
  if (row >= bg.rows) return;  // warp-uniform
  uint32_t mine = 0, cnt = 0;
  const bool in_row = row < bg.H;
  for (int k = 0; k < 32 && w0 + k < bg.wpr; ++k) {
    const uint32_t col = (w0 + k) * 32 + lane;
    const bool in = in_row && col < bg.W;
    const bool fr = in && occ[(size_t)row * bg.W + col] == 0;
    const uint32_t bits = __ballot_sync(0xffffffffu, fr);
    if (lane == k) mine = bits;
    if (in) field[(size_t)(row + g.pad) * g.pitch + g.pad + col] = fr ? (uint16_t)kFlag16 : (uint16_t)0;
  }
  if (w0 + lane < bg.wpr) F[(size_t)row * bg.wpr + w0 + lane] = mine;
  cnt = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(mine));
  if (lane == 0 && cnt) atomicAdd(free_cells, (unsigned long long)cnt);
}

// Sources (validated free cells): covered at layer 0 (activity lref + 1), and block 0's work list
// (the 3x3 tile neighbourhood of each source's tile, pushed as block "-1").  One warp per source.
__global__ void k_bits_sources(BitGeo bg, Geo g, const uint32_t* __restrict__ rc, uint64_t n, uint32_t* __restrict__ C,
                               uint16_t* __restrict__ field, BitBook bk, uint32_t lref) {
  const uint64_t s = blockIdx.x * (uint64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  if (s >= n) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const uint32_t r = rc[2 * s], c = rc[2 * s + 1];
  if (lane == 0) {
    const uint32_t bit = 1u << (c & 31);
    const uint32_t old = atomicOr(C + (size_t)r * bg.wpr + (c >> 5), bit);
    if (!(old & bit)) atomicAdd(&bk.stat[1], 1ull);
    field[(size_t)(r + g.pad) * g.pitch + g.pad + c] = (uint16_t)(kFlag16 | (lref + 1));
  }
  const int tc = (int)(r / kBTR), tb = (int)(c / (32 * kBTW));
  bit_push(bg, bk, 0xFFFFFFFFu, lane < 9, tc + lane / 3 - 1, tb + lane % 3 - 1);
}

}  // namespace

int bits_ctas_per_sm() {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_bits_tiles, kBThreads, 0) != cudaSuccess) n = 1;
  return n < 1 ? 1 : n;
}

void launch_bits_init(const BitGeo& bg, const Geo& g, const uint8_t* occ, BitBook bk, uint16_t* field,
                      cudaStream_t s) {
  const dim3 grid((bg.wpr + 31) / 32, (bg.rows + 7) / 8);
  k_bits_init<<<grid, 256, 0, s>>>(bg, g, occ, bk.F, field, bk.stat + 2);
}

void launch_bits_sources(const BitGeo& bg, const Geo& g, const uint32_t* rc, uint64_t n, BitBook bk, uint16_t* field,
                         uint32_t lref, cudaStream_t s) {
  if (!n) return;
  k_bits_sources<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(bg, g, rc, n, bk.C, field, bk, lref);
}

void launch_bits_tiles(const BitGeo& bg, const Geo& g, int ctas, uint16_t* field, BitBook bk, uint32_t blk,
                       uint32_t l0, uint32_t nl, uint32_t lref, FlagSink flag, FlagSink prev, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(kBThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_bits_tiles, bg, g, field, bk, blk, l0, nl, lref, flag, prev);
}

}  // namespace am
