// batch.cu -- small-grid throughput path (BASELINE.json config 5: 4096
// independent 256x256 mazes, 8 targets each).
//
// The mazes are packed side by side into one tall-and-wide field, each tile
// followed by an obstacle separator row/column, so the whole batch runs
// through the same temporally blocked stencil as one grid: separators are
// obstacles, which is exactly the zero padding every maze sees on its own
// (P6), so no activity crosses a tile border.  The global auto-L run stops
// when no maze gains cells; afterwards one CTA per maze reduces its smallest
// covered activity and whether a free cell is still zero.  Because a cell
// covered at layer l holds L_glob+1-l at the end, that minimum gives each
// maze's own last growing layer, hence its own layers_used / cause (pin P3)
// and its own exact rollback.  Path point counts are rollback invariant, so
// paths are traced on the packed field directly.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "am_host.hpp"

struct am_batch {
  am_grid* grid = nullptr;
  uint32_t n = 0, mw = 0, mh = 0, tiles_x = 0, tiles_y = 0;
  std::vector<uint32_t> layers_used, cause;  // per maze, after am_batch_propagate
  int have = 0;
  uint64_t* d_src_off = nullptr;  // K5: per-maze offsets into grid->src_rc (n + 1)
  uint32_t* d_k5 = nullptr;       // K5 scratch: used[n], cause[n], fetch counter
};

namespace am {

__global__ void k_batch_pack(const uint8_t* __restrict__ mazes, uint32_t n, uint32_t mw, uint32_t mh,
                             uint32_t tiles_x, uint32_t W, uint8_t* __restrict__ big) {
  const uint32_t i = blockIdx.y;  // maze
  const uint32_t cells = mw * mh;  // <= 65535^2 < 2^32
  const uint32_t tx = i % tiles_x, ty = i / tiles_x;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < cells; k += gridDim.x * blockDim.x) {
    const uint32_t r = k / mw, c = k - r * mw;
    big[(size_t)(ty * (mh + 1) + r) * W + tx * (mw + 1) + c] = mazes[(size_t)i * cells + k];
  }
  (void)n;
}

// per maze: min over covered free cells of a, and whether a free cell is 0
template <int CB>
__global__ void k_batch_stats(Geo g, const void* __restrict__ val, uint32_t mw, uint32_t mh, uint32_t tiles_x,
                              uint32_t* __restrict__ vmin, uint32_t* __restrict__ zero) {
  const uint32_t i = blockIdx.x;
  const uint32_t tx = i % tiles_x, ty = i / tiles_x;
  const uint32_t flag = CB == 16 ? kFlag16 : kFlag32, low = CB == 16 ? 0x7FFFu : kLow32;
  uint32_t m = 0xFFFFFFFFu, z = 0;
  // a warp per maze row (coalesced), no per-cell division
  const uint32_t lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (uint32_t rr = threadIdx.x >> 5; rr < mh; rr += nw) {
    const size_t base = g.idx(ty * (mh + 1) + rr, tx * (mw + 1));
    for (uint32_t cc = lane; cc < mw; cc += 32) {
      const uint32_t v = CB == 16 ? (uint32_t) static_cast<const uint16_t*>(val)[base + cc]
                                  : static_cast<const uint32_t*>(val)[base + cc];
      if (v & flag) {
        const uint32_t a = v & low;
        if (a == 0) z = 1;
        else m = a < m ? a : m;
      }
    }
  }
  m = __reduce_min_sync(0xffffffffu, m);
  z = __reduce_or_sync(0xffffffffu, z);
  __shared__ uint32_t sm[32], sz[32];
  if ((threadIdx.x & 31) == 0) {
    sm[threadIdx.x >> 5] = m;
    sz[threadIdx.x >> 5] = z;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const uint32_t nw = blockDim.x >> 5;
    m = threadIdx.x < nw ? sm[threadIdx.x] : 0xFFFFFFFFu;
    z = threadIdx.x < nw ? sz[threadIdx.x] : 0u;
    m = __reduce_min_sync(0xffffffffu, m);
    z = __reduce_or_sync(0xffffffffu, z);
    if (threadIdx.x == 0) {
      vmin[i] = m;
      zero[i] = z;
    }
  }
}

template <int CB>
__global__ void k_batch_decode(Geo g, const void* __restrict__ val, uint32_t mw, uint32_t mh, uint32_t tiles_x,
                               uint32_t computed, const uint32_t* __restrict__ used, uint32_t* __restrict__ out) {
  const uint32_t i = blockIdx.y;
  const uint32_t tx = i % tiles_x, ty = i / tiles_x;
  const uint32_t flag = CB == 16 ? kFlag16 : kFlag32, low = CB == 16 ? 0x7FFFu : kLow32;
  const uint32_t rb = computed - used[i];
  const uint32_t cells = mw * mh;  // <= 65535^2 < 2^32: 32-bit index arithmetic
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < cells; k += gridDim.x * blockDim.x) {
    const uint32_t kr = k / mw;
    const uint32_t r = ty * (mh + 1) + kr, c = tx * (mw + 1) + (k - kr * mw);
    const size_t idx = g.idx(r, c);
    const uint32_t v = CB == 16 ? (uint32_t) static_cast<const uint16_t*>(val)[idx] : static_cast<const uint32_t*>(val)[idx];
    const uint32_t a = v & low;
    out[(size_t)i * cells + k] = ((v & flag) && a) ? a - rb : 0u;
  }
}

// ---- K5: one CTA per maze, the whole maze on chip ------------------------------------------------------
//
// A layer's output differs from "every covered cell +1" (propagate.hpp:34-38 applied to a map whose covered
// cells already gained their +1) only at free, uncovered cells whose 3x3 neighbourhood holds a
// cell covered in the previous layer: there max3x3(A) = 1 > 0 and the ReLU output turns positive.  K5 runs
// the layer stack of one maze per CTA on that indicator, bit-parallel: the maze is held as bit planes (free,
// covered, last layer's new cells; 32 cells per word) in REGISTERS -- thread (g, k) owns word column k of
// the R rows [g*R, g*R+R) -- and a layer is, per word, the 3x3 max of the new-cell indicator (OR of the
// three rows: registers plus one halo word above and below published through shared memory; x | x<<1 |
// x>>1 plus the carries of the neighbour words: two lane shuffles), masked by free & ~covered.  Every
// other cell's value follows lazily: a cell covered at layer t holds L+1-t after L layers.  HBM is
// touched once for the occupancy (read) and once per cell for its encoded value (written into the packed
// field the trace and the download read, relative to L_ref = the cap / fixed L, so a maze's rollback is
// the existing `computed - layers_used` shift).  The per-layer count of new cells (one CTA barrier per
// layer) gives each maze's own auto-L outcome (pin P3) exactly.  CTAs fetch mazes dynamically.
constexpr int kWaveThreads = 256;

struct WaveArgs {
  Geo g;
  const uint8_t* occ;       // packed dense occupancy (g.W x g.H, row stride g.W)
  uint16_t* field;          // packed encoded field (16-bit cells)
  const uint32_t* src_rc;   // packed-field coordinates of every maze's sources, maze by maze
  const uint64_t* src_off;  // n + 1 offsets into src_rc (pairs)
  uint32_t n, mw, mh, tiles_x;
  uint32_t ww;              // words per maze row (ceil(mw / 32)); lanes per row group: wwp = pow2 >= ww
  uint32_t wwp_log2;
  uint32_t limit;           // auto: cap; fixed: L
  int autom;
  uint32_t lref;            // encoded values are lref + 1 - t
  uint32_t* used;           // per maze layers_used
  uint32_t* cause;          // per maze AM_STOP_*
  uint32_t* next;           // maze fetch counter (0 at launch)
};

// R rows per thread; shared memory: two staging planes (mh x ww words: free cells, sources) and the
// double-buffered halo rows (2 x groups x {top, bottom} x wwp words)
template <int R, int T>
__global__ void __launch_bounds__(T, (R * T) <= 2048 ? 1024 / T : ((R * T) <= 4096 ? 512 / T : 1)) k_batch_wave(WaveArgs a) {
  extern __shared__ uint32_t wsm[];
  const uint32_t ww = a.ww, wwp = 1u << a.wwp_log2, groups = T >> a.wwp_log2;
  const uint32_t nwords = a.mh * ww;
  uint32_t* s_free = wsm;
  uint32_t* s_src = s_free + nwords;
  uint32_t* halo = s_src + nwords;  // [2][groups][2][wwp]
  __shared__ uint32_t s_maze, s_cnt, s_new[3];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t k = tid & (wwp - 1), grp = tid >> a.wwp_log2, row0 = grp * R;
  const bool kin = k < ww;
  for (;;) {
    if (tid == 0) {
      s_maze = atomicAdd(a.next, 1u);
      s_cnt = 0;
      s_new[0] = s_new[1] = s_new[2] = 0;
    }
    for (uint32_t q = tid; q < nwords; q += T) s_src[q] = 0;
    __syncthreads();
    const uint32_t i = s_maze;
    if (i >= a.n) break;
    const uint32_t r0 = (i / a.tiles_x) * (a.mh + 1), c0 = (i % a.tiles_x) * (a.mw + 1);
    // occupancy -> free plane (a warp per row, one ballot per 32 cells, the row's loads issued together)
    // + the maze's layer-0 values in the field (free: flag, obstacle: 0)
    uint32_t nfree = 0;
    for (uint32_t r = warp; r < a.mh; r += T / 32) {
      const uint8_t* orow = a.occ + (size_t)(r0 + r) * a.g.W + c0;
      const size_t frow = a.g.idx(r0 + r, c0);
      for (uint32_t kb = 0; kb < ww; kb += 8) {
        uint8_t o[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t c = 32 * (kb + u) + lane;
          o[u] = (kb + u < ww && c < a.mw) ? orow[c] : 1;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t c = 32 * (kb + u) + lane;
          if (kb + u < ww && c < a.mw) a.field[frow + c] = o[u] ? (uint16_t)0 : (uint16_t)kFlag16;
          const uint32_t word = __ballot_sync(0xffffffffu, o[u] == 0);
          if (lane == 0 && kb + u < ww) {
            s_free[r * ww + kb + u] = word;
            nfree += __popc(word);
          }
        }
      }
    }
    if (lane == 0 && nfree) atomicAdd(&s_cnt, nfree);
    // sources (layer 0): value lref + 1
    const uint16_t vsrc = (uint16_t)(kFlag16 | (a.lref + 1));
    for (uint64_t s = a.src_off[i] + tid; s < a.src_off[i + 1]; s += T) {
      const uint32_t r = a.src_rc[2 * s] - r0, c = a.src_rc[2 * s + 1] - c0;
      atomicOr(&s_src[r * ww + (c >> 5)], 1u << (c & 31));
    }
    __syncthreads();
    // planes into registers; layer-0 new cells = the sources
    uint32_t fr[R], cv[R], nw[R];
    uint32_t nsrc = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const uint32_t r = row0 + j;
      const bool in = kin && r < a.mh;
      fr[j] = in ? s_free[r * ww + k] : 0u;
      cv[j] = in ? s_src[r * ww + k] : 0u;
      nw[j] = cv[j];
      nsrc += __popc(cv[j]);
      if (cv[j]) {
        const size_t base = a.g.idx(r0 + r, c0 + 32 * k);
        for (uint32_t m = cv[j]; m; m &= m - 1) a.field[base + (__ffs(m) - 1)] = vsrc;
      }
    }
    nsrc = __reduce_add_sync(0xffffffffu, nsrc);
    if (lane == 0 && nsrc) atomicAdd(&s_new[0], nsrc);
    halo[(grp * 2) * wwp + k] = nw[0];  // layer 0's halo rows: plane 0
    halo[(grp * 2 + 1) * wwp + k] = nw[R - 1];
    __syncthreads();
    const uint32_t free_total = s_cnt;
    uint32_t covered = s_new[0];
    uint32_t used = 0, why = AM_STOP_FIXED;
    const uint32_t hstride = groups * 2 * wwp;
    // per-thread constants of the layer loop: halo slots (read: the neighbours' rows of the other parity,
    // write: this group's top / bottom row) and the field address of the thread's first row
    const uint32_t* rd_up = halo + ((grp - 1) * 2 + 1) * wwp + k;  // + plane * hstride
    const uint32_t* rd_dn = halo + ((grp + 1) * 2) * wwp + k;
    uint32_t* wr_top = halo + (grp * 2) * wwp + k;
    const bool has_up = grp != 0, has_dn = grp + 1 < groups, kfirst = k == 0, klast = k + 1 == wwp;
    uint16_t* const mz = a.field + a.g.idx(r0 + row0, c0 + 32 * k);
    const uint32_t pitch = a.g.pitch;
    for (uint32_t l = 1;; ++l) {
      const uint32_t rp = (l - 1) & 1, wp = l & 1;  // halo plane read (last layer's) / written
      if (tid == 0) s_new[(l + 1) % 3] = 0;
      const uint32_t up = has_up ? rd_up[rp * hstride] : 0u;
      const uint32_t dn = has_dn ? rd_dn[rp * hstride] : 0u;
      uint32_t any = up | dn;
#pragma unroll
      for (int j = 0; j < R; ++j) any |= nw[j];
      uint32_t newc = 0;
      if (__any_sync(0xffffffffu, any)) {
        const uint16_t val = (uint16_t)(kFlag16 | (a.lref + 1 - l));
        uint32_t prev = up, v[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {  // vertical 3-row OR of last layer's new cells
          const uint32_t below = j + 1 < R ? nw[j + 1] : dn;
          v[j] = prev | nw[j] | below;
          prev = nw[j];
        }
#pragma unroll
        for (int j = 0; j < R; ++j) {  // horizontal: the word itself and the carries of its row neighbours
          uint32_t lft = __shfl_up_sync(0xffffffffu, v[j], 1);
          uint32_t rgt = __shfl_down_sync(0xffffffffu, v[j], 1);
          if (kfirst) lft = 0;
          if (klast) rgt = 0;
          const uint32_t h = v[j] | (v[j] << 1) | (v[j] >> 1) | (lft >> 31) | (rgt << 31);
          const uint32_t n = h & fr[j] & ~cv[j];
          cv[j] |= n;
          nw[j] = n;
          newc += __popc(n);
        }
        // the new cells' values
#pragma unroll
        for (int j = 0; j < R; ++j) {
          uint16_t* row = mz + j * pitch;
          for (uint32_t m = nw[j]; m; m &= m - 1) row[__ffs(m) - 1] = val;
        }
      } else {
#pragma unroll
        for (int j = 0; j < R; ++j) nw[j] = 0;
      }
      wr_top[wp * hstride] = nw[0];
      wr_top[wp * hstride + wwp] = nw[R - 1];
      newc = __reduce_add_sync(0xffffffffu, newc);
      if (lane == 0 && newc) atomicAdd(&s_new[l % 3], newc);
      __syncthreads();
      const uint32_t got = s_new[l % 3];
      covered += got;
      // pin P3: filled, else stalled, else cap; fixed L: stop at L (or once nothing moves:
      // the remaining layers only add the lazy +1, already in the values)
      if (a.autom) {
        if (covered == free_total) { used = l; why = AM_STOP_FILLED; break; }
        if (got == 0) { used = l; why = AM_STOP_STALLED; break; }
        if (l >= a.limit) { used = a.limit; why = AM_STOP_CAP; break; }
      } else if (l >= a.limit || got == 0) {
        used = a.limit;
        break;
      }
    }
    if (tid == 0) {
      a.used[i] = used;
      a.cause[i] = why;
    }
    __syncthreads();  // shared planes reused by the next maze
  }
}

// rows per thread for a maze of mh rows with 2^wwp_log2 lanes per row group (0: no instantiation fits)
inline int wave_rows(uint32_t mh, uint32_t wwp_log2, uint32_t threads) {
  const uint32_t groups = threads >> wwp_log2;
  const uint32_t need = (mh + groups - 1) / groups;
  for (int r = 1; r <= 32; r *= 2)
    if ((uint32_t)r >= need) return r;
  return 0;
}

}  // namespace am

using namespace am;

extern "C" {

am_status am_batch_create(am_ctx* ctx, uint32_t n, uint32_t mw, uint32_t mh, const uint8_t* occ,
                          const uint64_t* src_off, const uint32_t* src_rc, am_batch** out) {
  if (!ctx || !out || !occ || !src_off || !src_rc || n == 0 || mw == 0 || mh == 0) return AM_EINVAL;
  *out = nullptr;
  // near-square tile arrangement that fits kMaxGridDim
  uint32_t tx = (uint32_t)std::ceil(std::sqrt((double)n * (mh + 1) / (double)(mw + 1)));
  tx = std::max(1u, std::min(tx, n));
  const uint32_t ty = (n + tx - 1) / tx;
  const uint64_t W = (uint64_t)tx * (mw + 1), H = (uint64_t)ty * (mh + 1);
  if (W > 65535 || H > 65535) return fail(ctx, AM_EINVAL, "batch of %u mazes %ux%u does not fit one field", n, mw, mh);
  std::vector<uint32_t> big_src;
  for (uint32_t i = 0; i < n; ++i) {
    if (src_off[i + 1] <= src_off[i]) return fail(ctx, AM_EINVAL, "maze %u: SourceSet must be nonempty", i);
    for (uint64_t k = src_off[i]; k < src_off[i + 1]; ++k) {
      const uint32_t r = src_rc[2 * k], c = src_rc[2 * k + 1];
      if (r >= mh || c >= mw) return fail(ctx, AM_EINVAL, "maze %u: source (%u,%u) out of bounds", i, r, c);
      big_src.push_back((i / tx) * (mh + 1) + r);
      big_src.push_back((i % tx) * (mw + 1) + c);
    }
  }
  CK(cudaSetDevice(ctx->device));
  uint8_t *d_m = nullptr, *d_big = nullptr;
  CK(am::dmalloc(ctx, &d_big, W * H));
  cudaError_t e = am::dmalloc(ctx, &d_m, (size_t)n * mw * mh);
  if (!e) e = cudaMemsetAsync(d_big, 1, W * H, ctx->stream);  // separators / unused tiles are obstacles
  if (!e) e = cudaMemcpyAsync(d_m, occ, (size_t)n * mw * mh, cudaMemcpyHostToDevice, ctx->stream);
  if (!e) {
    k_batch_pack<<<dim3(64, n), 256, 0, ctx->stream>>>(d_m, n, mw, mh, tx, (uint32_t)W, d_big);
    ++ctx->launches;
    e = cudaPeekAtLastError();
  }
  if (!e) e = cudaStreamSynchronize(ctx->stream);
  if (e) {
    am::dfree(ctx, d_m);
    am::dfree(ctx, d_big);
    (void)cudaGetLastError();
    return fail(ctx, AM_ECUDA, "batch pack: %s", cudaGetErrorString(e));
  }
  am_batch* b = new (std::nothrow) am_batch();
  if (!b) return AM_EOOM;
  b->n = n;
  b->mw = mw;
  b->mh = mh;
  b->tiles_x = tx;
  b->tiles_y = ty;
  // sources are host data (big_src); the packed occupancy is device data
  uint32_t* d_src = nullptr;
  e = am::dmalloc(ctx, &d_src, big_src.size() * 4);
  if (!e) e = cudaMemcpyAsync(d_src, big_src.data(), big_src.size() * 4, cudaMemcpyHostToDevice, ctx->stream);
  am_status st = e ? fail(ctx, AM_ECUDA, "%s", cudaGetErrorString(e))
                   : grid_create_rows(ctx, (uint32_t)W, (uint32_t)H, 0, (uint32_t)H, d_big, d_src, big_src.size() / 2,
                                      true, false, &b->grid);
  am::dfree(ctx, d_src);
  am::dfree(ctx, d_m);
  am::dfree(ctx, d_big);
  if (!st) {  // K5 bookkeeping: where each maze's sources start in the packed list
    std::vector<uint64_t> off(src_off, src_off + n + 1);
    for (auto& o : off) o -= src_off[0];
    e = am::dmalloc(ctx, &b->d_src_off, (n + 1) * 8);
    if (!e) e = am::dmalloc(ctx, &b->d_k5, (2 * (size_t)n + 4) * 4);
    if (!e) e = cudaMemcpyAsync(b->d_src_off, off.data(), (n + 1) * 8, cudaMemcpyHostToDevice, ctx->stream);
    if (!e) e = cudaStreamSynchronize(ctx->stream);
    if (e) st = fail(ctx, AM_ECUDA, "batch: %s", cudaGetErrorString(e));
  }
  if (st) {
    if (b->grid) am_grid_destroy(ctx, b->grid);
    am::dfree(ctx, b->d_src_off);
    am::dfree(ctx, b->d_k5);
    delete b;
    return st;
  }
  *out = b;
  return AM_OK;
}

am_status am_batch_destroy(am_ctx* ctx, am_batch* b) {
  if (!b) return AM_OK;
  am_grid_destroy(ctx, b->grid);
  am::dfree(ctx, b->d_src_off);
  am::dfree(ctx, b->d_k5);
  delete b;
  return AM_OK;
}

}  // extern "C"

namespace {

struct WaveShape {
  uint32_t ww, wwp_log2;
  int rows;     // rows per thread (template instance), 0: the batch does not fit K5
  size_t smem;  // dynamic shared memory per CTA
  uint32_t threads;
};

// CTA size (A/B: AM_K5_THREADS = 128 / 256 / 512)
uint32_t wave_threads() {
  static const uint32_t t = [] {
    const char* e = std::getenv("AM_K5_THREADS");
    const int v = e ? std::atoi(e) : kWaveThreads;
    return (uint32_t)(v == 128 || v == 512 ? v : kWaveThreads);
  }();
  return t;
}

WaveShape wave_shape(const am_batch* b) {
  WaveShape w{};
  w.threads = wave_threads();
  w.ww = (b->mw + 31) / 32;
  if (w.ww > 32) return w;
  while ((1u << w.wwp_log2) < w.ww) ++w.wwp_log2;
  w.rows = wave_rows(b->mh, w.wwp_log2, w.threads);
  const uint32_t groups = w.threads >> w.wwp_log2;
  w.smem = (size_t)2 * b->mh * w.ww * 4 + (size_t)2 * groups * 2 * (1u << w.wwp_log2) * 4;
  if (w.smem > 200 * 1024) w.rows = 0;
  return w;
}

bool wave_eligible(const am_batch* b, uint32_t lref) {
  static const bool off = [] {
    const char* e = std::getenv("AM_BATCH_TILES");  // A/B: the packed tile path for every batch
    return e && *e == '1';
  }();
  return !off && (uint64_t)lref + 1 <= kMax16Activity && wave_shape(b).rows > 0;
}

template <int R, int T>
cudaError_t wave_launch_t(const WaveArgs& a, size_t smem, int sms, uint32_t n, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_batch_wave<R, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e) return e;
    attr = true;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_batch_wave<R, T>, T, smem);
  if (e) return e;
  const uint32_t grid = (uint32_t)std::min<uint64_t>(n, (uint64_t)std::max(per_sm, 1) * sms);
  k_batch_wave<R, T><<<grid, T, smem, s>>>(a);
  return cudaPeekAtLastError();
}

template <int R>
cudaError_t wave_launch(const WaveArgs& a, size_t smem, int sms, uint32_t n, uint32_t threads, cudaStream_t s) {
  if (threads == 128) return wave_launch_t<R, 128>(a, smem, sms, n, s);
  if (threads == 512) return wave_launch_t<R, 512>(a, smem, sms, n, s);
  return wave_launch_t<R, kWaveThreads>(a, smem, sms, n, s);
}

// K5: the whole batch in one launch, per-maze layers_used / cause straight from the wavefronts
am_status wave_propagate(am_ctx* ctx, am_batch* b, uint32_t layers, uint32_t auto_cap, uint32_t lref,
                         am_prop_result* r) {
  am_grid* g = b->grid;
  am_status st = set_cell_bits(ctx, g, 16);
  if (st) return st;
  cudaStream_t s = ctx->stream;
  const WaveShape w = wave_shape(b);
  uint32_t* used = b->d_k5;
  uint32_t* cause = used + b->n;
  uint32_t* next = cause + b->n;
  CK(cudaMemsetAsync(next, 0, 4, s));
  WaveArgs a{};
  a.g = g->g;
  a.occ = g->occ;
  a.field = static_cast<uint16_t*>(g->val[g->cur]);
  a.src_rc = g->src_rc;
  a.src_off = b->d_src_off;
  a.n = b->n;
  a.mw = b->mw;
  a.mh = b->mh;
  a.tiles_x = b->tiles_x;
  a.ww = w.ww;
  a.wwp_log2 = w.wwp_log2;
  a.autom = layers == 0;
  a.limit = layers ? layers : auto_cap;
  a.lref = lref;
  a.used = used;
  a.cause = cause;
  a.next = next;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const bool timing = ctx->flags & AM_CTX_TIMING;
  if (timing) {
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, s));
  }
  switch (w.rows) {
    case 1: CK(wave_launch<1>(a, w.smem, ctx->sms, b->n, w.threads, s)); break;
    case 2: CK(wave_launch<2>(a, w.smem, ctx->sms, b->n, w.threads, s)); break;
    case 4: CK(wave_launch<4>(a, w.smem, ctx->sms, b->n, w.threads, s)); break;
    case 8: CK(wave_launch<8>(a, w.smem, ctx->sms, b->n, w.threads, s)); break;
    case 16: CK(wave_launch<16>(a, w.smem, ctx->sms, b->n, w.threads, s)); break;
    default: CK(wave_launch<32>(a, w.smem, ctx->sms, b->n, w.threads, s)); break;
  }
  ++ctx->launches;
  if (timing) CK(cudaEventRecord(e1, s));
  b->layers_used.resize(b->n);
  b->cause.resize(b->n);
  CK(cudaMemcpyAsync(b->layers_used.data(), used, b->n * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(b->cause.data(), cause, b->n * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  float ms = 0.f;
  if (timing) {
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  g->computed = g->layers_used = lref;  // values are lref + 1 - t; maze i's rollback is lref - used[i]
  g->plain_active = 0;
  g->have_map = 1;
  g->bits_map = 0;
  uint32_t maxl = 0;
  uint64_t sum_used = 0;
  for (uint32_t u : b->layers_used) maxl = std::max(maxl, u), sum_used += u;
  *r = am_prop_result{};
  r->cells_executed = sum_used * (uint64_t)b->mw * b->mh;  // every maze's cells x its own layers (on chip)
  r->engine = AM_ENGINE_BATCH;
  r->block_layers = 0;  // one launch runs every maze to its fixed point
  r->layers_used = maxl;
  r->cause = layers ? AM_STOP_FIXED : AM_STOP_CAP;
  r->layers_computed = maxl;
  r->cell_bits = 16;
  r->block_launches = 1;
  r->stencil_ms = ms;
  return AM_OK;
}

}  // namespace

extern "C" {

am_status am_batch_propagate(am_ctx* ctx, am_batch* b, uint32_t layers, uint32_t auto_cap, uint32_t* layers_used,
                             uint32_t* cause, am_prop_result* global) {
  if (!ctx || !b) return AM_EINVAL;
  if (layers == 0 && auto_cap == 0) return fail(ctx, AM_EINVAL, "auto_cap must be >= 1");
  if (layers > kMaxLayers || auto_cap > kMaxLayers) return fail(ctx, AM_EINVAL, "layer count exceeds kMaxLayers");
  CK(cudaSetDevice(ctx->device));
  const uint32_t lref = layers ? layers : auto_cap;
  if (wave_eligible(b, lref)) {
    am_prop_result r{};
    am_status st = wave_propagate(ctx, b, layers, auto_cap, lref, &r);
    if (st) return st;
    if (layers_used) memcpy(layers_used, b->layers_used.data(), b->n * 4);
    if (cause) memcpy(cause, b->cause.data(), b->n * 4);
    if (global) *global = r;
    b->have = 1;
    return AM_OK;
  }
  std::vector<SlabRef> one{{ctx, b->grid}};
  am_prop_result r{};
  am_status st = drive_propagation(one, nullptr, layers, auto_cap, AM_MODE_BATCHED, &r);
  if (st) return st;
  am_grid* g = b->grid;
  b->layers_used.assign(b->n, r.layers_used);
  b->cause.assign(b->n, AM_STOP_FIXED);
  if (layers == 0) {
    uint32_t *d_min = nullptr, *d_zero = nullptr;
    CK(am::dmalloc(ctx, &d_min, b->n * 4));
    cudaError_t e = am::dmalloc(ctx, &d_zero, b->n * 4);
    std::vector<uint32_t> vmin(b->n), zero(b->n);
    if (!e) {
      if (g->cell_bits == 16)
        k_batch_stats<16><<<b->n, 256, 0, ctx->stream>>>(g->g, g->val[g->cur], b->mw, b->mh, b->tiles_x, d_min, d_zero);
      else
        k_batch_stats<32><<<b->n, 256, 0, ctx->stream>>>(g->g, g->val[g->cur], b->mw, b->mh, b->tiles_x, d_min, d_zero);
      ++ctx->launches;
      e = cudaPeekAtLastError();
    }
    if (!e) e = cudaMemcpyAsync(vmin.data(), d_min, b->n * 4, cudaMemcpyDeviceToHost, ctx->stream);
    if (!e) e = cudaMemcpyAsync(zero.data(), d_zero, b->n * 4, cudaMemcpyDeviceToHost, ctx->stream);
    if (!e) e = cudaStreamSynchronize(ctx->stream);
    am::dfree(ctx, d_min);
    am::dfree(ctx, d_zero);
    if (e) return fail(ctx, AM_ECUDA, "batch stats: %s", cudaGetErrorString(e));
    const uint32_t L = g->computed;
    for (uint32_t i = 0; i < b->n; ++i) {
      // last layer that covered a new cell in maze i (0: only its sources are covered)
      const uint64_t last = vmin[i] == 0xFFFFFFFFu ? 0 : (uint64_t)L + 1 - vmin[i];
      const uint64_t lp = last + 1;  // first layer without new cells
      uint32_t used, why;
      if (lp <= auto_cap) {
        if (!zero[i]) {
          used = (uint32_t)std::max<uint64_t>(1, lp - 1);
          why = AM_STOP_FILLED;
        } else {
          used = (uint32_t)lp;
          why = AM_STOP_STALLED;
        }
      } else {
        used = auto_cap;
        why = zero[i] ? AM_STOP_CAP : AM_STOP_FILLED;
      }
      b->layers_used[i] = used;
      b->cause[i] = why;
    }
  }
  if (layers_used) memcpy(layers_used, b->layers_used.data(), b->n * 4);
  if (cause) memcpy(cause, b->cause.data(), b->n * 4);
  if (global) *global = r;
  b->have = 1;
  return AM_OK;
}

am_status am_batch_download(am_ctx* ctx, am_batch* b, uint32_t* maps) {
  if (!ctx || !b || !maps) return AM_EINVAL;
  if (!b->have) return fail(ctx, AM_EINVAL, "batch: propagate first");
  am_grid* g = b->grid;
  const size_t bytes = (size_t)b->n * b->mw * b->mh * 4;
  uint32_t *d_out = nullptr, *d_used = nullptr;
  CK(am::dmalloc(ctx, &d_out, bytes));
  cudaError_t e = am::dmalloc(ctx, &d_used, b->n * 4);
  if (!e) e = cudaMemcpyAsync(d_used, b->layers_used.data(), b->n * 4, cudaMemcpyHostToDevice, ctx->stream);
  if (!e) {
    if (g->cell_bits == 16)
      k_batch_decode<16><<<dim3(16, b->n), 256, 0, ctx->stream>>>(g->g, g->val[g->cur], b->mw, b->mh, b->tiles_x,
                                                                  g->computed, d_used, d_out);
    else
      k_batch_decode<32><<<dim3(16, b->n), 256, 0, ctx->stream>>>(g->g, g->val[g->cur], b->mw, b->mh, b->tiles_x,
                                                                  g->computed, d_used, d_out);
    ++ctx->launches;
    e = cudaPeekAtLastError();
  }
  if (!e) e = cudaMemcpyAsync(maps, d_out, bytes, cudaMemcpyDeviceToHost, ctx->stream);
  if (!e) e = cudaStreamSynchronize(ctx->stream);
  am::dfree(ctx, d_out);
  am::dfree(ctx, d_used);
  if (e) return fail(ctx, AM_ECUDA, "batch download: %s", cudaGetErrorString(e));
  return AM_OK;
}

// targets: (maze, row, col) triples in maze-local coordinates
static am_status batch_targets(am_ctx* ctx, am_batch* b, const uint32_t* tgt, uint64_t n, std::vector<uint32_t>& big,
                               std::vector<uint8_t>& bad) {
  big.resize(2 * n);
  bad.assign(n, 0);
  for (uint64_t k = 0; k < n; ++k) {
    const uint32_t i = tgt[3 * k], r = tgt[3 * k + 1], c = tgt[3 * k + 2];
    if (i >= b->n || r >= b->mh || c >= b->mw) {
      bad[k] = 1;
      big[2 * k] = big[2 * k + 1] = 0xFFFFFFFFu;  // rejected by the device bounds check
      continue;
    }
    big[2 * k] = (i / b->tiles_x) * (b->mh + 1) + r;
    big[2 * k + 1] = (i % b->tiles_x) * (b->mw + 1) + c;
  }
  (void)ctx;
  return AM_OK;
}

am_status am_batch_path_counts(am_ctx* ctx, am_batch* b, const uint32_t* tgt, uint64_t n, uint32_t method,
                               uint64_t seed, uint64_t* offsets, int32_t* status) {
  if (!ctx || !b || (n && (!tgt || !status)) || !offsets) return AM_EINVAL;
  std::vector<uint32_t> big;
  std::vector<uint8_t> bad;
  batch_targets(ctx, b, tgt, n, big, bad);
  return am_path_counts(ctx, b->grid, big.data(), n, method, seed, offsets, status);
}

am_status am_batch_trace_paths(am_ctx* ctx, am_batch* b, const uint32_t* tgt, uint64_t n, uint32_t method,
                               uint64_t seed, const uint64_t* offsets, uint32_t* pts, uint64_t cap, int32_t* status) {
  if (!ctx || !b || (n && (!tgt || !status)) || !offsets) return AM_EINVAL;
  std::vector<uint32_t> big;
  std::vector<uint8_t> bad;
  batch_targets(ctx, b, tgt, n, big, bad);
  // maze-local coordinates are produced on the device (mazes sit on a (mh+1) x (mw+1) lattice)
  return trace_paths_host(ctx, b->grid, big.data(), n, method, seed, offsets, pts, cap, status, b->mh + 1, b->mw + 1);
}

}  // extern "C"
