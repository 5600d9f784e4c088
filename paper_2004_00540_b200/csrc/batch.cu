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
#include <cstring>
#include <new>
#include <vector>

#include "am_host.hpp"

struct am_batch {
  am_grid* grid = nullptr;
  uint32_t n = 0, mw = 0, mh = 0, tiles_x = 0, tiles_y = 0;
  std::vector<uint32_t> layers_used, cause;  // per maze, after am_batch_propagate
  int have = 0;
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
  if (st) {
    delete b;
    return st;
  }
  *out = b;
  return AM_OK;
}

am_status am_batch_destroy(am_ctx* ctx, am_batch* b) {
  if (!b) return AM_OK;
  am_grid_destroy(ctx, b->grid);
  delete b;
  return AM_OK;
}

am_status am_batch_propagate(am_ctx* ctx, am_batch* b, uint32_t layers, uint32_t auto_cap, uint32_t* layers_used,
                             uint32_t* cause, am_prop_result* global) {
  if (!ctx || !b) return AM_EINVAL;
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
