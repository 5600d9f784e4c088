// capi.cu -- host orchestration behind include/actmap_b200.h.
//
// propagate_auto on the device (propagate.hpp:57-61, pin P3): temporally
// blocked launches of kK layers each, with the fixed-point signal of block b
// read back (pinned copy + event) only after block b+1 is already queued, so
// the GPU never idles on the host.  Coverage growth is monotone
// (new cells at layer l imply new cells at layer l-1), so one number per
// block -- the smallest activity among covered cells -- locates the first
// layer without new cells exactly; blocks launched past it are undone by
// subtracting the overshoot from every covered cell (exact: a covered cell
// gains exactly +1 per layer once coverage is fixed).
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <deque>
#include <new>
#include <string>
#include <vector>

#include "../../include/actmap_b200.h"
#include "am_internal.cuh"

using am::Geo;

namespace {

constexpr int kFlagSlots = 64;
constexpr int kLag = 2;  // blocks in flight before the host reads a flag

struct Timer {
  cudaEvent_t a, b;
};

}  // namespace

struct am_ctx {
  int device = 0;
  uint32_t flags = 0;
  cudaStream_t stream = nullptr;
  int sms = 148;
  int warp_slots = 0;
  uint64_t launches = 0;
  std::string err;
  std::vector<Timer> timers;
};

struct am_grid {
  Geo g{};
  int cell_bits = 16;
  void* val[2] = {nullptr, nullptr};
  int cur = 0;
  uint8_t* srcmask = nullptr;        // pitched 0/1
  uint8_t* rowsrc = nullptr;         // per allocated row: any source
  uint8_t* occ = nullptr;            // dense W*H (kept for re-init / plain maps)
  uint8_t* srcmask_dense = nullptr;  // dense W*H (plain maps)
  uint32_t* d_flags = nullptr;       // kFlagSlots fixed-point slots
  uint32_t* h_flags = nullptr;       // pinned mirror
  cudaEvent_t flag_ev[kFlagSlots];
  uint32_t* plain = nullptr;         // caller-uploaded dense map
  int plain_active = 0;
  uint32_t plain_layers = 0;
  int have_map = 0;
  int dirty[2] = {0, 0};    // buffer reused as download staging: padding no longer unflagged
  uint32_t computed = 0;    // layers represented by val[cur]
  uint32_t layers_used = 0; // logical layers (val[cur] minus rollback)
  // scratch for path extraction
  uint32_t* d_tgt = nullptr;
  uint64_t* d_counts = nullptr;
  uint64_t* d_offsets = nullptr;
  int32_t* d_status = nullptr;
  uint64_t tgt_cap = 0;
  uint32_t* d_pts = nullptr;
  uint64_t pts_cap = 0;
};

static am_status fail(am_ctx* ctx, am_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return st;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      (void)cudaGetLastError();                                                         \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? AM_EOOM : AM_ECUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                   \
    }                                                                                   \
  } while (0)

#define CKL()                        \
  do {                               \
    ++ctx->launches;                 \
    CK(cudaPeekAtLastError());       \
  } while (0)

static bool dims_ok(uint32_t w, uint32_t h) { return w >= 1 && h >= 1 && w <= 65535 && h <= 65535; }

extern "C" {

am_status am_ctx_create(const am_ctx_opts* opts, am_ctx** out) {
  if (!out) return AM_EINVAL;
  *out = nullptr;
  am_ctx* ctx = new (std::nothrow) am_ctx();
  if (!ctx) return AM_EOOM;
  ctx->device = opts ? opts->device : 0;
  ctx->flags = opts ? opts->flags : 0;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    (void)cudaGetLastError();
    return AM_ECUDA;
  }
  cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, ctx->device);
  int bps = am::block_kernel_blocks_per_sm(16);
  if (bps < 1) bps = 1;
  ctx->warp_slots = ctx->sms * bps * (am::kBlockThreads / 32);
  *out = ctx;
  return AM_OK;
}

void am_ctx_destroy(am_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (auto& t : ctx->timers) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* am_last_error(const am_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

am_status am_ctx_stats(const am_ctx* ctx, am_stats* out) {
  if (!ctx || !out) return AM_EINVAL;
  out->kernel_launches = ctx->launches;
  return AM_OK;
}

am_status am_ctx_get_stream(const am_ctx* ctx, void** stream) {
  if (!ctx || !stream) return AM_EINVAL;
  *stream = (void*)ctx->stream;
  return AM_OK;
}

am_status am_ctx_synchronize(am_ctx* ctx) {
  if (!ctx) return AM_EINVAL;
  CK(cudaStreamSynchronize(ctx->stream));
  return AM_OK;
}

static void grid_free(am_grid* g) {
  if (!g) return;
  for (int i = 0; i < 2; ++i) cudaFree(g->val[i]);
  cudaFree(g->srcmask);
  cudaFree(g->rowsrc);
  cudaFree(g->occ);
  cudaFree(g->srcmask_dense);
  cudaFree(g->d_flags);
  if (g->h_flags) cudaFreeHost(g->h_flags);
  for (int i = 0; i < kFlagSlots; ++i)
    if (g->flag_ev[i]) cudaEventDestroy(g->flag_ev[i]);
  cudaFree(g->plain);
  cudaFree(g->d_tgt);
  cudaFree(g->d_counts);
  cudaFree(g->d_offsets);
  cudaFree(g->d_status);
  cudaFree(g->d_pts);
  delete g;
}

static am_status grid_create_impl(am_ctx* ctx, uint32_t W, uint32_t H, const uint8_t* occ, const uint32_t* src,
                                  uint64_t n_src, bool device_ptrs, am_grid** out) {
  if (!ctx || !out) return AM_EINVAL;
  *out = nullptr;
  if (!dims_ok(W, H)) return fail(ctx, AM_EINVAL, "grid dimensions %ux%u outside 1..65535", W, H);
  if (n_src == 0) return fail(ctx, AM_EINVAL, "SourceSet must be nonempty");
  if (!occ || !src) return fail(ctx, AM_EINVAL, "null occupancy or sources");
  CK(cudaSetDevice(ctx->device));
  am_grid* g = new (std::nothrow) am_grid();
  if (!g) return AM_EOOM;
  memset(g->flag_ev, 0, sizeof g->flag_ev);
  g->g = am::make_geo(W, H, ctx->warp_slots);
  const size_t cells = (size_t)g->g.rows * g->g.pitch;
  const size_t dense = (size_t)W * H;
  cudaStream_t s = ctx->stream;
  am_status st = AM_OK;
  auto bail = [&](am_status code) {
    grid_free(g);
    return code;
  };
#define GCK(call)                                                                             \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      (void)cudaGetLastError();                                                               \
      st = fail(ctx, e_ == cudaErrorMemoryAllocation ? AM_EOOM : AM_ECUDA, "%s: %s", #call,   \
                cudaGetErrorString(e_));                                                      \
      return bail(st);                                                                        \
    }                                                                                         \
  } while (0)
  GCK(cudaMalloc(&g->val[0], cells * 2));
  GCK(cudaMalloc(&g->val[1], cells * 2));
  GCK(cudaMalloc(&g->srcmask, cells));
  GCK(cudaMalloc(&g->rowsrc, g->g.rows));
  GCK(cudaMalloc(&g->occ, dense));
  GCK(cudaMalloc(&g->srcmask_dense, dense));
  GCK(cudaMalloc(&g->d_flags, kFlagSlots * sizeof(uint32_t)));
  GCK(cudaHostAlloc(&g->h_flags, kFlagSlots * sizeof(uint32_t), cudaHostAllocDefault));
  for (int i = 0; i < kFlagSlots; ++i) GCK(cudaEventCreateWithFlags(&g->flag_ev[i], cudaEventDisableTiming));
  GCK(cudaMemsetAsync(g->val[0], 0, cells * 2, s));
  GCK(cudaMemsetAsync(g->val[1], 0, cells * 2, s));
  GCK(cudaMemsetAsync(g->srcmask, 0, cells, s));
  GCK(cudaMemsetAsync(g->rowsrc, 0, g->g.rows, s));
  GCK(cudaMemsetAsync(g->srcmask_dense, 0, dense, s));
  GCK(cudaMemcpyAsync(g->occ, occ, dense, device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  uint32_t* d_src = nullptr;
  int* d_err = nullptr;
  GCK(cudaMalloc(&d_src, n_src * 2 * sizeof(uint32_t)));
  GCK(cudaMalloc(&d_err, sizeof(int)));
  GCK(cudaMemsetAsync(d_err, 0, sizeof(int), s));
  GCK(cudaMemcpyAsync(d_src, src, n_src * 2 * sizeof(uint32_t),
                      device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  am::launch_srcmask_dense(W, H, d_src, n_src, g->srcmask_dense, g->occ, d_err, s);
  ++ctx->launches;
  am::launch_scatter_sources(g->g, d_src, n_src, g->srcmask, g->rowsrc, d_err, s);
  ++ctx->launches;
  int h_err = 0;
  GCK(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  GCK(cudaStreamSynchronize(s));
  cudaFree(d_src);
  cudaFree(d_err);
  if (h_err) {
    grid_free(g);
    return fail(ctx, AM_EINVAL, "SourceSet: a source is out of bounds or on an obstacle (grid.hpp:78)");
  }
#undef GCK
  *out = g;
  return AM_OK;
}

am_status am_grid_create(am_ctx* ctx, uint32_t W, uint32_t H, const uint8_t* occ, const uint32_t* src,
                         uint64_t n_src, am_grid** out) {
  return grid_create_impl(ctx, W, H, occ, src, n_src, false, out);
}

am_status am_grid_create_device(am_ctx* ctx, uint32_t W, uint32_t H, const uint8_t* occ, const uint32_t* src,
                                uint64_t n_src, am_grid** out) {
  return grid_create_impl(ctx, W, H, occ, src, n_src, true, out);
}

am_status am_grid_destroy(am_ctx* ctx, am_grid* g) {
  if (ctx) cudaSetDevice(ctx->device);
  if (ctx && ctx->stream) cudaStreamSynchronize(ctx->stream);
  grid_free(g);
  return AM_OK;
}

am_status am_grid_get_info(const am_grid* g, am_grid_info* o) {
  if (!g || !o) return AM_EINVAL;
  o->width = g->g.W;
  o->height = g->g.H;
  o->pitch = g->g.pitch;
  o->rows = g->g.rows;
  o->bands = g->g.nbands;
  o->segments = g->g.nseg;
  o->seg_len = g->g.seg_len;
  o->halo = g->g.pad;
  o->cell_bits = g->cell_bits;
  o->layers_used = g->layers_used;
  o->layers_computed = g->computed;
  return AM_OK;
}

// ---------------------------------------------------------------- propagate

struct PendingBlock {
  int slot;
  uint32_t start;  // layers before the block
  uint32_t count;  // layers in the block
  int cell_bits;
};

// Layers-before-first-layer-without-new-cells (l'), or 0 if the block still
// added cells in its last layer.
static uint32_t block_termination(const PendingBlock& b, uint32_t m) {
  const uint32_t none = b.cell_bits == 16 ? 0x7FFFu : 0x7FFFFFFFu;
  uint64_t vmin = m >= none ? 0xFFFFFFFFull : (uint64_t)m + 1;  // smallest covered activity
  if (vmin < 2) return 0;                                        // a cell reached a=1 in the last layer
  const uint64_t capped = vmin < (uint64_t)b.count + 1 ? vmin : (uint64_t)b.count + 1;
  return (uint32_t)((uint64_t)b.start + b.count + 2 - capped);
}

static am_status promote(am_ctx* ctx, am_grid* g) {
  const size_t cells = (size_t)g->g.rows * g->g.pitch;
  void* n0 = nullptr;
  void* n1 = nullptr;
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaMalloc(&n0, cells * 4));
  cudaError_t e = cudaMalloc(&n1, cells * 4);
  if (e != cudaSuccess) {
    cudaFree(n0);
    (void)cudaGetLastError();
    return fail(ctx, AM_EOOM, "32-bit promotion: %s", cudaGetErrorString(e));
  }
  am::launch_promote(g->g, (const uint16_t*)g->val[g->cur], (uint32_t*)n0, ctx->stream);
  CKL();
  CK(cudaMemsetAsync(n1, 0, cells * 4, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  cudaFree(g->val[0]);
  cudaFree(g->val[1]);
  g->val[0] = n0;
  g->val[1] = n1;
  g->cur = 0;
  g->cell_bits = 32;
  return AM_OK;
}

static am_status reset_map(am_ctx* ctx, am_grid* g, int cell_bits) {
  const size_t cells = (size_t)g->g.rows * g->g.pitch;
  if (g->cell_bits != cell_bits) {
    cudaFree(g->val[0]);
    cudaFree(g->val[1]);
    g->val[0] = g->val[1] = nullptr;
    const size_t bytes = cells * (cell_bits / 8);
    CK(cudaMalloc(&g->val[0], bytes));
    CK(cudaMalloc(&g->val[1], bytes));
    CK(cudaMemsetAsync(g->val[0], 0, bytes, ctx->stream));
    CK(cudaMemsetAsync(g->val[1], 0, bytes, ctx->stream));
    g->cell_bits = cell_bits;
    g->dirty[0] = g->dirty[1] = 0;
  }
  for (int i = 0; i < 2; ++i)
    if (g->dirty[i]) {
      CK(cudaMemsetAsync(g->val[i], 0, cells * (cell_bits / 8), ctx->stream));
      g->dirty[i] = 0;
    }
  g->cur = 0;
  am::launch_init(g->g, g->occ, g->srcmask, g->val[0], cell_bits, ctx->stream);
  CKL();
  g->plain_active = 0;
  g->computed = g->layers_used = 0;
  g->have_map = 1;
  return AM_OK;
}

am_status am_propagate(am_ctx* ctx, am_grid* g, uint32_t layers, uint32_t auto_cap, uint32_t mode,
                       am_prop_result* res) {
  if (!ctx || !g) return AM_EINVAL;
  const bool autom = layers == 0;
  const uint32_t target = autom ? auto_cap : layers;
  if (target == 0) return fail(ctx, AM_EINVAL, "auto_cap must be >= 1");
  if (target > am::kMaxLayers) return fail(ctx, AM_EINVAL, "layer count %u exceeds kMaxLayers", target);
  if (mode != AM_MODE_BATCHED && mode != AM_MODE_ITERATIVE) return fail(ctx, AM_EINVAL, "bad mode");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  // 16-bit cells unless the run can never fit (fixed L beyond the 16-bit range)
  const int start_bits = (!autom && (uint64_t)target + 1 > am::kMax16Activity) ? 32 : 16;
  am_status st = reset_map(ctx, g, start_bits);
  if (st) return st;

  am_prop_result r{};
  const bool timing = (ctx->flags & AM_CTX_TIMING) != 0;
  size_t timer_used = 0;
  std::deque<PendingBlock> pend;
  uint32_t l = 0;             // layers applied so far
  uint32_t lprime = 0;        // first layer without new cells (0 = not found)
  uint64_t nblock = 0;
  const int K = am::kK;

  auto drain_one = [&]() -> am_status {
    PendingBlock b = pend.front();
    pend.pop_front();
    CK(cudaEventSynchronize(g->flag_ev[b.slot]));
    if (!lprime) {
      uint32_t t = block_termination(b, g->h_flags[b.slot]);
      if (t) lprime = t;
    }
    return AM_OK;
  };

  while (l < target && !lprime) {
    uint32_t kk;
    bool blocked;
    if (mode == AM_MODE_BATCHED && target - l >= (uint32_t)K) {
      kk = K;
      blocked = true;
    } else {
      kk = 1;
      blocked = false;
    }
    if (g->cell_bits == 16 && (uint64_t)l + kk + 1 > am::kMax16Activity) {
      while (!pend.empty() && !lprime) {
        st = drain_one();
        if (st) return st;
      }
      pend.clear();
      if (lprime) break;
      st = promote(ctx, g);
      if (st) return st;
    }
    const int slot = (int)(nblock % kFlagSlots);
    uint32_t* flag = g->d_flags + slot;
    if (autom) CK(cudaMemsetAsync(flag, 0xFF, sizeof(uint32_t), s));
    void* in = g->val[g->cur];
    void* outp = g->val[g->cur ^ 1];
    if (blocked) {
      if (timing) {
        if (timer_used == ctx->timers.size()) {
          Timer t;
          CK(cudaEventCreate(&t.a));
          CK(cudaEventCreate(&t.b));
          ctx->timers.push_back(t);
        }
        CK(cudaEventRecord(ctx->timers[timer_used].a, s));
      }
      am::launch_block(g->g, g->cell_bits, in, outp, g->srcmask, g->rowsrc, flag, s);
      CKL();
      if (timing) CK(cudaEventRecord(ctx->timers[timer_used++].b, s));
      ++r.block_launches;
    } else {
      am::launch_layer(g->g, g->cell_bits, in, outp, g->srcmask, flag, s);
      CKL();
      ++r.layer_launches;
    }
    g->cur ^= 1;
    if (autom) {
      CK(cudaMemcpyAsync(g->h_flags + slot, flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
      CK(cudaEventRecord(g->flag_ev[slot], s));
      pend.push_back(PendingBlock{slot, l, kk, g->cell_bits});
    }
    l += kk;
    ++nblock;
    if (mode == AM_MODE_ITERATIVE) CK(cudaStreamSynchronize(s));  // per-layer call boundary
    while ((int)pend.size() > kLag) {
      st = drain_one();
      if (st) return st;
    }
  }
  while (!pend.empty()) {
    st = drain_one();
    if (st) return st;
  }
  g->computed = l;
  uint32_t used = l, cause = AM_STOP_FIXED;
  if (autom) {
    uint32_t* zflag = g->d_flags + (int)(nblock % kFlagSlots);
    CK(cudaMemsetAsync(zflag, 0, sizeof(uint32_t), s));
    am::launch_zero_check(g->g, g->cell_bits, g->val[g->cur], zflag, s);
    CKL();
    uint32_t any_zero = 0;
    CK(cudaMemcpyAsync(&any_zero, zflag, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (lprime) {
      if (!any_zero) {
        used = lprime > 1 ? lprime - 1 : 1;
        cause = AM_STOP_FILLED;
      } else {
        used = lprime;
        cause = AM_STOP_STALLED;
      }
    } else {
      used = target;
      cause = any_zero ? AM_STOP_CAP : AM_STOP_FILLED;
    }
  } else {
    if (mode == AM_MODE_BATCHED) CK(cudaStreamSynchronize(s));
  }
  g->layers_used = used;
  if (timing) {
    CK(cudaStreamSynchronize(s));
    double ms = 0;
    for (size_t i = 0; i < timer_used; ++i) {
      float f = 0;
      CK(cudaEventElapsedTime(&f, ctx->timers[i].a, ctx->timers[i].b));
      ms += f;
    }
    r.stencil_ms = ms;
  }
  r.layers_used = used;
  r.cause = cause;
  r.layers_computed = l;
  r.cell_bits = g->cell_bits;
  if (res) *res = r;
  return AM_OK;
}

static am_status download_impl(am_ctx* ctx, am_grid* g, uint32_t* dst, bool dst_device) {
  if (!ctx || !g || !dst) return AM_EINVAL;
  if (!g->have_map) return fail(ctx, AM_EINVAL, "no activity map: call am_propagate first");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const size_t W = g->g.W, H = g->g.H;
  if (g->plain_active) {
    CK(cudaMemcpyAsync(dst, g->plain, W * H * 4, dst_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       s));
    CK(cudaStreamSynchronize(s));
    return AM_OK;
  }
  const uint32_t rollback = g->computed - g->layers_used;
  if (dst_device) {
    am::launch_decode(g->g, g->cell_bits, g->val[g->cur], rollback, 0, (uint32_t)H, dst, s);
    CKL();
    CK(cudaStreamSynchronize(s));
    return AM_OK;
  }
  // decode into the idle ping-pong buffer in row chunks, copy out chunk by chunk
  uint32_t* stage = (uint32_t*)g->val[g->cur ^ 1];
  g->dirty[g->cur ^ 1] = 1;
  const size_t stage_bytes = (size_t)g->g.rows * g->g.pitch * (g->cell_bits / 8);
  size_t rows_per = stage_bytes / (W * 4 * 2);
  if (rows_per < 1) rows_per = 1;
  uint32_t* bufs[2] = {stage, stage + rows_per * W};
  int k = 0;
  for (size_t r0 = 0; r0 < H; r0 += rows_per, k ^= 1) {
    const size_t r1 = std::min(H, r0 + rows_per);
    am::launch_decode(g->g, g->cell_bits, g->val[g->cur], rollback, (uint32_t)r0, (uint32_t)r1, bufs[k], s);
    CKL();
    CK(cudaMemcpyAsync(dst + r0 * W, bufs[k], (r1 - r0) * W * 4, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  return AM_OK;
}

am_status am_activity_download(am_ctx* ctx, am_grid* g, uint32_t* dense) {
  return download_impl(ctx, g, dense, false);
}

am_status am_activity_download_device(am_ctx* ctx, am_grid* g, uint32_t* dense) {
  return download_impl(ctx, g, dense, true);
}

am_status am_activity_upload(am_ctx* ctx, am_grid* g, const uint32_t* dense, uint32_t layers_applied) {
  if (!ctx || !g || !dense) return AM_EINVAL;
  CK(cudaSetDevice(ctx->device));
  const size_t n = (size_t)g->g.W * g->g.H;
  if (!g->plain) CK(cudaMalloc(&g->plain, n * 4));
  CK(cudaMemcpyAsync(g->plain, dense, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  g->plain_active = 1;
  g->plain_layers = layers_applied;
  g->have_map = 1;
  return AM_OK;
}

// ------------------------------------------------------------------ paths

static am::MapView view_of(am_grid* g) {
  am::MapView m{};
  m.g = g->g;
  if (g->plain_active) {
    m.val = g->plain;
    m.srcmask = g->srcmask_dense;
    m.cell_bits = 0;
    m.occ = g->occ;
    m.layers = g->plain_layers;
  } else {
    m.val = g->val[g->cur];
    m.srcmask = g->srcmask;
    m.cell_bits = g->cell_bits;
    m.occ = g->occ;
    m.layers = g->computed;  // point counts are invariant under the rollback
  }
  return m;
}

static am_status ensure_targets(am_ctx* ctx, am_grid* g, uint64_t n) {
  if (n <= g->tgt_cap) return AM_OK;
  cudaFree(g->d_tgt);
  cudaFree(g->d_counts);
  cudaFree(g->d_offsets);
  cudaFree(g->d_status);
  g->d_tgt = nullptr;
  g->d_counts = g->d_offsets = nullptr;
  g->d_status = nullptr;
  g->tgt_cap = 0;
  CK(cudaMalloc(&g->d_tgt, n * 2 * sizeof(uint32_t)));
  CK(cudaMalloc(&g->d_counts, n * sizeof(uint64_t)));
  CK(cudaMalloc(&g->d_offsets, (n + 1) * sizeof(uint64_t)));
  CK(cudaMalloc(&g->d_status, n * sizeof(int32_t)));
  g->tgt_cap = n;
  return AM_OK;
}

am_status am_path_counts(am_ctx* ctx, am_grid* g, const uint32_t* tgt, uint64_t n, uint32_t method, uint64_t seed,
                         uint64_t* offsets, int32_t* status) {
  if (!ctx || !g || (n && (!tgt || !status)) || !offsets) return AM_EINVAL;
  if (!g->have_map) return fail(ctx, AM_EINVAL, "no activity map");
  if (method > 1) return fail(ctx, AM_EINVAL, "bad method");
  CK(cudaSetDevice(ctx->device));
  offsets[0] = 0;
  if (!n) return AM_OK;
  am_status st = ensure_targets(ctx, g, n);
  if (st) return st;
  cudaStream_t s = ctx->stream;
  CK(cudaMemcpyAsync(g->d_tgt, tgt, n * 8, cudaMemcpyHostToDevice, s));
  am::launch_path_counts(view_of(g), g->d_tgt, n, (int)method, seed, g->d_counts, g->d_status, s);
  CKL();
  am::launch_scan(g->d_counts, n, g->d_offsets, s);
  CKL();
  CK(cudaMemcpyAsync(offsets, g->d_offsets, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(status, g->d_status, n * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return AM_OK;
}

// Host straighten (reconstruct.hpp:54-58, pin P4, strict rule) -- only needed
// for caller-uploaded maps; see the header.
static uint64_t straighten_strict(uint32_t* p, uint64_t n, const std::vector<uint8_t>& occ, uint32_t W) {
  if (n < 3) return n;
  uint64_t m = 0;
  for (uint64_t i = 0; i < n; ++i) {
    p[2 * m] = p[2 * i];
    p[2 * m + 1] = p[2 * i + 1];
    ++m;
    while (m >= 3) {
      const int64_t ar = p[2 * (m - 3)], ac = p[2 * (m - 3) + 1], br = p[2 * (m - 1)], bc = p[2 * (m - 1) + 1];
      const int64_t dr = ar - br, dc = ac - bc;
      if (dr * dr + dc * dc != 2) break;
      if (occ[(size_t)ar * W + bc] && occ[(size_t)br * W + ac]) break;
      p[2 * (m - 2)] = p[2 * (m - 1)];
      p[2 * (m - 2) + 1] = p[2 * (m - 1) + 1];
      --m;
    }
  }
  return m;
}

am_status am_trace_paths(am_ctx* ctx, am_grid* g, const uint32_t* tgt, uint64_t n, uint32_t method, uint64_t seed,
                         const uint64_t* offsets, uint32_t* pts, uint64_t cap, int32_t* status) {
  if (!ctx || !g || !offsets || (n && (!tgt || !status))) return AM_EINVAL;
  if (!g->have_map) return fail(ctx, AM_EINVAL, "no activity map");
  if (method > 1) return fail(ctx, AM_EINVAL, "bad method");
  if (!n) return AM_OK;
  const uint64_t total = offsets[n];
  if (total > cap || (total && !pts)) return fail(ctx, AM_EINVAL, "point buffer too small (%llu < %llu)",
                                                  (unsigned long long)cap, (unsigned long long)total);
  CK(cudaSetDevice(ctx->device));
  am_status st = ensure_targets(ctx, g, n);
  if (st) return st;
  cudaStream_t s = ctx->stream;
  if (total > g->pts_cap) {
    cudaFree(g->d_pts);
    g->d_pts = nullptr;
    g->pts_cap = 0;
    CK(cudaMalloc(&g->d_pts, total * 8));
    g->pts_cap = total;
  }
  CK(cudaMemcpyAsync(g->d_tgt, tgt, n * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(g->d_offsets, offsets, (n + 1) * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(g->d_status, status, n * 4, cudaMemcpyHostToDevice, s));
  am::launch_trace(view_of(g), g->d_tgt, n, (int)method, seed, g->d_offsets, g->d_pts, g->d_status, s);
  CKL();
  if (total) CK(cudaMemcpyAsync(pts, g->d_pts, total * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(status, g->d_status, n * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (g->plain_active && method == AM_METHOD_EUCLIDEAN) {
    std::vector<uint8_t> occ((size_t)g->g.W * g->g.H);
    CK(cudaMemcpy(occ.data(), g->occ, occ.size(), cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < n; ++i) {
      if (status[i] != AM_OK) continue;
      uint32_t* p = pts + 2 * offsets[i];
      const uint64_t len = offsets[i + 1] - offsets[i];
      const uint64_t m = straighten_strict(p, len, occ, g->g.W);
      for (uint64_t k = m; k < len; ++k) p[2 * k] = p[2 * k + 1] = 0xFFFFFFFFu;  // removed points
    }
  }
  return AM_OK;
}

am_status am_trace_paths_device(am_ctx* ctx, am_grid* g, const uint32_t* d_tgt, uint64_t n, uint32_t method,
                                uint64_t seed, uint64_t* d_offsets, uint32_t* d_pts, uint64_t cap,
                                int32_t* d_status) {
  if (!ctx || !g || !d_offsets || (n && (!d_tgt || !d_status))) return AM_EINVAL;
  if (!g->have_map) return fail(ctx, AM_EINVAL, "no activity map");
  if (g->plain_active) return fail(ctx, AM_EINVAL, "device path tracing needs a propagated map");
  if (method > 1) return fail(ctx, AM_EINVAL, "bad method");
  (void)cap;
  if (!n) return AM_OK;
  CK(cudaSetDevice(ctx->device));
  am_status st = ensure_targets(ctx, g, n);
  if (st) return st;
  cudaStream_t s = ctx->stream;
  am::MapView m = view_of(g);
  am::launch_path_counts(m, d_tgt, n, (int)method, seed, g->d_counts, d_status, s);
  CKL();
  am::launch_scan(g->d_counts, n, d_offsets, s);
  CKL();
  am::launch_trace(m, d_tgt, n, (int)method, seed, d_offsets, d_pts, d_status, s);
  CKL();
  return AM_OK;
}

// -------------------------------------------------------- single-shot ops

am_status am_propagate_layer(am_ctx* ctx, uint32_t W, uint32_t H, const uint8_t* occ, const uint32_t* src,
                             uint64_t n_src, const uint32_t* in, uint32_t* out) {
  if (!ctx || !occ || !in || !out || (n_src && !src)) return AM_EINVAL;
  if (!dims_ok(W, H)) return fail(ctx, AM_EINVAL, "grid dimensions %ux%u outside 1..65535", W, H);
  if (!n_src) return fail(ctx, AM_EINVAL, "SourceSet must be nonempty");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const size_t n = (size_t)W * H;
  uint8_t *d_occ = nullptr, *d_sm = nullptr;
  uint32_t *d_in = nullptr, *d_out = nullptr, *d_src = nullptr;
  int* d_err = nullptr;
  int h_err = 0;
  am_status st = AM_OK;
  cudaError_t e = cudaMalloc(&d_occ, n);
  if (!e) e = cudaMalloc(&d_sm, n);
  if (!e) e = cudaMalloc(&d_in, n * 4);
  if (!e) e = cudaMalloc(&d_out, n * 4);
  if (!e) e = cudaMalloc(&d_src, n_src * 8);
  if (!e) e = cudaMalloc(&d_err, 4);
  if (!e) e = cudaMemsetAsync(d_sm, 0, n, s);
  if (!e) e = cudaMemsetAsync(d_err, 0, 4, s);
  if (!e) e = cudaMemcpyAsync(d_occ, occ, n, cudaMemcpyHostToDevice, s);
  if (!e) e = cudaMemcpyAsync(d_in, in, n * 4, cudaMemcpyHostToDevice, s);
  if (!e) e = cudaMemcpyAsync(d_src, src, n_src * 8, cudaMemcpyHostToDevice, s);
  if (!e) {
    am::launch_srcmask_dense(W, H, d_src, n_src, d_sm, d_occ, d_err, s);
    am::launch_plain_layer(W, H, d_occ, d_sm, d_in, d_out, s);
    ctx->launches += 2;
    e = cudaMemcpyAsync(out, d_out, n * 4, cudaMemcpyDeviceToHost, s);
  }
  if (!e) e = cudaMemcpyAsync(&h_err, d_err, 4, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  if (e) st = fail(ctx, e == cudaErrorMemoryAllocation ? AM_EOOM : AM_ECUDA, "%s", cudaGetErrorString(e));
  else if (h_err) st = fail(ctx, AM_EINVAL, "SourceSet: a source is out of bounds or on an obstacle");
  (void)cudaGetLastError();
  cudaFree(d_occ);
  cudaFree(d_sm);
  cudaFree(d_in);
  cudaFree(d_out);
  cudaFree(d_src);
  cudaFree(d_err);
  return st;
}

am_status am_propagate_reference(am_ctx* ctx, uint32_t W, uint32_t H, const uint8_t* occ, const uint32_t* src,
                                 uint64_t n_src, uint32_t layers, uint32_t* out) {
  if (!ctx || !occ || !out || (n_src && !src)) return AM_EINVAL;
  if (!dims_ok(W, H)) return fail(ctx, AM_EINVAL, "grid dimensions %ux%u outside 1..65535", W, H);
  if (!n_src) return fail(ctx, AM_EINVAL, "SourceSet must be nonempty");
  if (layers == 0 || layers > am::kMaxLayers) return fail(ctx, AM_EINVAL, "layer count %u out of range", layers);
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const size_t n = (size_t)W * H;
  uint8_t *d_occ = nullptr, *d_sm = nullptr;
  int32_t *a = nullptr, *b = nullptr;
  uint32_t* d_src = nullptr;
  int* d_err = nullptr;
  int h_err = 0;
  am_status st = AM_OK;
  cudaError_t e = cudaMalloc(&d_occ, n);
  if (!e) e = cudaMalloc(&d_sm, n);
  if (!e) e = cudaMalloc(&a, n * 4);
  if (!e) e = cudaMalloc(&b, n * 4);
  if (!e) e = cudaMalloc(&d_src, n_src * 8);
  if (!e) e = cudaMalloc(&d_err, 4);
  if (!e) e = cudaMemsetAsync(d_sm, 0, n, s);
  if (!e) e = cudaMemsetAsync(d_err, 0, 4, s);
  if (!e) e = cudaMemcpyAsync(d_occ, occ, n, cudaMemcpyHostToDevice, s);
  if (!e) e = cudaMemcpyAsync(d_src, src, n_src * 8, cudaMemcpyHostToDevice, s);
  if (!e) {
    am::launch_srcmask_dense(W, H, d_src, n_src, d_sm, d_occ, d_err, s);
    ++ctx->launches;
    // A_0 = I_s: the dense source mask widened to int32
    std::vector<int32_t> a0(n, 0);
    for (uint64_t k = 0; k < n_src; ++k) {
      const uint32_t r = src[2 * k], c = src[2 * k + 1];
      if (r < H && c < W) a0[(size_t)r * W + c] = 1;
    }
    e = cudaMemcpyAsync(a, a0.data(), n * 4, cudaMemcpyHostToDevice, s);
    if (!e) e = cudaStreamSynchronize(s);
    for (uint32_t l = 0; !e && l < layers; ++l) {
      am::launch_sentinel_layer(W, H, d_occ, d_sm, a, b, s);
      ++ctx->launches;
      std::swap(a, b);
    }
    if (!e) e = cudaMemcpyAsync(out, a, n * 4, cudaMemcpyDeviceToHost, s);
  }
  if (!e) e = cudaMemcpyAsync(&h_err, d_err, 4, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  if (e) st = fail(ctx, e == cudaErrorMemoryAllocation ? AM_EOOM : AM_ECUDA, "%s", cudaGetErrorString(e));
  else if (h_err) st = fail(ctx, AM_EINVAL, "SourceSet: a source is out of bounds or on an obstacle");
  (void)cudaGetLastError();
  cudaFree(d_occ);
  cudaFree(d_sm);
  cudaFree(a);
  cudaFree(b);
  cudaFree(d_src);
  cudaFree(d_err);
  return st;
}

}  // extern "C"
