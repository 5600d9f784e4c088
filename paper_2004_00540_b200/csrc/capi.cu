// capi.cu -- host orchestration behind include/actmap_b200.h.
//
// propagate_auto on the device (propagate.hpp:57-61, pin P3): temporally
// blocked launches of kK layers each, with the fixed-point signal of block b
// read back (a device-mapped pinned slot the kernels write, or a copy +
// event for slab groups) only blocks after b+1 is queued, so the GPU never
// idles on the host.  Coverage growth is monotone
// (new cells at layer l imply new cells at layer l-1), so one number per
// block -- the smallest activity among covered cells -- locates the first
// layer without new cells exactly; blocks launched past it are undone by
// subtracting the overshoot from every covered cell (exact: a covered cell
// gains exactly +1 per layer once coverage is fixed).
//
// The same driver runs a stack of row slabs in lock step (multigpu.cu):
// halos are refreshed through a Transport before every launch and the
// per-block number is reduced across slabs.
#include <algorithm>
#include <cstring>
#include <deque>
#include <new>

#include "am_host.hpp"

using am::Geo;

namespace am {
void comm_destroy(Comm* c);
Transport* make_nccl_transport(am_ctx* ctx, am_grid* g);
}  // namespace am
static void flag_set_free(am::FlagSet* f);

extern "C" {

am_status am_ctx_create(const am_ctx_opts* opts, am_ctx** out) {
  if (!out) return AM_EINVAL;
  *out = nullptr;
  am_ctx* ctx = new (std::nothrow) am_ctx();
  if (!ctx) return AM_EOOM;
  ctx->device = opts ? opts->device : 0;
  ctx->flags = opts ? opts->flags : 0;
  cudaError_t e = cudaSetDevice(ctx->device);
  // the context stream at the highest priority: work beside it (the field encoding on the map stream)
  // gives up SM slots to the path walkers as its short CTAs retire
  int prio_least = 0, prio_greatest = 0;
  if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&ctx->stream, cudaStreamNonBlocking, prio_greatest);
  if (e == cudaSuccess) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = ctx->device;
    e = cudaMemPoolCreate(&ctx->pool, &props);
    uint64_t keep = UINT64_MAX;  // never shrink at synchronisation points; am_ctx_trim does
    if (e == cudaSuccess) e = cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  if (e != cudaSuccess) {
    if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
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
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  am::comm_destroy(ctx->comm);
  for (auto& t : ctx->timers) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (auto* f : ctx->flag_sets) flag_set_free(f);
  am::host_pool_destroy(ctx->hpool);
  if (ctx->h_pack) cudaFreeHost(ctx->h_pack);
  am::dfree(ctx, ctx->d_pack);
  for (auto& e : ctx->copy_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->map_stream) {
    cudaStreamSynchronize(ctx->map_stream);
    cudaStreamDestroy(ctx->map_stream);
  }
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->pool) cudaMemPoolDestroy(ctx->pool);  // deferred by the driver while grids still hold memory
  delete ctx;
}

const char* am_last_error(const am_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

am_status am_ctx_stats(const am_ctx* ctx, am_stats* out) {
  if (!ctx || !out) return AM_EINVAL;
  out->kernel_launches = ctx->launches;
  uint64_t v = 0;
  out->pool_reserved = cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrReservedMemCurrent, &v) ? 0 : v;
  v = 0;
  out->pool_used = cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrUsedMemCurrent, &v) ? 0 : v;
  out->h2d_bytes = ctx->h2d_bytes;
  return AM_OK;
}

am_status am_ctx_trim(am_ctx* ctx) {
  if (!ctx) return AM_EINVAL;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaMemPoolTrimTo(ctx->pool, 0));
  return AM_OK;
}

am_status am_host_alloc(am_ctx* ctx, size_t bytes, void** out) {
  if (!ctx || !out) return AM_EINVAL;
  *out = nullptr;
  CK(cudaSetDevice(ctx->device));
  CK(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocMapped));
  return AM_OK;
}

am_status am_host_free(am_ctx* ctx, void* p) {
  if (!ctx) return AM_EINVAL;
  if (p) CK(cudaFreeHost(p));
  return AM_OK;
}

am_status am_ctx_get_stream(const am_ctx* ctx, void** stream) {
  if (!ctx || !stream) return AM_EINVAL;
  *stream = (void*)ctx->stream;
  return AM_OK;
}

am_status am_ctx_synchronize(am_ctx* ctx) {
  if (!ctx) return AM_EINVAL;
  if (ctx->map_stream) CK(cudaStreamSynchronize(ctx->map_stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return AM_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ grids

static void flag_set_free(am::FlagSet* f) {
  if (f->h) cudaFreeHost(f->h);
  for (auto& e : f->ev)
    if (e) cudaEventDestroy(e);
  delete f;
}

static cudaError_t take_flag_set(am_ctx* ctx, am::FlagSet** out) {
  if (!ctx->flag_sets.empty()) {
    *out = ctx->flag_sets.back();
    ctx->flag_sets.pop_back();
    return cudaSuccess;
  }
  auto* f = new (std::nothrow) am::FlagSet();
  if (!f) return cudaErrorMemoryAllocation;
  // slots, then each bit-plane block's items by slot and the k_bits_run record (drive_bits)
  cudaError_t e = cudaHostAlloc(&f->h, (2 * am::kFlagSlots + 8) * sizeof(uint32_t), cudaHostAllocMapped);
  if (!e) e = cudaHostGetDevicePointer((void**)&f->hdev, f->h, 0);
  for (int i = 0; !e && i < am::kFlagSlots; ++i) e = cudaEventCreateWithFlags(&f->ev[i], cudaEventDisableTiming);
  if (e) {
    flag_set_free(f);
    return e;
  }
  *out = f;
  return cudaSuccess;
}

static void grid_free(am_ctx* ctx, am_grid* g) {
  if (!g) return;
  for (int i = 0; i < 2; ++i) am::dfree(ctx, g->val[i]);
  am::dfree(ctx, g->srcmask);
  am::dfree(ctx, g->rowsrc);
  am::dfree(ctx, g->occ);
  am::dfree(ctx, g->src_rc);
  am::dfree(ctx, g->srcmask_dense);
  am::dfree(ctx, g->d_flags);
  if (g->fs) ctx->flag_sets.push_back(g->fs);
  am::dfree(ctx, g->plain);
  am::dfree(ctx, g->d_tgt);
  am::dfree(ctx, g->d_counts);
  am::dfree(ctx, g->d_sched);
  if (g->map_ev) cudaEventDestroy(g->map_ev);
  am::dfree(ctx, g->d_offsets);
  am::dfree(ctx, g->d_status);
  am::dfree(ctx, g->d_pts);
  am::dfree(ctx, g->t_state);
  am::dfree(ctx, g->t_sched);
  am::dfree(ctx, g->t_list[0]);
  am::dfree(ctx, g->t_list[1]);
  am::dfree(ctx, g->t_count);
  am::dfree(ctx, g->t_bnd);
  am::dfree(ctx, g->t_processed);
  am::dfree(ctx, g->t_src);
  if (g->bits) {
    am::dfree(ctx, g->bits->bk.P);
    am::dfree(ctx, g->bits->bk.state);
    am::dfree(ctx, g->bits->bk.sched);
    am::dfree(ctx, g->bits->bk.list[0]);
    am::dfree(ctx, g->bits->bk.list[1]);
    am::dfree(ctx, g->bits->bk.count);
    am::dfree(ctx, g->bits->bk.stat);
    am::dfree(ctx, g->bits->own_t);
    delete g->bits;
  }
  am::peer_destroy(g->peer);
  delete g;
}

namespace am {

// Rows [row0, row1) of an H_total-row grid.  occ_full / src use global
// coordinates (host or device per device_ptrs).  For slabs, sources inside
// the K-row halo bands are marked too (their +1 matters for the recomputed
// halo rows); the halo values themselves arrive through the transport.
am_status grid_create_rows(am_ctx* ctx, uint32_t W, uint32_t H_total, uint32_t row0, uint32_t row1,
                           const uint8_t* occ_full, const uint32_t* src, uint64_t n_src, bool device_ptrs,
                           bool slab, am_grid** out) {
  if (!ctx || !out) return AM_EINVAL;
  *out = nullptr;
  if (!dims_ok(W, H_total)) return fail(ctx, AM_EINVAL, "grid dimensions %ux%u outside 1..65535", W, H_total);
  if (n_src == 0) return fail(ctx, AM_EINVAL, "SourceSet must be nonempty");
  if (!occ_full || !src) return fail(ctx, AM_EINVAL, "null occupancy or sources");
  if (row1 <= row0 || row1 > H_total) return fail(ctx, AM_EINVAL, "bad slab rows [%u, %u)", row0, row1);
  if (slab && row1 - row0 < (uint32_t)kK) return fail(ctx, AM_EINVAL, "slab of %u rows < halo depth %d", row1 - row0, kK);
  CK(cudaSetDevice(ctx->device));
  am_grid* g = new (std::nothrow) am_grid();
  if (!g) return AM_EOOM;
  const uint32_t H = row1 - row0;
  g->g = make_geo(W, H, ctx->warp_slots);
  g->slab = slab ? 1 : 0;
  g->total_h = H_total;
  g->row0 = row0;
  const size_t cells = (size_t)g->g.rows * g->g.pitch;
  const size_t dense = (size_t)W * H;
  cudaStream_t s = ctx->stream;
  uint32_t* d_src = nullptr;
  int* d_err = nullptr;
  am_status st = AM_OK;
  int h_err = 0;
  cudaError_t e = am::dmalloc(ctx, &g->val[0], cells * 2);
  if (!e) e = am::dmalloc(ctx, &g->val[1], cells * 2);
  if (!e) e = am::dmalloc(ctx, &g->srcmask, cells);
  if (!e) e = am::dmalloc(ctx, &g->rowsrc, g->g.rowsrc_bytes());
  if (!e) e = am::dmalloc(ctx, &g->occ, dense);
  if (!e) e = am::dmalloc(ctx, &g->srcmask_dense, dense);
  if (!e) e = am::dmalloc(ctx, &g->d_flags, kFlagWords * sizeof(uint32_t));
  if (!e) e = take_flag_set(ctx, &g->fs);
  {  // active-tile skipping state
    const size_t nt = g->g.ntiles();
    if (!e) e = am::dmalloc(ctx, &g->t_state, nt * 8);
    if (!e) e = am::dmalloc(ctx, &g->t_sched, nt * 4);
    if (!e) e = am::dmalloc(ctx, &g->t_list[0], nt * 4);
    if (!e) e = am::dmalloc(ctx, &g->t_list[1], nt * 4);
    if (!e) e = am::dmalloc(ctx, &g->t_count, 6 * 4);
    if (slab && !e) e = am::dmalloc(ctx, &g->t_bnd, (size_t)2 * kK * g->g.pitch * 4);  // room for 32-bit cells
    if (slab && !e) e = cudaMemsetAsync(g->t_bnd, 0, (size_t)2 * kK * g->g.pitch * 4, s);
    if (!e) e = am::dmalloc(ctx, &g->t_processed, 8);
    if (!e) e = am::dmalloc(ctx, &g->t_src, nt);
  }
  if (!e) e = cudaMemsetAsync(g->val[0], 0, cells * 2, s);
  if (!e) e = cudaMemsetAsync(g->val[1], 0, cells * 2, s);
  if (!e) e = cudaMemsetAsync(g->srcmask, 0, cells, s);
  if (!e) e = cudaMemsetAsync(g->rowsrc, 0, g->g.rowsrc_bytes(), s);
  if (!e) e = cudaMemsetAsync(g->d_flags, 0xFF, kFlagSlots * sizeof(uint32_t), s);  // armed slots
  if (!e) e = cudaMemsetAsync(g->d_flags + kFlagSlots, 0, sizeof(uint32_t), s);     // arrival counter
  if (!e) e = cudaMemsetAsync(g->d_flags + kFlagRecvUp, 0xFF, 2 * kFlagSlots * sizeof(uint32_t), s);  // no neighbour
  if (!e) e = cudaMemsetAsync(g->srcmask_dense, 0, dense, s);
  // host occupancy of a large grid: packed to bits by host workers on the way (upload.cu, 8x fewer PCIe
  // bytes); small grids and device pointers: a plain copy
  static const bool pack_off = [] {
    const char* v = getenv("AM_PACKED_UPLOAD");
    return v && v[0] == '0';
  }();
  const bool packed = !e && !device_ptrs && !pack_off && dense >= ((size_t)1 << 20);
  if (packed) {
    if ((st = upload_occupancy_packed(ctx, occ_full + (size_t)row0 * W, W, H, g->occ))) {
      grid_free(ctx, g);
      return st;
    }
  } else if (!e) {
    e = cudaMemcpyAsync(g->occ, occ_full + (size_t)row0 * W, dense,
                        device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s);
    if (!device_ptrs) ctx->h2d_bytes += dense;
  }
  if (!e) e = am::dmalloc(ctx, &d_src, n_src * 2 * sizeof(uint32_t));
  if (!e) e = am::dmalloc(ctx, &d_err, sizeof(int));
  if (!e) e = cudaMemsetAsync(d_err, 0, sizeof(int), s);
  if (!e)
    e = cudaMemcpyAsync(d_src, src, n_src * 2 * sizeof(uint32_t),
                        device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s);
  if (!e && !device_ptrs) ctx->h2d_bytes += n_src * 2 * sizeof(uint32_t);
  if (!e) {
    launch_srcmask_rows(g->g, H_total, row0, d_src, n_src, g->srcmask_dense, g->occ, g->srcmask, g->rowsrc, d_err,
                        s);
    launch_tile_src(g->g, g->rowsrc, g->t_src, s);
    ctx->launches += 2;
    e = cudaPeekAtLastError();
  }
  if (!e) e = cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  g->src_rc = d_src;  // kept: the sources of every re-initialisation (freed with the grid)
  g->n_src = n_src;
  am::dfree(ctx, d_err);
  if (e) {
    (void)cudaGetLastError();
    st = fail(ctx, e == cudaErrorMemoryAllocation ? AM_EOOM : AM_ECUDA, "grid create: %s", cudaGetErrorString(e));
  } else if (h_err) {
    st = fail(ctx, AM_EINVAL, "SourceSet: a source is out of bounds or on an obstacle (grid.hpp:78)");
  }
  // single grids: the free plane of the bit-plane engine is part of the grid's device form (built once)
  if (!st && !slab && !(ctx->flags & AM_CTX_DENSE)) st = bits_alloc(ctx, g, packed ? ctx->d_pack : nullptr);
  if (st) {
    grid_free(ctx, g);
    return st;
  }
  *out = g;
  return AM_OK;
}

}  // namespace am

extern "C" {

am_status am_grid_create(am_ctx* ctx, uint32_t W, uint32_t H, const uint8_t* occ, const uint32_t* src,
                         uint64_t n_src, am_grid** out) {
  return am::grid_create_rows(ctx, W, H, 0, H, occ, src, n_src, false, false, out);
}

am_status am_grid_create_device(am_ctx* ctx, uint32_t W, uint32_t H, const uint8_t* occ, const uint32_t* src,
                                uint64_t n_src, am_grid** out) {
  return am::grid_create_rows(ctx, W, H, 0, H, occ, src, n_src, true, false, out);
}

am_status am_grid_clone(am_ctx* ctx, const am_grid* g, am_grid** out) {
  if (!ctx || !g || !out) return AM_EINVAL;
  if (g->slab) return am::fail(ctx, AM_EINVAL, "am_grid_clone: slab grids are not cloneable");
  return am::grid_create_rows(ctx, g->g.W, g->g.H, 0, g->g.H, g->occ, g->src_rc, g->n_src, true, false, out);
}

am_status am_grid_destroy(am_ctx* ctx, am_grid* g) {
  if (!g) return AM_OK;
  if (!ctx) return AM_EINVAL;  // the grid's buffers belong to the context's pool
  cudaSetDevice(ctx->device);
  am::join_map(ctx, g);
  cudaStreamSynchronize(ctx->stream);
  grid_free(ctx, g);
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
  o->tile_rows = am::kTileRows;
  o->tile_cols = am::kTileCols;
  o->tiles = g->t_state ? g->g.ntiles() : 0;
  return AM_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- propagate

namespace am {

struct PendingBlock {
  int slot;
  uint32_t start;  // layers before the block
  uint32_t count;  // layers in the block
  int cell_bits;
  bool polled;     // mapped slot written by the kernel itself: poll, no event
};

// Marks a mapped slot "not yet written" (the kernel's word is never this value:
// minima are < 0x7FFFFFFF or the all-ones "no covered cell").
constexpr uint32_t kSlotPending = 0xFFFFFFFEu;

// First layer without new cells (l'), or 0 if the block still added cells
// in its last layer.  m = min over covered cells of (a-1) at the block end.
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
  CK(am::dmalloc(ctx, &n0, cells * 4));
  cudaError_t e = am::dmalloc(ctx, &n1, cells * 4);
  if (e != cudaSuccess) {
    am::dfree(ctx, n0);
    (void)cudaGetLastError();
    return fail(ctx, AM_EOOM, "32-bit promotion: %s", cudaGetErrorString(e));
  }
  launch_promote(g->g, (const uint16_t*)g->val[g->cur], (uint32_t*)n0, ctx->stream);
  CKL();
  CK(cudaMemsetAsync(n1, 0, cells * 4, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  am::dfree(ctx, g->val[0]);
  am::dfree(ctx, g->val[1]);
  g->val[0] = n0;
  g->val[1] = n1;
  g->cur = 0;
  g->cell_bits = 32;
  g->dirty[0] = g->dirty[1] = 0;
  return AM_OK;
}

// (Re)allocates both fields at cell_bits and clears stale padding.
am_status set_cell_bits(am_ctx* ctx, am_grid* g, int cell_bits) {
  const size_t cells = (size_t)g->g.rows * g->g.pitch;
  if (g->cell_bits != cell_bits) {
    am::dfree(ctx, g->val[0]);
    am::dfree(ctx, g->val[1]);
    g->val[0] = g->val[1] = nullptr;
    const size_t bytes = cells * (cell_bits / 8);
    CK(am::dmalloc(ctx, &g->val[0], bytes));
    CK(am::dmalloc(ctx, &g->val[1], bytes));
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
  return AM_OK;
}

static am_status reset_map(am_ctx* ctx, am_grid* g, int cell_bits) {
  am_status st = set_cell_bits(ctx, g, cell_bits);
  if (st) return st;
  g->cur = 0;
  launch_init(g->g, g->occ, g->val[0], cell_bits, ctx->stream);
  CKL();
  launch_src_init(g->g, g->src_rc, g->n_src, g->row0, g->val[0], cell_bits, ctx->stream);
  CKL();
  g->plain_active = 0;
  g->computed = g->layers_used = 0;
  g->have_map = 1;
  return AM_OK;
}

// Bit-plane propagation of a single grid (bits.cu).  The field is
// written once per cell, relative to lref = min(target, kBitsMaxRef = 16382) layers, so the map
// needs no decode: computed = lref, layers_used = the outcome, rollback = lref - used.
// Auto runs that have not reached their fixed point by lref (beyond the 16-bit
// range) return handoff = true with the field exactly at layer lref; the caller
// continues there with the 16/32-bit tile kernels.

static am_status bits_build_planes(am_ctx* ctx, am_grid* g, const uint32_t* packed) {
  BitState& B = *g->bits;
  cudaStream_t s = ctx->stream;
  CK(cudaMemsetAsync(B.bk.stat, 0, 3 * 8, s));
  if (packed)
    launch_bits_init_packed(B.bg, packed, B.bk, s);
  else
    launch_bits_init(B.bg, g->occ, B.bk, s);
  CKL();
  ++ctx->launches;
  unsigned long long fc = 0;
  CK(cudaMemcpyAsync(&fc, B.bk.stat + 2, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  B.free_cells = fc;
  B.planes_ready = true;
  return AM_OK;
}

am_status join_map(am_ctx* ctx, am_grid* g) {
  if (!g || !g->map_pending) return AM_OK;
  g->map_pending = 0;
  CK(cudaStreamWaitEvent(ctx->stream, g->map_ev, 0));
  return AM_OK;
}

// Allocates the bit-plane state and builds the free plane from the grid's occupancy (occupancy is
// immutable, so this runs once per grid: at creation for single grids, else on first use).
am_status bits_alloc(am_ctx* ctx, am_grid* g, const uint32_t* packed) {
  if (g->bits && g->bits->planes_ready) return AM_OK;
  if (g->bits) return bits_build_planes(ctx, g, packed);
  auto* b = new (std::nothrow) BitState();
  if (!b) return fail(ctx, AM_EOOM, "bit state");
  g->bits = b;
  b->bg = make_bit_geo(g->g.W, g->g.H);
  const size_t pw = b->bg.plane_words(), nt = b->bg.ntiles();
  BitBook& k = b->bk;
  CK(am::dmalloc(ctx, &k.P, pw * 16));
  CK(am::dmalloc(ctx, &k.state, nt * 8));
  CK(am::dmalloc(ctx, &k.sched, nt * 4));
  CK(am::dmalloc(ctx, &k.list[0], nt * 4));
  CK(am::dmalloc(ctx, &k.list[1], nt * 4));
  CK(am::dmalloc(ctx, &k.count, 12 * 4));
  CK(am::dmalloc(ctx, &k.stat, 8 * 8));
  b->ctas = ctx->sms * bits_ctas_per_sm();
  return bits_build_planes(ctx, g, packed);
}

static am_status drive_bits(am_ctx* ctx, am_grid* g, uint32_t target, bool autom, am_prop_result* res,
                            bool* handoff) {
  *handoff = false;
  am_status st = bits_alloc(ctx, g);
  if (st) return st;
  if ((st = set_cell_bits(ctx, g, 16))) return st;
  BitState& B = *g->bits;
  const BitGeo& bg = B.bg;
  const size_t pw = bg.plane_words(), nt = bg.ntiles();
  cudaStream_t s = ctx->stream;
  const uint32_t lref = std::min(target, kBitsMaxRef);
  uint16_t* field = static_cast<uint16_t*>(g->val[0]);
  // time planes (64 B per plane word): the second 16-bit field when it is large enough
  const size_t tbytes = pw * 64, vbytes = (size_t)g->g.rows * g->g.pitch * 2;
  if (tbytes <= vbytes) {
    B.bk.T = static_cast<uint32_t*>(g->val[1]);
    g->dirty[1] = 1;  // holds time planes now, not a clean field
  } else {
    if (!B.own_t) CK(am::dmalloc(ctx, &B.own_t, tbytes));
    B.bk.T = B.own_t;
  }
  CK(cudaMemsetAsync(B.bk.state, 0, nt * 8, s));
  CK(cudaMemsetAsync(B.bk.sched, 0, nt * 4, s));
  CK(cudaMemsetAsync(B.bk.count, 0, 6 * 4, s));
  CK(cudaMemsetAsync(B.bk.count + 6, 0xFF, 3 * 4, s));  // k_bits_run's fixed-point words
  CK(cudaMemsetAsync(B.bk.stat, 0, 2 * 8, s));
  CK(cudaMemsetAsync(B.bk.stat + 3, 0, 5 * 8, s));  // experiment counters (AM_BITS_STATS)
  // the planes are not reset: the cleared states mark every tile's coverage stale (bits.cu)
  launch_bits_sources(bg, g->src_rc, g->n_src, B.bk, s);
  CKL();
  ctx->launches += 2;
  g->cur = 0;
  g->plain_active = 0;
  g->have_map = 1;

  am_prop_result r{};
  const bool timing = (ctx->flags & AM_CTX_TIMING) != 0;
  if (timing) {
    while (ctx->timers.size() < 1) {
      am_ctx::Timer t;
      CK(cudaEventCreate(&t.a));
      CK(cudaEventCreate(&t.b));
      ctx->timers.push_back(t);
    }
    CK(cudaEventRecord(ctx->timers[0].a, s));
  }
  if (autom) CK(cudaMemsetAsync(g->d_flags, 0xFF, kFlagSlots * sizeof(uint32_t), s));
  std::deque<PendingBlock> pend;
  FlagSink unpublished{nullptr, nullptr, nullptr};
  uint32_t l = 0, lprime = 0, blk = 0;
  // Light stretches run in one cluster (k_bits_run) while a block lists at most run_max tiles: entered
  // from the start when the sources fit, later when a drained block (kLagTiles behind) listed few tiles;
  // after a stretch ends on a heavy block, normal launches for at least run_gap blocks (hysteresis).
  // (AM_BITS_RUN=0 disables the stretches, AM_BITS_RUN_MAX overrides run_max; both read per run)
  const char* run_env = getenv("AM_BITS_RUN");
  const char* max_env = getenv("AM_BITS_RUN_MAX");
  const int run_cluster = run_env && run_env[0] == '0' ? 0 : bits_run_cluster();
  const uint32_t run_max = !run_cluster ? 0 : max_env ? (uint32_t)atoi(max_env) : bits_run_warps(run_cluster);
  const uint32_t run_gap = kLagTiles + 8;
  B.bk.hcount = g->fs->hdev + kFlagSlots;
  bool want_run = run_cluster && g->n_src <= run_max;
  uint32_t since_run = run_gap;
  auto drain_one = [&]() -> am_status {
    const PendingBlock b = pend.front();
    pend.pop_front();
    volatile uint32_t* h = g->fs->h + b.slot;
    for (uint64_t spin = 1; *h == kSlotPending; ++spin) {
      if ((spin & 4095) == 0) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess && *h == kSlotPending) return fail(ctx, AM_ECUDA, "flag slot never written");
        if (q != cudaSuccess && q != cudaErrorNotReady) return fail(ctx, AM_ECUDA, "bits: %s", cudaGetErrorString(q));
      }
    }
    if (!lprime) {
      const uint32_t t = block_termination(b, *h);
      if (t) lprime = t;
    }
    if (run_cluster && since_run >= run_gap && g->fs->h[kFlagSlots + b.slot] <= run_max) want_run = true;
    return AM_OK;
  };
  while (l < lref && !lprime) {
    if (want_run && lref - l >= (uint32_t)kBK) {
      want_run = false;
      if (unpublished.host) {
        launch_publish_flag(unpublished, s);
        CKL();
        unpublished = FlagSink{nullptr, nullptr, nullptr};
      }
      // the cluster's fixed-point words start clean: a stretch that ended on a heavy block left the words
      // of its last two blocks set, and the next stretch may start on either
      CK(cudaMemsetAsync(B.bk.count + 6, 0xFF, 3 * 4, s));
      volatile uint32_t* rec = g->fs->h + 2 * kFlagSlots;
      const uint32_t seq = rec[0] + 1;
      launch_bits_run(bg, run_cluster, B.bk, blk, blk + (lref - l) / kBK, run_max, autom, seq,
                      g->fs->hdev + 2 * kFlagSlots, s);
      ++ctx->launches;
      if (cudaError_t e = cudaPeekAtLastError()) return fail(ctx, AM_ECUDA, "k_bits_run: %s", cudaGetErrorString(e));
      while (!pend.empty())  // the blocks before the stretch (an earlier fixed point wins)
        if ((st = drain_one())) return st;
      for (uint64_t spin = 1; rec[0] != seq; ++spin) {
        if ((spin & 4095) == 0) {
          const cudaError_t q = cudaStreamQuery(s);
          if (q == cudaSuccess && rec[0] != seq) return fail(ctx, AM_ECUDA, "run record never written");
          if (q != cudaSuccess && q != cudaErrorNotReady) return fail(ctx, AM_ECUDA, "bits: %s", cudaGetErrorString(q));
        }
      }
      const uint32_t nb = rec[4];
      static const bool run_print = getenv("AM_BITS_RUN_PRINT") != nullptr;
      if (run_print) fprintf(stderr, "bits run: blocks %u..%u, next items %u, end %u\n", blk, rec[1], rec[3], rec[2]);
      blk = rec[1];
      l += nb * kBK;
      r.block_launches += nb;
      if (autom && !lprime && rec[2]) lprime = rec[2];
      since_run = 0;
      continue;
    }
    ++since_run;
    const uint32_t nl = std::min<uint32_t>(kBK, lref - l);
    const int slot = (int)(blk % kFlagSlots);
    FlagSink sink{g->d_flags + slot, g->d_flags + kFlagSlots, nullptr};
    const FlagSink prev = unpublished;
    if (autom) {
      g->fs->h[slot] = kSlotPending;  // consumed kFlagSlots blocks ago (lag < kFlagSlots)
      unpublished = FlagSink{sink.word, sink.done, g->fs->hdev + slot};  // published by the next launch
    }
    launch_bits_tiles(bg, B.ctas, B.bk, blk, nl, sink, prev, s);
    ++ctx->launches;
    if (cudaError_t e = cudaPeekAtLastError()) return fail(ctx, AM_ECUDA, "k_bits_tiles: %s", cudaGetErrorString(e));
    ++r.block_launches;
    if (autom) pend.push_back(PendingBlock{slot, l, nl, 16, true});
    l += nl;
    ++blk;
    while ((int)pend.size() > kLagTiles)
      if ((st = drain_one())) return st;
  }
  if (unpublished.host) {
    launch_publish_flag(unpublished, s);
    CKL();
  }
  if (timing) CK(cudaEventRecord(ctx->timers[0].b, s));
  // the encoded field, once, on the map stream: path counts and walkers read the planes meanwhile
  if (!ctx->map_stream) {
    int least = 0, greatest = 0;
    CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CK(cudaStreamCreateWithPriority(&ctx->map_stream, cudaStreamNonBlocking, least));
  }
  if (!g->map_ev) CK(cudaEventCreateWithFlags(&g->map_ev, cudaEventDisableTiming));
  CK(cudaEventRecord(g->map_ev, s));
  CK(cudaStreamWaitEvent(ctx->map_stream, g->map_ev, 0));
  launch_bits_finalize(bg, g->g, B.bk, lref, field, ctx->sms, ctx->map_stream);
  CKL();
  CK(cudaEventRecord(g->map_ev, ctx->map_stream));
  g->map_pending = 1;
  ctx->launches += 1;
  while (!pend.empty())
    if ((st = drain_one())) return st;
  unsigned long long stat[8] = {};
  CK(cudaMemcpyAsync(stat, B.bk.stat, sizeof stat, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (getenv("AM_BITS_STATS_PRINT"))
    fprintf(stderr, "bits: items %llu, without new cells %llu, own rows fully covered %llu, no new but not full %llu\n",
            stat[0], stat[3], stat[4], stat[5]);
  const bool any_zero = stat[1] < B.free_cells;
  uint32_t used = l, cause = AM_STOP_FIXED;
  if (autom) {
    if (lprime) {
      used = any_zero ? lprime : (lprime > 1 ? lprime - 1 : 1);
      cause = any_zero ? AM_STOP_STALLED : AM_STOP_FILLED;
    } else if (l == target) {
      used = target;
      cause = any_zero ? AM_STOP_CAP : AM_STOP_FILLED;
    } else {
      if ((st = join_map(ctx, g))) return st;
      *handoff = true;  // field at layer lref, beyond the 16-bit range: continue with the tile kernels
      CK(cudaMemsetAsync(g->val[1], 0, vbytes, s));
      g->dirty[1] = 0;
    }
  }
  g->computed = lref;
  g->layers_used = *handoff ? lref : used;
  g->bits_map = *handoff ? 0 : 1;  // the walkers may read the planes (until val[1] is reused)
  if (timing) {
    float f = 0;
    CK(cudaEventElapsedTime(&f, ctx->timers[0].a, ctx->timers[0].b));
    r.stencil_ms = f;
  }
  r.layers_used = used;
  r.cause = cause;
  r.layers_computed = l;
  r.cell_bits = 16;
  r.tiles_processed = stat[0];
  r.tiles_total = (uint64_t)nt * r.block_launches;
  r.cells_executed = stat[0] * (uint64_t)(kBTR * kBTW * 32) * kBK;
  r.engine = AM_ENGINE_BITS;
  r.block_layers = kBK;
  if (res) *res = r;
  return AM_OK;
}

// bit-plane runs: a single grid, batched mode, 16-bit cells, not forced dense (AM_BITS=0 disables)
static bool bits_eligible(std::vector<SlabRef>& slabs, Transport* tr, uint32_t mode, int start_bits) {
  static const bool off = [] {
    const char* e = getenv("AM_BITS");
    return e && e[0] == '0';
  }();
  return !off && slabs.size() == 1 && !tr && !slabs[0].g->slab && mode == AM_MODE_BATCHED && start_bits == 16 &&
         !(slabs[0].ctx->flags & AM_CTX_DENSE);
}

am_status drive_propagation(std::vector<SlabRef>& slabs, Transport* tr, uint32_t layers, uint32_t auto_cap,
                            uint32_t mode, am_prop_result* res) {
  am_ctx* ctx = slabs[0].ctx;
  const bool autom = layers == 0;
  const uint32_t target = autom ? auto_cap : layers;
  if (target == 0) return fail(ctx, AM_EINVAL, "auto_cap must be >= 1");
  if (target > kMaxLayers) return fail(ctx, AM_EINVAL, "layer count %u exceeds kMaxLayers", target);
  if (mode != AM_MODE_BATCHED && mode != AM_MODE_ITERATIVE) return fail(ctx, AM_EINVAL, "bad mode");
  CK(cudaSetDevice(ctx->device));
  for (auto& sr : slabs) sr.g->bits_map = 0;
  // 16-bit cells unless the run can never fit (fixed L beyond the 16-bit range)
  const int start_bits = (!autom && (uint64_t)target + 1 > kMax16Activity) ? 32 : 16;
  am_status st;
  for (auto& sr : slabs)  // a previous run's field encoding still reads the planes this run rewrites
    if ((st = join_map(sr.ctx, sr.g))) return st;
  uint32_t l_init = 0;  // layer the field holds when the loop below starts
  am_prop_result pre{};
  if (bits_eligible(slabs, tr, mode, start_bits)) {
    bool handoff = false;
    if ((st = drive_bits(ctx, slabs[0].g, target, autom, &pre, &handoff))) return st;
    if (!handoff) {
      if (res) *res = pre;
      return AM_OK;
    }
    l_init = slabs[0].g->computed;
  } else {
    for (auto& s : slabs)
      if ((st = reset_map(s.ctx, s.g, start_bits))) return st;
  }

  // exact active-tile skipping in batched mode.  Row slabs
  // must meet at tile-chunk boundaries, so their halo rows lie outside every
  // tile (am_comm_slab_rows aligns them); the halos then carry the
  // neighbours' boundary rows at the block's layer (k_tiles_boundary).
  bool tiles = mode == AM_MODE_BATCHED && !(ctx->flags & AM_CTX_DENSE);
  for (size_t i = 0; i < slabs.size(); ++i) {
    tiles = tiles && slabs[i].g->t_state;
    if (i + 1 < slabs.size()) tiles = tiles && slabs[i].g->g.H % kTileRows == 0;
  }
  // one slab per process: the same rule for every rank of the chain, so all ranks take the same mode
  // (and the same number of exchanges: the transports pair them up in lock step)
  if (tr) tiles = tiles && tr->chain_tiles_ok();
  const bool halos = tiles && (slabs.size() > 1 || tr);  // boundary exchange + halo scan every block
  uint64_t nt = 0;
  for (auto& sr : slabs) nt += tiles ? sr.g->g.ntiles() : 0;
  const int tile_ctas = ctx->sms * kTileCtasPerSm;  // persistent k_block_tiles
  // after dense work: every tile current at at_layer in val[cur], all active next block
  auto tiles_all_active = [&](uint32_t at_layer) -> am_status {
    for (auto& sr : slabs) {
      am_ctx* c = sr.ctx;
      launch_tiles_all(sr.g->g, sr.g->book(), sr.g->t_blk, at_layer, sr.g->cur, c->stream);
      CKL();
    }
    return AM_OK;
  };
  // every tile current at at_layer in val[0] (then cur = 0); zslot >= 0: fused zero check into that flag slot
  auto tiles_finalize = [&](uint32_t at_layer, int zslot = -1) -> am_status {
    for (auto& sr : slabs) {
      am_ctx* c = sr.ctx;
      am_grid* g = sr.g;
      uint32_t* z = zslot >= 0 ? g->d_flags + zslot : nullptr;
      if (z) CK(cudaMemsetAsync(z, 0, sizeof(uint32_t), c->stream));
      launch_tiles_finalize(g->g, g->cell_bits, g->t_state, g->val[0], g->val[1], 0, at_layer, z, c->stream);
      CKL();
      g->cur = 0;
    }
    return AM_OK;
  };
  if (tiles) {  // layer 0 lives in val[cur] (= val[0] after reset_map): state 0 << 1 | 0
    for (auto& sr : slabs) {
      am_ctx* c = sr.ctx;
      am_grid* g = sr.g;
      const size_t n = g->g.ntiles();
      g->t_blk = 0;
      CK(cudaMemsetAsync(g->t_state, 0, n * 8, c->stream));
      CK(cudaMemsetAsync(g->t_sched, 0, n * 4, c->stream));
      CK(cudaMemsetAsync(g->t_processed, 0, 8, c->stream));
      CK(cudaMemsetAsync(g->t_count, 0, 6 * 4, c->stream));
      if (l_init)  // handed over by the bit-plane run: every tile at l_init in val[0], all listed
        launch_tiles_all(g->g, g->book(), 0, l_init, 0, c->stream);
      else
        launch_tiles_init(g->g, g->srcmask, g->book(), c->stream);
      CKL();
    }
  }

  am_prop_result r{};
  const bool timing = (ctx->flags & AM_CTX_TIMING) != 0;
  size_t timer_used = 0;
  // Timing brackets each run of consecutive blocked launches with one event
  // pair (stencil_ms includes the gaps between them, not per-launch events).
  bool run_open = false;
  auto close_run = [&]() -> am_status {
    if (run_open) {
      CK(cudaEventRecord(ctx->timers[timer_used++].b, ctx->stream));
      run_open = false;
    }
    return AM_OK;
  };
  // One grid, no transport: blocked launches publish their fixed-point word
  // straight into the mapped pinned slot (FlagSink), and re-arm the slot.
  const bool mapped = autom && slabs.size() == 1 && !tr;
  bool armed[kFlagSlots];
  for (int i = 0; i < kFlagSlots; ++i) armed[i] = mapped;
  if (mapped) CK(cudaMemsetAsync(slabs[0].g->d_flags, 0xFF, kFlagSlots * sizeof(uint32_t), ctx->stream));
  std::deque<PendingBlock> pend;
  // Mapped tile blocks publish the PREVIOUS block's word (k_block_tiles' prologue); the last one
  // of a run is published by a one-thread kernel before anything else touches the field.
  FlagSink unpublished{nullptr, nullptr, nullptr};
  auto publish_pending = [&]() -> am_status {
    if (unpublished.host) {
      launch_publish_flag(unpublished, ctx->stream);
      CKL();
      unpublished = FlagSink{nullptr, nullptr, nullptr};
    }
    return AM_OK;
  };
  uint32_t l = l_init;  // layers applied so far
  uint32_t lprime = 0;  // first layer without new cells (0 = not found)
  uint64_t nblock = 0;
  const int K = kK;
  std::vector<uint32_t*> words(slabs.size());

  // Row slabs: a block's word is global once span - 1 exchanges have carried it (Transport); until then
  // the block waits here, then its word is copied to the host and it joins `pend`.
  const bool diffuse = autom && tr != nullptr;
  const uint32_t hops = diffuse ? tr->span() - 1 : 0;
  struct Awaiting {
    PendingBlock b;
    uint32_t done;  // exchanges since the block
  };
  std::deque<Awaiting> awaiting;
  auto copy_out = [&](const PendingBlock& b) -> am_status {
    for (auto& sr : slabs) {
      am_ctx* c = sr.ctx;
      if (b.polled) continue;  // the kernel writes the mapped slot itself
      cudaError_t e = cudaMemcpyAsync(sr.g->fs->h + b.slot, sr.g->d_flags + b.slot, sizeof(uint32_t),
                                      cudaMemcpyDeviceToHost, c->stream);
      if (!e) e = cudaEventRecord(sr.g->fs->ev[b.slot], c->stream);
      if (e) return fail(c, AM_ECUDA, "flag copy: %s", cudaGetErrorString(e));
    }
    pend.push_back(b);
    return AM_OK;
  };
  auto after_exchange = [&]() -> am_status {
    for (auto& a : awaiting) ++a.done;
    while (!awaiting.empty() && awaiting.front().done >= hops) {
      if (am_status s2 = copy_out(awaiting.front().b)) return s2;
      awaiting.pop_front();
    }
    return AM_OK;
  };
  auto flush_flags = [&]() -> am_status {  // flag-only exchanges until every launched block's word is global
    while (!awaiting.empty()) {
      if (am_status s2 = tr->exchange_flags()) return s2;
      if (am_status s2 = after_exchange()) return s2;
    }
    return AM_OK;
  };
  auto drain_one = [&]() -> am_status {
    PendingBlock b = pend.front();
    pend.pop_front();
    uint32_t m = 0xFFFFFFFFu, mx = 0u;
    for (auto& s : slabs) {
      am_ctx* c = s.ctx;
      volatile uint32_t* h = s.g->fs->h + b.slot;
      if (b.polled) {  // the kernel's last CTA writes the slot through the mapping
        for (uint64_t spin = 1; *h == kSlotPending; ++spin) {
          if ((spin & 4095) == 0) {
            const cudaError_t q = cudaStreamQuery(c->stream);
            if (q == cudaSuccess && *h == kSlotPending) return fail(c, AM_ECUDA, "flag slot never written");
            if (q != cudaSuccess && q != cudaErrorNotReady) return fail(c, AM_ECUDA, "stencil: %s", cudaGetErrorString(q));
          }
        }
      } else {
        cudaError_t e = cudaEventSynchronize(s.g->fs->ev[b.slot]);
        if (e) return fail(c, AM_ECUDA, "flag event: %s", cudaGetErrorString(e));
      }
      m = std::min(m, (uint32_t)*h);
      mx = std::max(mx, (uint32_t)*h);
    }
    if (diffuse && m != mx) return fail(ctx, AM_EINTERNAL, "slab fixed-point words disagree after %u exchanges", hops);
    if (!lprime) {
      const uint32_t t = block_termination(b, m);
      if (t) lprime = t;
    }
    return AM_OK;
  };

  while (l < target && !lprime) {
    const bool blocked = mode == AM_MODE_BATCHED && target - l >= (uint32_t)K;
    const uint32_t kk = blocked ? (uint32_t)K : 1u;
    const bool promoting = slabs[0].g->cell_bits == 16 && (uint64_t)l + kk + 1 > kMax16Activity;
    if ((!blocked || promoting) && (st = close_run())) return st;
    if ((!blocked || promoting || !tiles) && (st = publish_pending())) return st;
    if (promoting) {
      if (diffuse && (st = flush_flags())) return st;
      while (!pend.empty() && !lprime)
        if ((st = drain_one())) return st;
      pend.clear();
      if (lprime) break;
      if (tiles && (st = tiles_finalize(l))) return st;
      for (auto& s : slabs)
        if ((st = promote(s.ctx, s.g))) return st;
      if (tiles && (st = tiles_all_active(l))) return st;
    }
    if (tiles && !blocked) {  // a dense single layer needs every tile current
      if ((st = tiles_finalize(l))) return st;
    }
    if (halos && blocked) {
      for (auto& sr : slabs) {  // boundary rows at layer l from the tiles' homes
        am_grid* g = sr.g;
        void* top = tr ? tr->boundary_dst(0) : nullptr;
        void* bot = tr ? tr->boundary_dst(1) : nullptr;
        if (!top) top = g->t_bnd;
        if (!bot) bot = static_cast<uint8_t*>(g->t_bnd) + (size_t)kK * g->g.pitch * (g->cell_bits / 8);
        launch_tiles_boundary(g->g, g->cell_bits, g->t_state, g->val[0], g->val[1], l, top, bot, sr.ctx->stream);
        CKL();
      }
      if (tr && (st = tr->exchange_tiles())) return st;  // (a lone slab has no neighbours: halos stay padding)
      if (diffuse && (st = after_exchange())) return st;
      for (auto& sr : slabs) {  // boundary tiles the received frontier reaches
        am_grid* g = sr.g;
        launch_tiles_halo_scan(g->g, g->cell_bits, g->val[0], g->book(), g->t_blk, sr.ctx->stream);
        CKL();
      }
    } else if (tr) {  // dense blocks / single layers (tiles gathered into val[0])
      if ((st = tr->exchange())) return st;
      if (diffuse && (st = after_exchange())) return st;
    }
    const int slot = (int)(nblock % kFlagSlots);
    for (size_t i = 0; i < slabs.size(); ++i) {
      am_ctx* c = slabs[i].ctx;
      am_grid* g = slabs[i].g;
      uint32_t* flag = g->d_flags + slot;
      words[i] = flag;
      cudaStream_t s = c->stream;
      // a mapped slot is re-armed by the launch that used it
      if (autom && !(mapped && blocked && armed[slot])) {
        cudaError_t e = cudaMemsetAsync(flag, 0xFF, sizeof(uint32_t), s);
        if (e) return fail(c, AM_ECUDA, "memset: %s", cudaGetErrorString(e));
      }
      armed[slot] = mapped && blocked;
      if (mapped && blocked) g->fs->h[slot] = kSlotPending;  // consumed 64 blocks ago (lag < kFlagSlots)
      FlagSink sink{flag, g->d_flags + kFlagSlots, mapped ? g->fs->hdev + slot : nullptr};
      void* in = g->val[g->cur];
      void* outp = g->val[g->cur ^ 1];
      if (blocked) {
        if (timing && i == 0 && !run_open) {
          if (timer_used == ctx->timers.size()) {
            am_ctx::Timer t;
            CK(cudaEventCreate(&t.a));
            CK(cudaEventCreate(&t.b));
            ctx->timers.push_back(t);
          }
          CK(cudaEventRecord(ctx->timers[timer_used].a, s));
          run_open = true;
        }
        if (tiles) {
          // the tiles of this block list the next block's tiles themselves (TileBook)
          const FlagSink prev = unpublished;
          if (sink.host) {  // published by the next tile launch (or publish_pending)
            unpublished = sink;
            sink.host = nullptr;
          }
          launch_block_tiles(g->g, g->cell_bits, tile_ctas, g->val[0], g->val[1], g->srcmask, g->rowsrc, g->book(),
                             g->t_blk, l, sink, prev, !halos, s);
          ++g->t_blk;
        } else {
          launch_block(g->g, g->cell_bits, g->slab != 0, in, outp, g->srcmask, g->rowsrc, sink, s);
        }
        ++c->launches;
        if (cudaError_t e = cudaPeekAtLastError()) return fail(c, AM_ECUDA, "k_block: %s", cudaGetErrorString(e));
        ++r.block_launches;
      } else {
        launch_layer(g->g, g->cell_bits, in, outp, g->srcmask, flag, s);
        ++c->launches;
        if (cudaError_t e = cudaPeekAtLastError()) return fail(c, AM_ECUDA, "k_layer: %s", cudaGetErrorString(e));
        ++r.layer_launches;
      }
      g->cur ^= 1;
    }
    if (tiles && !blocked && (st = tiles_all_active(l + kk))) return st;
    if (autom) {
      const PendingBlock pb{slot, l, kk, slabs[0].g->cell_bits, mapped && blocked};
      if (hops) awaiting.push_back(Awaiting{pb, 0});
      else if ((st = copy_out(pb))) return st;
    }
    l += kk;
    ++nblock;
    if (mode == AM_MODE_ITERATIVE)  // per-layer call boundary
      for (auto& sr : slabs) {
        am_ctx* c = sr.ctx;
        CK(cudaStreamSynchronize(c->stream));
      }
    // Tile mode runs far ahead of the host: blocks past the fixed point have
    // no frontier, so they cost a near-empty launch each.  Dense blocks past
    // it cost a full sweep, so the dense path keeps the lag short.
    while ((int)pend.size() > (tiles ? kLagTiles : kLag))
      if ((st = drain_one())) return st;
  }
  if ((st = close_run())) return st;
  if ((st = publish_pending())) return st;
  if (diffuse && (st = flush_flags())) return st;
  while (!pend.empty())
    if ((st = drain_one())) return st;
  const int zslot = (int)(nblock % kFlagSlots);
  if (tiles) {
    if ((st = tiles_finalize(l, autom ? zslot : -1))) return st;  // the gather also runs the zero check
    for (auto& sr : slabs) {
      unsigned long long proc = 0;
      CK(cudaMemcpyAsync(&proc, sr.g->t_processed, 8, cudaMemcpyDeviceToHost, sr.ctx->stream));
      CK(cudaStreamSynchronize(sr.ctx->stream));
      r.tiles_processed += proc;
    }
    r.tiles_total = nt * r.block_launches;
  }
  uint32_t used = l, cause = AM_STOP_FIXED;
  if (autom) {
    for (size_t i = 0; i < slabs.size(); ++i) {
      am_ctx* c = slabs[i].ctx;
      am_grid* g = slabs[i].g;
      uint32_t* z = g->d_flags + zslot;
      words[i] = z;
      if (tiles) continue;  // done by the gather
      CK(cudaMemsetAsync(z, 0, sizeof(uint32_t), c->stream));
      launch_zero_check(g->g, g->cell_bits, g->val[g->cur], z, c->stream);
      CKL();
    }
    if (tr && (st = tr->reduce(words, true))) return st;
    uint32_t any_zero = 0;
    for (auto& sr : slabs) {
      am_ctx* c = sr.ctx;
      uint32_t v = 0;
      CK(cudaMemcpyAsync(&v, sr.g->d_flags + zslot, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      any_zero |= v;
    }
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
    for (auto& sr : slabs) {
      am_ctx* c = sr.ctx;
      CK(cudaStreamSynchronize(c->stream));
    }
  }
  for (auto& sr : slabs) {
    sr.g->computed = l;
    sr.g->layers_used = used;
  }
  if (timing) {
    CK(cudaStreamSynchronize(ctx->stream));
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
  r.cell_bits = slabs[0].g->cell_bits;
  if (tiles) {
    r.cells_executed = r.tiles_processed * (uint64_t)(kTileRows * kTileCols) * kK;
    r.engine = AM_ENGINE_TILES;
  } else {
    uint64_t cells = 0;
    for (auto& sr : slabs) cells += (uint64_t)sr.g->g.W * sr.g->g.H;  // owned rows of each slab
    r.cells_executed = cells * kK * (r.block_launches / slabs.size());
    r.engine = AM_ENGINE_DENSE;
  }
  r.block_layers = kK;
  if (pre.block_launches) {  // a bit-plane run did the layers up to the handoff
    r.engine = pre.engine;
    r.block_layers = pre.block_layers;
  }
  r.block_launches += pre.block_launches;
  r.tiles_processed += pre.tiles_processed;
  r.cells_executed += pre.cells_executed;
  if (res) *res = r;
  return AM_OK;
}

}  // namespace am

extern "C" {

am_status am_propagate(am_ctx* ctx, am_grid* g, uint32_t layers, uint32_t auto_cap, uint32_t mode,
                       am_prop_result* res) {
  if (!ctx || !g) return AM_EINVAL;
  std::vector<am::SlabRef> one{{ctx, g}};
  am::Transport* tr = nullptr;
  if (g->slab && g->peer) {
    tr = am::make_peer_transport(ctx, g);
  } else if (g->slab) {
    if (!ctx->comm)
      return am::fail(ctx, AM_EINVAL, "slab grid: call am_peer_connect / am_comm_init or use am_slabs_propagate");
    tr = am::make_nccl_transport(ctx, g);
    if (!tr) return am::fail(ctx, AM_ENCCL, "cannot build the NCCL halo transport");
  }
  am_status st = am::drive_propagation(one, tr, layers, auto_cap, mode, res);
  delete tr;
  return st;
}

}  // extern "C"

// ------------------------------------------------------------- download

static am_status download_impl(am_ctx* ctx, am_grid* g, uint32_t* dst, bool dst_device) {
  if (!ctx || !g || !dst) return AM_EINVAL;
  if (!g->have_map) return am::fail(ctx, AM_EINVAL, "no activity map: call am_propagate first");
  CK(cudaSetDevice(ctx->device));
  am_status jst = am::join_map(ctx, g);
  if (jst) return jst;
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
  // decode into the idle ping-pong buffer in row chunks (ctx stream) while the previous chunk is
  // copied out on the copy stream: the PCIe copy is the floor, the decode hides behind it
  uint32_t* stage = (uint32_t*)g->val[g->cur ^ 1];
  g->dirty[g->cur ^ 1] = 1;
  if (g->cur == 0) g->bits_map = 0;  // val[1] (the time planes) is the staging buffer now
  const size_t stage_bytes = (size_t)g->g.rows * g->g.pitch * (g->cell_bits / 8);
  constexpr int kChunks = 4;  // stage buffers in flight
  size_t rows_per = std::min(stage_bytes / (W * 4 * kChunks), std::max<size_t>(1, (256u << 20) / (W * 4)));
  if (rows_per < 1) rows_per = 1;
  if (!ctx->copy_stream) CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  for (auto& e : ctx->copy_ev)
    if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  int k = 0;
  for (size_t r0 = 0; r0 < H; r0 += rows_per, k = (k + 1) % kChunks) {
    const size_t r1 = std::min(H, r0 + rows_per);
    uint32_t* buf = stage + (size_t)k * rows_per * W;
    if (r0 >= kChunks * rows_per) CK(cudaStreamWaitEvent(s, ctx->copy_ev[2 * k + 1], 0));  // buffer copied out
    am::launch_decode(g->g, g->cell_bits, g->val[g->cur], rollback, (uint32_t)r0, (uint32_t)r1, buf, s);
    CKL();
    CK(cudaEventRecord(ctx->copy_ev[2 * k], s));
    CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_ev[2 * k], 0));
    CK(cudaMemcpyAsync(dst + r0 * W, buf, (r1 - r0) * W * 4, cudaMemcpyDeviceToHost, ctx->copy_stream));
    CK(cudaEventRecord(ctx->copy_ev[2 * k + 1], ctx->copy_stream));
  }
  CK(cudaStreamSynchronize(ctx->copy_stream));
  CK(cudaStreamWaitEvent(s, ctx->copy_ev[2 * ((k + kChunks - 1) % kChunks) + 1], 0));  // later decodes order after
  return AM_OK;
}

extern "C" {

am_status am_activity_download(am_ctx* ctx, am_grid* g, uint32_t* dense) { return download_impl(ctx, g, dense, false); }

am_status am_activity_download_device(am_ctx* ctx, am_grid* g, uint32_t* dense) {
  return download_impl(ctx, g, dense, true);
}

am_status am_activity_upload(am_ctx* ctx, am_grid* g, const uint32_t* dense, uint32_t layers_applied) {
  if (!ctx || !g || !dense) return AM_EINVAL;
  if (g->slab) return am::fail(ctx, AM_EINVAL, "activity upload on a slab grid");
  CK(cudaSetDevice(ctx->device));
  if (am_status jst = am::join_map(ctx, g)) return jst;
  const size_t n = (size_t)g->g.W * g->g.H;
  if (!g->plain) CK(am::dmalloc(ctx, &g->plain, n * 4));
  CK(cudaMemcpyAsync(g->plain, dense, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  ctx->h2d_bytes += n * 4;
  CK(cudaStreamSynchronize(ctx->stream));
  g->plain_active = 1;
  g->plain_layers = layers_applied;
  g->have_map = 1;
  return AM_OK;
}

}  // extern "C"

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
    if (g->bits_map && g->bits && g->cur == 0 && g->cell_bits == 16) {
      m.bp = g->bits->bk.P;
      m.bt = g->bits->bk.T;
      m.bstate = g->bits->bk.state;
      m.bg = g->bits->bg;
    }
  }
  return m;
}

static am_status ensure_targets(am_ctx* ctx, am_grid* g, uint64_t n) {
  if (!g->d_sched) CK(am::dmalloc(ctx, &g->d_sched, am::kTraceSchedWords * sizeof(uint32_t)));
  if (n <= g->tgt_cap) return AM_OK;
  am::dfree(ctx, g->d_tgt);
  am::dfree(ctx, g->d_counts);
  am::dfree(ctx, g->d_offsets);
  am::dfree(ctx, g->d_status);
  g->d_tgt = nullptr;
  g->d_counts = g->d_offsets = nullptr;
  g->d_status = nullptr;
  g->tgt_cap = 0;
  CK(am::dmalloc(ctx, &g->d_tgt, n * 2 * sizeof(uint32_t)));
  CK(am::dmalloc(ctx, &g->d_counts, n * sizeof(uint64_t)));
  CK(am::dmalloc(ctx, &g->d_offsets, (n + 1) * sizeof(uint64_t)));
  CK(am::dmalloc(ctx, &g->d_status, n * sizeof(int32_t)));
  g->tgt_cap = n;
  return AM_OK;
}

namespace am {
am_status trace_scratch(am_ctx* ctx, am_grid* g, uint64_t n) { return ensure_targets(ctx, g, n); }
}  // namespace am

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

extern "C" {

am_status am_path_counts(am_ctx* ctx, am_grid* g, const uint32_t* tgt, uint64_t n, uint32_t method, uint64_t seed,
                         uint64_t* offsets, int32_t* status) {
  if (!ctx || !g || (n && (!tgt || !status)) || !offsets) return AM_EINVAL;
  if (!g->have_map) return am::fail(ctx, AM_EINVAL, "no activity map");
  if (g->slab) return am::fail(ctx, AM_EINVAL, "path extraction on a slab: gather the map first");
  if (method > 1) return am::fail(ctx, AM_EINVAL, "bad method");
  CK(cudaSetDevice(ctx->device));
  offsets[0] = 0;
  if (!n) return AM_OK;
  am_status st = ensure_targets(ctx, g, n);
  if (st) return st;
  cudaStream_t s = ctx->stream;
  CK(cudaMemcpyAsync(g->d_tgt, tgt, n * 8, cudaMemcpyHostToDevice, s));
  ctx->h2d_bytes += n * 8;
  am::launch_path_counts(view_of(g), g->d_tgt, n, (int)method, seed, g->d_counts, g->d_status, s);
  CKL();
  am::launch_scan(g->d_counts, n, g->d_offsets, s);
  CKL();
  CK(cudaMemcpyAsync(offsets, g->d_offsets, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(status, g->d_status, n * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return AM_OK;
}

am_status am_trace_paths(am_ctx* ctx, am_grid* g, const uint32_t* tgt, uint64_t n, uint32_t method, uint64_t seed,
                         const uint64_t* offsets, uint32_t* pts, uint64_t cap, int32_t* status) {
  return am::trace_paths_host(ctx, g, tgt, n, method, seed, offsets, pts, cap, status, 0, 0);
}

}  // extern "C"

namespace am {
// am_trace_paths; cell_h / cell_w > 0: the grid packs mazes on a (cell_h x cell_w) lattice
// (am_batch) and every path is returned in its maze's local coordinates (device pass before the copy)
am_status trace_paths_host(am_ctx* ctx, am_grid* g, const uint32_t* tgt, uint64_t n, uint32_t method, uint64_t seed,
                           const uint64_t* offsets, uint32_t* pts, uint64_t cap, int32_t* status, uint32_t cell_h,
                           uint32_t cell_w) {
  if (!ctx || !g || !offsets || (n && (!tgt || !status))) return AM_EINVAL;
  if (!g->have_map) return am::fail(ctx, AM_EINVAL, "no activity map");
  if (g->slab) return am::fail(ctx, AM_EINVAL, "path extraction on a slab: gather the map first");
  if (method > 1) return am::fail(ctx, AM_EINVAL, "bad method");
  if (!n) return AM_OK;
  const uint64_t total = offsets[n];
  if (total > cap || (total && !pts))
    return am::fail(ctx, AM_EINVAL, "point buffer too small (%llu < %llu)", (unsigned long long)cap,
                    (unsigned long long)total);
  CK(cudaSetDevice(ctx->device));
  am_status st = ensure_targets(ctx, g, n);
  if (st) return st;
  cudaStream_t s = ctx->stream;
  // A pinned (device-mapped) destination takes the points straight from the walkers: the 32-point
  // warp stores cross PCIe while the walk runs instead of a separate copy afterwards.
  uint32_t* direct = nullptr;
  if (total) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, pts) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer)
      direct = static_cast<uint32_t*>(at.devicePointer);
    (void)cudaGetLastError();
  }
  if (!direct && total > g->pts_cap) {
    am::dfree(ctx, g->d_pts);
    g->d_pts = nullptr;
    g->pts_cap = 0;
    CK(am::dmalloc(ctx, &g->d_pts, total * 8));
    g->pts_cap = total;
  }
  CK(cudaMemcpyAsync(g->d_tgt, tgt, n * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(g->d_offsets, offsets, (n + 1) * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(g->d_status, status, n * 4, cudaMemcpyHostToDevice, s));
  ctx->h2d_bytes += n * 8 + (n + 1) * 8 + n * 4;
  // the counts are consumed (offsets came from the caller): their buffer holds the trace order
  {
    am::MapView m = view_of(g);
    m.cell_h = cell_h;  // batch lattices: the walkers write maze-local points
    m.cell_w = cell_w;
    if (!m.bt && (st = am::join_map(ctx, g))) return st;  // the walkers read the field
    am::launch_trace(m, g->d_tgt, n, (int)method, seed, g->d_offsets, direct ? direct : g->d_pts, g->d_status, s,
                     ~0ull, reinterpret_cast<uint32_t*>(g->d_counts), g->d_sched, ctx->sms);
    CKL();
    if ((st = am::join_map(ctx, g))) return st;  // the map is complete when the paths are
  }
  if (total && !direct) CK(cudaMemcpyAsync(pts, g->d_pts, total * 8, cudaMemcpyDeviceToHost, s));
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

}  // namespace am

extern "C" {

am_status am_trace_paths_device(am_ctx* ctx, am_grid* g, const uint32_t* d_tgt, uint64_t n, uint32_t method,
                                uint64_t seed, uint64_t* d_offsets, uint32_t* d_pts, uint64_t cap,
                                int32_t* d_status) {
  if (!ctx || !g || !d_offsets || (n && (!d_tgt || !d_status))) return AM_EINVAL;
  if (!g->have_map) return am::fail(ctx, AM_EINVAL, "no activity map");
  if (g->plain_active) return am::fail(ctx, AM_EINVAL, "device path tracing needs a propagated map");
  if (g->slab) return am::fail(ctx, AM_EINVAL, "path extraction on a slab: gather the map first");
  if (method > 1) return am::fail(ctx, AM_EINVAL, "bad method");
  if (!n) return AM_OK;
  if (!d_pts && cap) return am::fail(ctx, AM_EINVAL, "null point buffer");
  CK(cudaSetDevice(ctx->device));
  am_status st = ensure_targets(ctx, g, n);
  if (st) return st;
  cudaStream_t s = ctx->stream;
  am::MapView m = view_of(g);
  am::launch_path_counts(m, d_tgt, n, (int)method, seed, g->d_counts, d_status, s);
  CKL();
  am::launch_scan(g->d_counts, n, d_offsets, s);
  CKL();
  // paths past cap: AM_EINVAL; the counts are scanned into d_offsets, so their buffer holds the trace order
  if (!m.bt && (st = am::join_map(ctx, g))) return st;  // the walkers read the field
  am::launch_trace(m, d_tgt, n, (int)method, seed, d_offsets, d_pts, d_status, s, cap,
                   reinterpret_cast<uint32_t*>(g->d_counts), g->d_sched, ctx->sms);
  CKL();
  return am::join_map(ctx, g);  // the map is complete when the paths are
}

// -------------------------------------------------------- single-shot ops

am_status am_propagate_layer(am_ctx* ctx, uint32_t W, uint32_t H, const uint8_t* occ, const uint32_t* src,
                             uint64_t n_src, const uint32_t* in, uint32_t* out) {
  if (!ctx || !occ || !in || !out || (n_src && !src)) return AM_EINVAL;
  if (!am::dims_ok(W, H)) return am::fail(ctx, AM_EINVAL, "grid dimensions %ux%u outside 1..65535", W, H);
  if (!n_src) return am::fail(ctx, AM_EINVAL, "SourceSet must be nonempty");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const size_t n = (size_t)W * H;
  uint8_t *d_occ = nullptr, *d_sm = nullptr;
  uint32_t *d_in = nullptr, *d_out = nullptr, *d_src = nullptr;
  int* d_err = nullptr;
  int h_err = 0;
  am_status st = AM_OK;
  cudaError_t e = am::dmalloc(ctx, &d_occ, n);
  if (!e) e = am::dmalloc(ctx, &d_sm, n);
  if (!e) e = am::dmalloc(ctx, &d_in, n * 4);
  if (!e) e = am::dmalloc(ctx, &d_out, n * 4);
  if (!e) e = am::dmalloc(ctx, &d_src, n_src * 8);
  if (!e) e = am::dmalloc(ctx, &d_err, 4);
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
  if (e) st = am::fail(ctx, e == cudaErrorMemoryAllocation ? AM_EOOM : AM_ECUDA, "%s", cudaGetErrorString(e));
  else if (h_err) st = am::fail(ctx, AM_EINVAL, "SourceSet: a source is out of bounds or on an obstacle");
  (void)cudaGetLastError();
  am::dfree(ctx, d_occ);
  am::dfree(ctx, d_sm);
  am::dfree(ctx, d_in);
  am::dfree(ctx, d_out);
  am::dfree(ctx, d_src);
  am::dfree(ctx, d_err);
  return st;
}

am_status am_propagate_reference(am_ctx* ctx, uint32_t W, uint32_t H, const uint8_t* occ, const uint32_t* src,
                                 uint64_t n_src, uint32_t layers, uint32_t* out) {
  if (!ctx || !occ || !out || (n_src && !src)) return AM_EINVAL;
  if (!am::dims_ok(W, H)) return am::fail(ctx, AM_EINVAL, "grid dimensions %ux%u outside 1..65535", W, H);
  if (!n_src) return am::fail(ctx, AM_EINVAL, "SourceSet must be nonempty");
  if (layers == 0 || layers > am::kMaxLayers) return am::fail(ctx, AM_EINVAL, "layer count %u out of range", layers);
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const size_t n = (size_t)W * H;
  uint8_t *d_occ = nullptr, *d_sm = nullptr;
  int32_t *a = nullptr, *b = nullptr;
  uint32_t* d_src = nullptr;
  int* d_err = nullptr;
  int h_err = 0;
  am_status st = AM_OK;
  cudaError_t e = am::dmalloc(ctx, &d_occ, n);
  if (!e) e = am::dmalloc(ctx, &d_sm, n);
  if (!e) e = am::dmalloc(ctx, &a, n * 4);
  if (!e) e = am::dmalloc(ctx, &b, n * 4);
  if (!e) e = am::dmalloc(ctx, &d_src, n_src * 8);
  if (!e) e = am::dmalloc(ctx, &d_err, 4);
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
  if (e) st = am::fail(ctx, e == cudaErrorMemoryAllocation ? AM_EOOM : AM_ECUDA, "%s", cudaGetErrorString(e));
  else if (h_err) st = am::fail(ctx, AM_EINVAL, "SourceSet: a source is out of bounds or on an obstacle");
  (void)cudaGetLastError();
  am::dfree(ctx, d_occ);
  am::dfree(ctx, d_sm);
  am::dfree(ctx, a);
  am::dfree(ctx, b);
  am::dfree(ctx, d_src);
  am::dfree(ctx, d_err);
  return st;
}

am_status am_bench_tile_kernel(am_ctx* ctx, am_grid* g, uint32_t items, uint32_t stride, uint32_t reps,
                               float* ms_per_launch) {
  if (!ctx || !g || !ms_per_launch || !g->t_state || reps == 0 || stride == 0) return AM_EINVAL;
  CK(cudaSetDevice(ctx->device));
  if (am_status jst = am::join_map(ctx, g)) return jst;
  am_status st = am::reset_map(ctx, g, 16);
  if (st) return st;
  g->have_map = 0;
  const uint32_t nt = (uint32_t)g->g.ntiles();
  const uint32_t n = std::min<uint64_t>((uint64_t)items * 2, nt);
  std::vector<uint8_t> tsrc(nt);
  CK(cudaMemcpy(tsrc.data(), g->t_src, nt, cudaMemcpyDeviceToHost));
  std::vector<uint32_t> list(n);
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t t = (uint32_t)(((uint64_t)i * stride) % nt);
    list[i] = (t % g->g.tbands) << 16 | (t / g->g.tbands) | (tsrc[t] ? am::kListSrc : 0u);
  }
  cudaStream_t s = ctx->stream;
  // block 0 every launch: list[0] / count[0] stay, the pushes for block 1 are deduplicated away
  CK(cudaMemsetAsync(g->t_state, 0, (size_t)nt * 8, s));
  CK(cudaMemsetAsync(g->t_sched, 0, (size_t)nt * 4, s));
  CK(cudaMemsetAsync(g->t_count, 0, 6 * 4, s));
  CK(cudaMemcpyAsync(g->t_list[0], list.data(), (size_t)n * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(g->t_count, &n, 4, cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  const am::FlagSink sink{g->d_flags, g->d_flags + am::kFlagSlots, nullptr};
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (uint32_t r = 0; r < reps + 2; ++r) {
    CK(cudaMemsetAsync(g->t_count + 3, 0, 4, s));  // block 0's item fetch counter
    if (r == 2) CK(cudaEventRecord(a, s));
    am::launch_block_tiles(g->g, 16, ctx->sms * am::kTileCtasPerSm, g->val[0], g->val[1], g->srcmask, g->rowsrc,
                           g->book(), 0, 0, sink, am::FlagSink{nullptr, nullptr, nullptr}, true, s);
    ++ctx->launches;
  }
  CK(cudaEventRecord(b, s));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  CK(cudaMemsetAsync(g->d_flags, 0xFF, am::kFlagSlots * sizeof(uint32_t), s));
  *ms_per_launch = ms / reps;
  return AM_OK;
}

}  // extern "C"
