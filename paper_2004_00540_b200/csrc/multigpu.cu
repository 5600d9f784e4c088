// multigpu.cu -- row-slab decomposition.
//
// A grid of H rows is cut into slabs of consecutive rows.  Each slab's
// device field keeps K = kK halo rows above and below its own rows (the
// padding rows of the single-GPU layout), and before every launch the
// slabs refresh those halos from their neighbours' boundary rows at the
// current layer -- exactly the K rows a K-layer block needs.  The per-block
// fixed-point number is min-reduced across slabs so every slab stops at the
// same layer with the same rollback.
//
// Two transports share the driver in capi.cu:
//  * NCCL (one process per GPU): grouped ncclSend/ncclRecv of the K
//    boundary rows over NVLink, ncclAllReduce(min/max) for the flags.
//    libnccl.so.2 is opened at am_comm_init time (the process may already
//    hold torch's copy), so the library has no link-time NCCL dependency.
//  * in-process groups on one device (am_slabs_*): device-to-device copies
//    on the shared stream.  They run the identical decomposition, so the
//    slab logic is tested on a single GPU against the oracle.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "am_host.hpp"

namespace am {

struct NcclApi {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  bool ok = false;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.h = h;
#define LOAD(field, sym) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, #sym))
  LOAD(getUniqueId, ncclGetUniqueId);
  LOAD(commInitRank, ncclCommInitRank);
  LOAD(commDestroy, ncclCommDestroy);
  LOAD(groupStart, ncclGroupStart);
  LOAD(groupEnd, ncclGroupEnd);
  LOAD(send, ncclSend);
  LOAD(recv, ncclRecv);
  LOAD(allReduce, ncclAllReduce);
  LOAD(broadcast, ncclBroadcast);
  LOAD(errorString, ncclGetErrorString);
#undef LOAD
  api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.groupStart && api.groupEnd && api.send &&
           api.recv && api.allReduce && api.broadcast && api.errorString;
  return api;
}

struct Comm {
  ncclComm_t comm = nullptr;
  uint32_t nranks = 1, rank = 0;
};

void comm_destroy(Comm* c) {
  if (!c) return;
  if (c->comm && nccl().ok) nccl().commDestroy(c->comm);
  delete c;
}

#define NK(call)                                                                                   \
  do {                                                                                             \
    ncclResult_t r_ = (call);                                                                      \
    if (r_ != ncclSuccess) return fail(ctx, AM_ENCCL, "%s: %s", #call, nccl().errorString(r_));    \
  } while (0)

static size_t row_bytes(const am_grid* g) { return (size_t)g->g.pitch * (g->cell_bits / 8); }

// halo rows of slab g live at allocated rows [0, K) (top) and [K+H, 2K+H) (bottom);
// its own boundary rows at [K, 2K) (top) and [H, H+K) (bottom)
static uint8_t* alloc_rows(am_grid* g, uint32_t arow) {
  return static_cast<uint8_t*>(g->val[g->cur]) + (size_t)arow * row_bytes(g);
}

struct NcclTransport final : Transport {
  am_ctx* ctx;
  am_grid* g;
  NcclTransport(am_ctx* c, am_grid* gg) : ctx(c), g(gg) {}
  // the slot words to / from both neighbours (inside the caller's group), then folded in
  am_status flags_p2p() {
    Comm* cm = ctx->comm;
    const size_t n = kFlagSlots;
    if (cm->rank > 0) {
      NK(nccl().send(g->d_flags, n, ncclUint32, (int)cm->rank - 1, cm->comm, ctx->stream));
      NK(nccl().recv(g->d_flags + kFlagRecvUp, n, ncclUint32, (int)cm->rank - 1, cm->comm, ctx->stream));
    }
    if (cm->rank + 1 < cm->nranks) {
      NK(nccl().send(g->d_flags, n, ncclUint32, (int)cm->rank + 1, cm->comm, ctx->stream));
      NK(nccl().recv(g->d_flags + kFlagRecvDn, n, ncclUint32, (int)cm->rank + 1, cm->comm, ctx->stream));
    }
    return AM_OK;
  }
  am_status merge() {
    launch_flags_merge(g->d_flags, ctx->stream);
    ++ctx->launches;
    if (cudaError_t e = cudaPeekAtLastError()) return fail(ctx, AM_ECUDA, "flags merge: %s", cudaGetErrorString(e));
    return AM_OK;
  }
  am_status exchange() override {
    Comm* cm = ctx->comm;
    const size_t bytes = (size_t)kK * row_bytes(g);
    const uint32_t H = g->g.H;
    NK(nccl().groupStart());
    if (cm->rank > 0) {
      NK(nccl().send(alloc_rows(g, kK), bytes, ncclUint8, (int)cm->rank - 1, cm->comm, ctx->stream));
      NK(nccl().recv(alloc_rows(g, 0), bytes, ncclUint8, (int)cm->rank - 1, cm->comm, ctx->stream));
    }
    if (cm->rank + 1 < cm->nranks) {
      NK(nccl().send(alloc_rows(g, H), bytes, ncclUint8, (int)cm->rank + 1, cm->comm, ctx->stream));
      NK(nccl().recv(alloc_rows(g, kK + H), bytes, ncclUint8, (int)cm->rank + 1, cm->comm, ctx->stream));
    }
    if (am_status st = flags_p2p()) return st;
    NK(nccl().groupEnd());
    return merge();
  }
  am_status exchange_flags() override {
    NK(nccl().groupStart());
    if (am_status st = flags_p2p()) return st;
    NK(nccl().groupEnd());
    return merge();
  }
  uint32_t span() const override { return ctx->comm->nranks; }
  am_status exchange_tiles() override {
    Comm* cm = ctx->comm;
    const size_t bytes = (size_t)kK * row_bytes(g);
    uint8_t* bnd = static_cast<uint8_t*>(g->t_bnd);
    uint8_t* f0 = static_cast<uint8_t*>(g->val[0]);
    const uint32_t H = g->g.H;
    NK(nccl().groupStart());
    if (cm->rank > 0) {
      NK(nccl().send(bnd, bytes, ncclUint8, (int)cm->rank - 1, cm->comm, ctx->stream));
      NK(nccl().recv(f0, bytes, ncclUint8, (int)cm->rank - 1, cm->comm, ctx->stream));
    }
    if (cm->rank + 1 < cm->nranks) {
      NK(nccl().send(bnd + bytes, bytes, ncclUint8, (int)cm->rank + 1, cm->comm, ctx->stream));
      NK(nccl().recv(f0 + (size_t)(kK + H) * row_bytes(g), bytes, ncclUint8, (int)cm->rank + 1, cm->comm,
                     ctx->stream));
    }
    if (am_status st = flags_p2p()) return st;
    NK(nccl().groupEnd());
    return merge();
  }
  am_status reduce(std::vector<uint32_t*>& words, bool take_max) override {
    NK(nccl().allReduce(words[0], words[0], 1, ncclUint32, take_max ? ncclMax : ncclMin, ctx->comm->comm,
                        ctx->stream));
    return AM_OK;
  }
  bool host_combine() const override { return false; }
  bool lower_neighbour() const override { return ctx->comm->rank + 1 < ctx->comm->nranks; }
};

Transport* make_nccl_transport(am_ctx* ctx, am_grid* g) {
  if (!ctx->comm || !nccl().ok) return nullptr;
  return new NcclTransport(ctx, g);
}

// In-process slabs sharing one context (one stream): plain D2D copies.
struct LocalTransport final : Transport {
  am_ctx* ctx;
  std::vector<SlabRef>& s;
  LocalTransport(am_ctx* c, std::vector<SlabRef>& v) : ctx(c), s(v) {}
  // every slab's slot words into its neighbours' receive rings (all copies before any merge, as
  // the NCCL exchange delivers them), then each slab folds them in
  am_status flags() {
    const size_t bytes = kFlagSlots * sizeof(uint32_t);
    for (size_t i = 0; i < s.size(); ++i) {
      if (i > 0) CK(cudaMemcpyAsync(s[i].g->d_flags + kFlagRecvUp, s[i - 1].g->d_flags, bytes, cudaMemcpyDeviceToDevice,
                                    ctx->stream));
      if (i + 1 < s.size())
        CK(cudaMemcpyAsync(s[i].g->d_flags + kFlagRecvDn, s[i + 1].g->d_flags, bytes, cudaMemcpyDeviceToDevice,
                           ctx->stream));
    }
    for (size_t i = 0; i < s.size(); ++i) {
      launch_flags_merge(s[i].g->d_flags, ctx->stream);
      ++ctx->launches;
    }
    CK(cudaPeekAtLastError());
    return AM_OK;
  }
  am_status exchange_flags() override { return flags(); }
  uint32_t span() const override { return (uint32_t)s.size(); }
  am_status exchange() override {
    for (size_t i = 0; i < s.size(); ++i) {
      am_grid* g = s[i].g;
      const size_t bytes = (size_t)kK * row_bytes(g);
      if (i > 0) {
        am_grid* up = s[i - 1].g;
        CK(cudaMemcpyAsync(alloc_rows(g, 0), alloc_rows(up, up->g.H), bytes, cudaMemcpyDeviceToDevice, ctx->stream));
      }
      if (i + 1 < s.size()) {
        am_grid* dn = s[i + 1].g;
        CK(cudaMemcpyAsync(alloc_rows(g, kK + g->g.H), alloc_rows(dn, kK), bytes, cudaMemcpyDeviceToDevice,
                           ctx->stream));
      }
    }
    return flags();
  }
  am_status exchange_tiles() override {
    for (size_t i = 0; i < s.size(); ++i) {
      am_grid* g = s[i].g;
      const size_t bytes = (size_t)kK * row_bytes(g);
      uint8_t* f0 = static_cast<uint8_t*>(g->val[0]);
      if (i > 0)  // the slab above's last rows become this slab's top halo
        CK(cudaMemcpyAsync(f0, static_cast<uint8_t*>(s[i - 1].g->t_bnd) + bytes, bytes, cudaMemcpyDeviceToDevice,
                           ctx->stream));
      if (i + 1 < s.size())
        CK(cudaMemcpyAsync(f0 + (size_t)(kK + g->g.H) * row_bytes(g), s[i + 1].g->t_bnd, bytes,
                           cudaMemcpyDeviceToDevice, ctx->stream));
    }
    return flags();
  }
  am_status reduce(std::vector<uint32_t*>&, bool) override { return AM_OK; }
  bool host_combine() const override { return true; }
};

// Places a propagated slab's own rows into the full grid's field.
static am_status adopt_full(am_ctx* ctx, am_grid* full, const am_grid* like) {
  am_status st = set_cell_bits(ctx, full, like->cell_bits);
  if (st) return st;
  full->cur = 0;
  full->plain_active = 0;
  full->have_map = 1;
  full->computed = like->computed;
  full->layers_used = like->layers_used;
  return AM_OK;
}

}  // namespace am

using namespace am;

extern "C" {

am_status am_grid_create_slab(am_ctx* ctx, uint32_t W, uint32_t H, uint32_t row0, uint32_t row1,
                              const uint8_t* occupancy_full, const uint32_t* src_rc, uint64_t n_src, am_grid** out) {
  return grid_create_rows(ctx, W, H, row0, row1, occupancy_full, src_rc, n_src, false, true, out);
}

am_status am_slabs_propagate(am_ctx* ctx, am_grid** slabs, uint32_t n, uint32_t layers, uint32_t auto_cap,
                             uint32_t mode, am_prop_result* res) {
  if (!ctx || !slabs || n == 0) return AM_EINVAL;
  std::vector<SlabRef> v;
  for (uint32_t i = 0; i < n; ++i) {
    if (!slabs[i] || !slabs[i]->slab) return fail(ctx, AM_EINVAL, "am_slabs_propagate: grid %u is not a slab", i);
    if (i && (slabs[i]->row0 != slabs[i - 1]->row0 + slabs[i - 1]->g.H || slabs[i]->g.pitch != slabs[0]->g.pitch))
      return fail(ctx, AM_EINVAL, "am_slabs_propagate: slabs must be consecutive rows of one grid");
    v.push_back(SlabRef{ctx, slabs[i]});
  }
  LocalTransport tr(ctx, v);
  return drive_propagation(v, n > 1 ? &tr : nullptr, layers, auto_cap, mode, res);
}

am_status am_slabs_gather(am_ctx* ctx, am_grid** slabs, uint32_t n, am_grid* full) {
  if (!ctx || !slabs || !n || !full) return AM_EINVAL;
  if (full->slab || full->g.pitch != slabs[0]->g.pitch || full->g.H != slabs[0]->total_h)
    return fail(ctx, AM_EINVAL, "am_slabs_gather: full grid does not match the slabs");
  CK(cudaSetDevice(ctx->device));
  am_status st = adopt_full(ctx, full, slabs[0]);
  if (st) return st;
  for (uint32_t i = 0; i < n; ++i) {
    am_grid* s = slabs[i];
    const size_t rb = row_bytes(s);
    CK(cudaMemcpyAsync(static_cast<uint8_t*>(full->val[0]) + (size_t)(kK + s->row0) * rb, alloc_rows(s, kK),
                       (size_t)s->g.H * rb, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return AM_OK;
}

am_status am_comm_unique_id(uint8_t* id_out) {
  if (!id_out) return AM_EINVAL;
  if (!nccl().ok) return AM_ENCCL;
  ncclUniqueId id;
  if (nccl().getUniqueId(&id) != ncclSuccess) return AM_ENCCL;
  static_assert(sizeof(id) == 128, "NCCL unique id size");
  memcpy(id_out, &id, sizeof id);
  return AM_OK;
}

am_status am_comm_init(am_ctx* ctx, uint32_t nranks, uint32_t rank, const uint8_t* id_in) {
  if (!ctx || !id_in || nranks == 0 || rank >= nranks) return AM_EINVAL;
  if (!nccl().ok) return fail(ctx, AM_ENCCL, "libnccl.so.2 not found");
  CK(cudaSetDevice(ctx->device));
  ncclUniqueId id;
  memcpy(&id, id_in, sizeof id);
  Comm* c = new Comm();
  c->nranks = nranks;
  c->rank = rank;
  ncclResult_t r = nccl().commInitRank(&c->comm, (int)nranks, id, (int)rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(ctx, AM_ENCCL, "ncclCommInitRank: %s", nccl().errorString(r));
  }
  comm_destroy(ctx->comm);
  ctx->comm = c;
  return AM_OK;
}

am_status am_comm_slab_rows(const am_ctx* ctx, uint32_t height, uint32_t* row0, uint32_t* row1) {
  if (!ctx || !row0 || !row1) return AM_EINVAL;
  const uint32_t n = ctx->comm ? ctx->comm->nranks : 1, r = ctx->comm ? ctx->comm->rank : 0;
  slab_rows(height, n, r, row0, row1);
  return AM_OK;
}

am_status am_comm_gather(am_ctx* ctx, am_grid* slab, am_grid* full) {
  if (!ctx || !slab || !full || !ctx->comm) return AM_EINVAL;
  if (full->slab || full->g.pitch != slab->g.pitch || full->g.H != slab->total_h)
    return fail(ctx, AM_EINVAL, "am_comm_gather: full grid does not match the slab");
  CK(cudaSetDevice(ctx->device));
  am_status st = adopt_full(ctx, full, slab);
  if (st) return st;
  Comm* cm = ctx->comm;
  const size_t rb = row_bytes(slab);
  NK(nccl().groupStart());
  for (uint32_t r = 0; r < cm->nranks; ++r) {
    uint32_t f, l;
    slab_rows(full->g.H, cm->nranks, r, &f, &l);
    uint8_t* dst = static_cast<uint8_t*>(full->val[0]) + (size_t)(kK + f) * rb;
    const void* srcp = r == cm->rank ? (const void*)alloc_rows(slab, kK) : (const void*)dst;
    NK(nccl().broadcast(srcp, dst, (size_t)(l - f) * rb, ncclUint8, (int)r, cm->comm, ctx->stream));
  }
  NK(nccl().groupEnd());
  CK(cudaStreamSynchronize(ctx->stream));
  return AM_OK;
}

}  // extern "C"
