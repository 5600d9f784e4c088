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
//  * peer memory (am_peer_*, one process per GPU or several on one GPU): the
//    boundary kernel stores a slab's first / last K rows straight into the
//    neighbours' halo inboxes through CUDA-IPC-mapped peer pointers (P2P
//    stores over NVLink / NVSwitch), the slot words follow with one small
//    peer copy, and the neighbour's stream waits on the writer's IPC event
//    (a stream-ordered dependency: no kernel ever spins on another rank, so
//    ranks sharing one GPU are safe).  A shared-memory counter per rank tells
//    a host that the peer's event record for an exchange has been issued.
//    No NCCL call and no collective sits on the per-block path.
//  * in-process groups on one device (am_slabs_*): device-to-device copies
//    on the shared stream.  They run the identical decomposition, so the
//    slab logic is tested on a single GPU against the oracle.
#include <dlfcn.h>
#include <fcntl.h>
#include <sched.h>
#include <nccl.h>
#include <sys/mman.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <new>

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
  bool chain_tiles_ok() const override {
    for (uint32_t r = 0; r + 1 < ctx->comm->nranks; ++r) {
      uint32_t a = 0, z = 0;
      slab_rows(g->total_h, ctx->comm->nranks, r, &a, &z);
      if ((z - a) % kTileRows) return false;
    }
    return true;
  }
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

// ---------------------------------------------------------------- peer-memory transport
//
// Inbox of a slab (cudaMalloc, exported with cudaIpcGetMemHandle), by exchange parity p:
//   rows from the slab above (its last kK rows)  -> from_up[p]   (kK rows x pitch x 4 B: room for 32-bit cells)
//   rows from the slab below (its first kK rows) -> from_dn[p]
//   slot words from above / below               -> words_up[p], words_dn[p] (kFlagSlots u32)
//   one word per rank for reductions            -> red[p][kPeerMaxRanks]
// Publish buffer: the slab's own rows for am_peer_gather (rows x pitch x 4 B).
constexpr uint32_t kPeerMaxRanks = 64;
constexpr uint32_t kPeerMagic = 0x41504545u;  // "EEPA"
enum { kEvX0, kEvX1, kEvA0, kEvA1, kEvD0, kEvD1, kPeerEvents };
enum { kChX, kChA, kChD, kPeerChannels };  // shm counters: exchanges, aux (reduce / publish), gather done

struct PeerBlob {
  uint32_t magic, rank_hint, pitch, rows;
  uint64_t token;
  cudaIpcMemHandle_t inbox, publish;
  cudaIpcEventHandle_t ev[kPeerEvents];
};
static_assert(sizeof(PeerBlob) <= AM_PEER_BLOB_BYTES, "peer blob size");

struct PeerLink {
  // local, exported
  uint8_t* inbox = nullptr;
  uint8_t* publish = nullptr;
  size_t halo_bytes = 0, inbox_bytes = 0, publish_bytes = 0;
  cudaEvent_t ev[kPeerEvents] = {};
  uint64_t token = 0;
  // connection
  bool connected = false;
  uint32_t nranks = 1, rank = 0;
  std::vector<uint8_t*> p_inbox, p_publish;          // per rank (own entry: local pointers)
  std::vector<std::vector<cudaEvent_t>> p_ev;        // per rank x kPeerEvents (own entry: local events)
  std::vector<uint32_t> row0, rows;                  // slab rows of every rank
  std::atomic<uint64_t>* shm = nullptr;              // nranks x kPeerChannels counters (64 B apart)
  size_t shm_bytes = 0;
  char shm_name[64] = {};
  uint64_t n[kPeerChannels] = {};                    // operations issued on each channel
  int device = 0;
  SlabDir* dir = nullptr;                            // device: every rank's published rows (peer traces)
  void* zero_row = nullptr;                          // device: one zero row (pitch x 4 B)

  size_t off_from_up(uint32_t p) const { return p * halo_bytes; }
  size_t off_from_dn(uint32_t p) const { return (2 + p) * halo_bytes; }
  size_t off_words_up(uint32_t p) const { return 4 * halo_bytes + p * kFlagSlots * 4; }
  size_t off_words_dn(uint32_t p) const { return 4 * halo_bytes + (2 + p) * kFlagSlots * 4; }
  size_t off_red(uint32_t p) const { return 4 * halo_bytes + 4 * kFlagSlots * 4 + p * kPeerMaxRanks * 4; }
  std::atomic<uint64_t>& counter(uint32_t r, int ch) { return shm[(r * kPeerChannels + ch) * 8]; }
};

void peer_destroy(PeerLink* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();
  for (uint32_t r = 0; r < p->p_inbox.size(); ++r) {
    if (r == p->rank) continue;
    if (p->p_inbox[r]) cudaIpcCloseMemHandle(p->p_inbox[r]);
    if (p->p_publish[r]) cudaIpcCloseMemHandle(p->p_publish[r]);
    for (cudaEvent_t e : p->p_ev[r])
      if (e) cudaEventDestroy(e);
  }
  for (cudaEvent_t e : p->ev)
    if (e) cudaEventDestroy(e);
  if (p->dir) cudaFree(p->dir);
  if (p->zero_row) cudaFree(p->zero_row);
  if (p->inbox) cudaFree(p->inbox);
  if (p->publish) cudaFree(p->publish);
  if (p->shm) munmap(p->shm, p->shm_bytes);
  if (p->shm && p->rank == 0 && p->shm_name[0]) shm_unlink(p->shm_name);
  (void)cudaGetLastError();
  delete p;
}

// Host side of "rank r has issued the record of its op number `target` on channel ch".
static am_status peer_await(am_ctx* ctx, PeerLink* p, uint32_t r, int ch, uint64_t target) {
  std::atomic<uint64_t>& c = p->counter(r, ch);
  const auto t0 = std::chrono::steady_clock::now();
  for (uint64_t spin = 0; c.load(std::memory_order_acquire) < target; ++spin) {
    if ((spin & 1023) == 1023) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
        return fail(ctx, AM_EINTERNAL, "peer transport: rank %u never reached op %llu on channel %d", r,
                    (unsigned long long)target, ch);
      sched_yield();
    }
  }
  return AM_OK;
}

// Record this rank's event for op `idx` on channel ch (event parity idx & 1) and announce it.
static am_status peer_signal(am_ctx* ctx, PeerLink* p, int ch, int ev0, uint64_t idx) {
  CK(cudaEventRecord(p->ev[ev0 + (idx & 1)], ctx->stream));
  p->counter(p->rank, ch).store(idx + 1, std::memory_order_release);
  return AM_OK;
}

// Make ctx's stream wait for rank r's op `idx` on channel ch.
static am_status peer_wait(am_ctx* ctx, PeerLink* p, uint32_t r, int ch, int ev0, uint64_t idx) {
  if (am_status st = peer_await(ctx, p, r, ch, idx + 1)) return st;
  CK(cudaStreamWaitEvent(ctx->stream, p->p_ev[r][ev0 + (idx & 1)], 0));
  return AM_OK;
}

struct PeerTransport final : Transport {
  am_ctx* ctx;
  am_grid* g;
  PeerLink* p;
  PeerTransport(am_ctx* c, am_grid* gg) : ctx(c), g(gg), p(gg->peer) {}
  bool has_up() const { return p->rank > 0; }
  bool has_dn() const { return p->rank + 1 < p->nranks; }
  uint32_t parity() const { return (uint32_t)(p->n[kChX] & 1); }
  void* boundary_dst(int side) override {
    if (side == 0) return has_up() ? p->p_inbox[p->rank - 1] + p->off_from_dn(parity()) : nullptr;
    return has_dn() ? p->p_inbox[p->rank + 1] + p->off_from_up(parity()) : nullptr;
  }
  // rows: copy this slab's boundary rows into the neighbours' inboxes (dense exchange; the tile exchange
  // stored them from the boundary kernel already); always the slot words; then signal, wait, consume
  am_status exchange_impl(bool rows_dense, bool rows_tiles) {
    const uint32_t q = parity();
    const uint64_t idx = p->n[kChX];
    const size_t rb = row_bytes(g), bytes = (size_t)kK * rb;
    uint8_t* cur = static_cast<uint8_t*>(g->val[rows_tiles ? 0 : g->cur]);
    const uint32_t H = g->g.H;
    if (has_up()) {
      uint8_t* dst = p->p_inbox[p->rank - 1];
      if (rows_dense)
        CK(cudaMemcpyAsync(dst + p->off_from_dn(q), cur + (size_t)kK * rb, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaMemcpyAsync(dst + p->off_words_dn(q), g->d_flags, kFlagSlots * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    if (has_dn()) {
      uint8_t* dst = p->p_inbox[p->rank + 1];
      if (rows_dense)
        CK(cudaMemcpyAsync(dst + p->off_from_up(q), cur + (size_t)H * rb, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaMemcpyAsync(dst + p->off_words_up(q), g->d_flags, kFlagSlots * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    if (am_status st = peer_signal(ctx, p, kChX, kEvX0, idx)) return st;
    if (has_up())
      if (am_status st = peer_wait(ctx, p, p->rank - 1, kChX, kEvX0, idx)) return st;
    if (has_dn())
      if (am_status st = peer_wait(ctx, p, p->rank + 1, kChX, kEvX0, idx)) return st;
    if (has_up()) {
      if (rows_dense || rows_tiles)
        CK(cudaMemcpyAsync(cur, p->inbox + p->off_from_up(q), bytes, cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaMemcpyAsync(g->d_flags + kFlagRecvUp, p->inbox + p->off_words_up(q), kFlagSlots * 4,
                         cudaMemcpyDeviceToDevice, ctx->stream));
    }
    if (has_dn()) {
      if (rows_dense || rows_tiles)
        CK(cudaMemcpyAsync(cur + (size_t)(kK + H) * rb, p->inbox + p->off_from_dn(q), bytes, cudaMemcpyDeviceToDevice,
                           ctx->stream));
      CK(cudaMemcpyAsync(g->d_flags + kFlagRecvDn, p->inbox + p->off_words_dn(q), kFlagSlots * 4,
                         cudaMemcpyDeviceToDevice, ctx->stream));
    }
    ++p->n[kChX];
    launch_flags_merge(g->d_flags, ctx->stream);
    ++ctx->launches;
    if (cudaError_t e = cudaPeekAtLastError()) return fail(ctx, AM_ECUDA, "flags merge: %s", cudaGetErrorString(e));
    return AM_OK;
  }
  am_status exchange() override { return exchange_impl(true, false); }
  am_status exchange_tiles() override { return exchange_impl(false, true); }
  am_status exchange_flags() override { return exchange_impl(false, false); }
  uint32_t span() const override { return p->nranks; }
  am_status reduce(std::vector<uint32_t*>& words, bool take_max) override {
    const uint64_t idx = p->n[kChA];
    const uint32_t q = (uint32_t)(idx & 1);
    for (uint32_t r = 0; r < p->nranks; ++r)
      CK(cudaMemcpyAsync(p->p_inbox[r] + p->off_red(q) + 4 * p->rank, words[0], 4, cudaMemcpyDeviceToDevice,
                         ctx->stream));
    if (am_status st = peer_signal(ctx, p, kChA, kEvA0, idx)) return st;
    for (uint32_t r = 0; r < p->nranks; ++r)
      if (r != p->rank)
        if (am_status st = peer_wait(ctx, p, r, kChA, kEvA0, idx)) return st;
    ++p->n[kChA];
    launch_peer_reduce(reinterpret_cast<const uint32_t*>(p->inbox + p->off_red(q)), p->nranks, take_max ? 1 : 0,
                       words[0], ctx->stream);
    ++ctx->launches;
    CK(cudaPeekAtLastError());
    return AM_OK;
  }
  bool host_combine() const override { return false; }
  bool lower_neighbour() const override { return has_dn(); }
  bool chain_tiles_ok() const override {
    for (uint32_t r = 0; r + 1 < p->nranks; ++r)
      if (p->rows[r] % kTileRows) return false;
    return true;
  }
};

Transport* make_peer_transport(am_ctx* ctx, am_grid* g) { return new PeerTransport(ctx, g); }

// Places a propagated slab's own rows into the full grid's field.
static am_status adopt_full(am_ctx* ctx, am_grid* full, const am_grid* like) {
  if (am_status jst = join_map(ctx, full)) return jst;  // the full grid's own field encoding
  am_status st = set_cell_bits(ctx, full, like->cell_bits);
  if (st) return st;
  full->cur = 0;
  full->plain_active = 0;
  full->have_map = 1;
  full->bits_map = 0;
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

am_status am_slab_rows(uint32_t height, uint32_t nranks, uint32_t rank, uint32_t* row0, uint32_t* row1) {
  if (!row0 || !row1 || nranks == 0 || rank >= nranks) return AM_EINVAL;
  slab_rows(height, nranks, rank, row0, row1);
  return AM_OK;
}

am_status am_peer_export(am_ctx* ctx, am_grid* g, uint8_t* blob) {
  if (!ctx || !g || !blob) return AM_EINVAL;
  if (!g->slab) return fail(ctx, AM_EINVAL, "am_peer_export: not a slab grid");
  CK(cudaSetDevice(ctx->device));
  peer_destroy(g->peer);
  g->peer = nullptr;
  PeerLink* p = new (std::nothrow) PeerLink();
  if (!p) return AM_EOOM;
  p->device = ctx->device;
  const size_t rb4 = (size_t)g->g.pitch * 4;
  p->halo_bytes = (size_t)kK * rb4;
  p->inbox_bytes = p->off_red(2);
  p->publish_bytes = (size_t)g->g.H * rb4;
  cudaError_t e = cudaMalloc(&p->inbox, p->inbox_bytes);
  if (!e) e = cudaMalloc(&p->publish, p->publish_bytes);
  if (!e) e = cudaMemset(p->inbox, 0, p->inbox_bytes);
  for (int i = 0; i < kPeerEvents && !e; ++i)
    e = cudaEventCreateWithFlags(&p->ev[i], cudaEventDisableTiming | cudaEventInterprocess);
  PeerBlob b{};
  b.magic = kPeerMagic;
  b.pitch = g->g.pitch;
  b.rows = g->g.H;
  {
    timespec ts{};
    clock_gettime(CLOCK_REALTIME, &ts);
    p->token = ((uint64_t)getpid() << 40) ^ (uint64_t)ts.tv_nsec ^ ((uint64_t)ts.tv_sec << 20) ^
               reinterpret_cast<uintptr_t>(p);
  }
  b.token = p->token;
  if (!e) e = cudaIpcGetMemHandle(&b.inbox, p->inbox);
  if (!e) e = cudaIpcGetMemHandle(&b.publish, p->publish);
  for (int i = 0; i < kPeerEvents && !e; ++i) e = cudaIpcGetEventHandle(&b.ev[i], p->ev[i]);
  if (e) {
    peer_destroy(p);
    (void)cudaGetLastError();
    return fail(ctx, e == cudaErrorMemoryAllocation ? AM_EOOM : AM_ECUDA, "am_peer_export: %s", cudaGetErrorString(e));
  }
  memset(blob, 0, AM_PEER_BLOB_BYTES);
  memcpy(blob, &b, sizeof b);
  g->peer = p;
  return AM_OK;
}

am_status am_peer_connect(am_ctx* ctx, am_grid* g, uint32_t nranks, uint32_t rank, const uint8_t* blobs) {
  if (!ctx || !g || !blobs || nranks == 0 || rank >= nranks || nranks > kPeerMaxRanks) return AM_EINVAL;
  PeerLink* p = g->peer;
  if (!p || p->connected) return fail(ctx, AM_EINVAL, "am_peer_connect: export this slab (once) first");
  uint32_t r0 = 0, r1 = 0;
  slab_rows(g->total_h, nranks, rank, &r0, &r1);
  if (r0 != g->row0 || r1 - r0 != g->g.H)
    return fail(ctx, AM_EINVAL, "am_peer_connect: slab rows [%u, %u) are not rank %u's share [%u, %u)", g->row0,
                g->row0 + g->g.H, rank, r0, r1);
  CK(cudaSetDevice(ctx->device));
  std::vector<PeerBlob> b(nranks);
  for (uint32_t r = 0; r < nranks; ++r) {
    memcpy(&b[r], blobs + (size_t)r * AM_PEER_BLOB_BYTES, sizeof(PeerBlob));
    if (b[r].magic != kPeerMagic || b[r].pitch != g->g.pitch)
      return fail(ctx, AM_EINVAL, "am_peer_connect: blob %u is not a slab of this grid", r);
  }
  if (b[rank].token != p->token) return fail(ctx, AM_EINVAL, "am_peer_connect: blob %u is not this slab's", rank);
  p->nranks = nranks;
  p->rank = rank;
  p->p_inbox.assign(nranks, nullptr);
  p->p_publish.assign(nranks, nullptr);
  p->p_ev.assign(nranks, std::vector<cudaEvent_t>(kPeerEvents, nullptr));
  p->row0.resize(nranks);
  p->rows.resize(nranks);
  for (uint32_t r = 0; r < nranks; ++r) {
    uint32_t a = 0, z = 0;
    slab_rows(g->total_h, nranks, r, &a, &z);
    p->row0[r] = a;
    p->rows[r] = z - a;
    if (r == rank) {
      p->p_inbox[r] = p->inbox;
      p->p_publish[r] = p->publish;
      for (int i = 0; i < kPeerEvents; ++i) p->p_ev[r][i] = p->ev[i];
      continue;
    }
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, b[r].inbox, cudaIpcMemLazyEnablePeerAccess);
    p->p_inbox[r] = static_cast<uint8_t*>(ptr);
    if (!e) e = cudaIpcOpenMemHandle(&ptr, b[r].publish, cudaIpcMemLazyEnablePeerAccess);
    if (!e) p->p_publish[r] = static_cast<uint8_t*>(ptr);
    for (int i = 0; i < kPeerEvents && !e; ++i) e = cudaIpcOpenEventHandle(&p->p_ev[r][i], b[r].ev[i]);
    if (e) {
      (void)cudaGetLastError();
      return fail(ctx, AM_ECUDA, "am_peer_connect: rank %u handles: %s", r, cudaGetErrorString(e));
    }
  }
  // host counters shared by the ranks (one node): named after rank 0's token
  snprintf(p->shm_name, sizeof p->shm_name, "/actmap_peer_%016llx", (unsigned long long)b[0].token);
  p->shm_bytes = (size_t)nranks * kPeerChannels * 64;
  const int fd = shm_open(p->shm_name, O_CREAT | O_RDWR, 0600);
  if (fd < 0) return fail(ctx, AM_EINTERNAL, "am_peer_connect: shm_open(%s) failed", p->shm_name);
  if (ftruncate(fd, (off_t)p->shm_bytes) != 0) {
    close(fd);
    return fail(ctx, AM_EINTERNAL, "am_peer_connect: ftruncate failed");
  }
  void* m = mmap(nullptr, p->shm_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (m == MAP_FAILED) return fail(ctx, AM_EINTERNAL, "am_peer_connect: mmap failed");
  p->shm = static_cast<std::atomic<uint64_t>*>(m);
  // the directory of every rank's published rows, for traces that read across slab edges
  {
    SlabDir d{};
    d.n = nranks;
    for (uint32_t r = 0; r < nranks; ++r) {
      d.row0[r] = p->row0[r];
      d.base[r] = p->p_publish[r];
    }
    d.row0[nranks] = g->total_h;
    cudaError_t e = cudaMalloc(&p->zero_row, (size_t)g->g.pitch * 4);
    if (!e) e = cudaMemset(p->zero_row, 0, (size_t)g->g.pitch * 4);
    d.zero = p->zero_row;
    if (!e) e = cudaMalloc(&p->dir, sizeof(SlabDir));
    if (!e) e = cudaMemcpy(p->dir, &d, sizeof(SlabDir), cudaMemcpyHostToDevice);
    if (e) {
      (void)cudaGetLastError();
      return fail(ctx, AM_ECUDA, "am_peer_connect: slab directory: %s", cudaGetErrorString(e));
    }
  }
  p->connected = true;
  return AM_OK;
}

namespace {
// Every rank publishes its rows (after the peers finished reading its previous publish) and waits for
// all the others' publishes: afterwards every rank's publish buffer holds its slab at the final layer.
am_status peer_publish(am_ctx* ctx, am_grid* slab, PeerLink* p) {
  const size_t rb = (size_t)slab->g.pitch * (slab->cell_bits / 8);
  const uint64_t ia = p->n[kChA], id = p->n[kChD];
  am_status st;
  if (id > 0)
    for (uint32_t r = 0; r < p->nranks; ++r)
      if (r != p->rank && (st = peer_wait(ctx, p, r, kChD, kEvD0, id - 1))) return st;
  CK(cudaMemcpyAsync(p->publish, static_cast<uint8_t*>(slab->val[slab->cur]) + (size_t)kK * rb,
                     (size_t)slab->g.H * rb, cudaMemcpyDeviceToDevice, ctx->stream));
  if ((st = peer_signal(ctx, p, kChA, kEvA0, ia))) return st;
  for (uint32_t r = 0; r < p->nranks; ++r)
    if (r != p->rank && (st = peer_wait(ctx, p, r, kChA, kEvA0, ia))) return st;
  ++p->n[kChA];
  return AM_OK;
}
// this rank is done reading the peers' publish buffers
am_status peer_release(am_ctx* ctx, PeerLink* p) {
  am_status st = peer_signal(ctx, p, kChD, kEvD0, p->n[kChD]);
  if (!st) ++p->n[kChD];
  return st;
}
}  // namespace

am_status am_peer_gather(am_ctx* ctx, am_grid* slab, am_grid* full) {
  if (!ctx || !slab || !full) return AM_EINVAL;
  PeerLink* p = slab->peer;
  if (!p || !p->connected) return fail(ctx, AM_EINVAL, "am_peer_gather: slab not connected");
  if (full->slab || full->g.pitch != slab->g.pitch || full->g.H != slab->total_h)
    return fail(ctx, AM_EINVAL, "am_peer_gather: full grid does not match the slab");
  CK(cudaSetDevice(ctx->device));
  am_status st = adopt_full(ctx, full, slab);
  if (st) return st;
  if ((st = peer_publish(ctx, slab, p))) return st;
  const size_t rb = row_bytes(slab);
  for (uint32_t r = 0; r < p->nranks; ++r)  // peer-to-peer copies of every slab into the full field
    CK(cudaMemcpyAsync(static_cast<uint8_t*>(full->val[0]) + (size_t)(kK + p->row0[r]) * rb, p->p_publish[r],
                       (size_t)p->rows[r] * rb, cudaMemcpyDeviceToDevice, ctx->stream));
  if ((st = peer_release(ctx, p))) return st;
  CK(cudaStreamSynchronize(ctx->stream));
  return AM_OK;
}

am_status am_peer_trace_paths_device(am_ctx* ctx, am_grid* slab, const uint32_t* d_tgt, uint64_t n, uint32_t method,
                                     uint64_t seed, uint64_t* d_offsets, uint32_t* d_pts, uint64_t cap,
                                     int32_t* d_status) {
  if (!ctx || !slab || !d_offsets || (n && (!d_tgt || !d_status))) return AM_EINVAL;
  PeerLink* p = slab->peer;
  if (!p || !p->connected) return fail(ctx, AM_EINVAL, "am_peer_trace_paths_device: slab not connected");
  if (!slab->have_map || slab->plain_active) return fail(ctx, AM_EINVAL, "no propagated map");
  if (method > 1) return fail(ctx, AM_EINVAL, "bad method");
  if (!d_pts && cap) return fail(ctx, AM_EINVAL, "null point buffer");
  CK(cudaSetDevice(ctx->device));
  am_status st = peer_publish(ctx, slab, p);
  if (st) return st;
  MapView m{};
  m.g = slab->g;
  m.g.H = slab->total_h;                // grid coordinates of the whole map
  m.g.rows = slab->total_h + 2 * m.g.pad;
  m.val = nullptr;
  m.dir = p->dir;
  m.cell_bits = slab->cell_bits;
  m.layers = slab->computed;  // point counts are rollback invariant (the same on every rank)
  if (n) {
    if ((st = trace_scratch(ctx, slab, n))) return st;
    launch_path_counts(m, d_tgt, n, (int)method, seed, slab->d_counts, d_status, ctx->stream);
    CKL();
    launch_scan(slab->d_counts, n, d_offsets, ctx->stream);
    CKL();
    launch_trace(m, d_tgt, n, (int)method, seed, d_offsets, d_pts, d_status, ctx->stream, cap,
                 reinterpret_cast<uint32_t*>(slab->d_counts), slab->d_sched, ctx->sms);
    CKL();
  }
  return peer_release(ctx, p);
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
