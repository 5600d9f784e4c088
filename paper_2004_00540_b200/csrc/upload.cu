// upload.cu -- occupancy upload from host memory, packed to 1 bit per cell on the way.
//
// GridMap holds one byte per cell (grid.hpp:56), and a C4 grid is 537 MB: copied as bytes it is ~10 ms of
// PCIe, half of an end-to-end solve.  Only "obstacle or not" matters (grid.hpp:20, nonzero = obstacle), so
// host worker threads pack the caller's rows to 32-cell words (pack.cpp: AVX-512BW / AVX2 / SSE2
// compares) into a pinned staging buffer, chunk by chunk, and each chunk is copied (1/8 of the bytes)
// and expanded back to the dense byte form on the device while the workers pack the next ones.  The packed
// words stay on the device for the grid's free plane (bits.cu), so the bytes are read once.  From a pinned
// source a share of the rows crosses as raw bytes beside the workers and is packed on the device.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <functional>
#include <mutex>
#include <thread>

#include "am_host.hpp"

namespace am {

// ---- host worker pool (one per context; the calling thread packs too) ----
struct HostPool {
  std::vector<std::thread> th;
  std::mutex mu;
  std::condition_variable cv, idle_cv;
  std::function<void(int)> fn;
  std::atomic<int> next{0};
  int n = 0;
  uint64_t gen = 0;
  int busy = 0;
  bool stop = false;

  explicit HostPool(int workers) {
    for (int i = 0; i < workers; ++i) th.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> l(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : th) t.join();
  }
  void drain() {  // take items until none are left
    for (int k; (k = next.fetch_add(1)) < n;) fn(k);
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(mu);
        cv.wait(l, [&] { return stop || gen != seen; });
        if (stop) return;
        seen = gen;
        ++busy;
      }
      drain();
      {
        std::lock_guard<std::mutex> l(mu);
        if (--busy == 0) idle_cv.notify_all();
      }
    }
  }
  // Starts items 0 .. items-1 on the workers (returns at once).
  void start(int items, std::function<void(int)> f) {
    std::lock_guard<std::mutex> l(mu);
    fn = std::move(f);
    n = items;
    next.store(0);
    ++gen;
    cv.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> l(mu);
    idle_cv.wait(l, [&] { return busy == 0; });
  }
};

void host_pool_destroy(HostPool* p) { delete p; }

static int pool_workers() {
  if (const char* e = getenv("AM_HOST_THREADS")) return std::max(0, atoi(e) - 1);
  const unsigned hw = std::thread::hardware_concurrency();
  return (int)std::min(31u, hw > 1 ? hw - 1 : 0u);
}

// pack.cpp
void pack_rows(const uint8_t* occ, uint32_t W, uint32_t r0, uint32_t r1, uint32_t pw, uint32_t* out);
int pack_isa();  // 0 SSE2, 1 AVX2, 2 AVX-512BW

namespace {
// Dense bytes (0 free / 1 obstacle) of packed rows [r0, r1): one warp per 32 packed words (1024 cells),
// each word's 32 bytes written by the 32 lanes (coalesced).
__global__ void k_unpack_occ(const uint32_t* __restrict__ packed, uint32_t W, uint32_t pw, uint32_t r0, uint32_t r1,
                             uint8_t* __restrict__ occ) {
  const int lane = threadIdx.x & 31;
  const uint32_t r = r0 + blockIdx.y;
  const uint32_t w0 = (blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * 32;
  if (r >= r1 || w0 >= pw) return;  // warp-uniform
  const uint32_t mine = w0 + lane < pw ? __ldg(packed + (size_t)r * pw + w0 + lane) : 0u;
  uint8_t* row = occ + (size_t)r * W;
#pragma unroll 4
  for (int k = 0; k < 32; ++k) {
    const uint32_t v = __shfl_sync(0xffffffffu, mine, k);
    const uint32_t c = (w0 + k) * 32 + lane;
    if (c < W) row[c] = (uint8_t)((v >> lane) & 1u);
  }
}
// Packed rows [r0, r1) from dense bytes already on the device (the raw-copied share of an upload): a warp
// per 32 words of a row, 32 ballots over coalesced byte loads.
__global__ void k_pack_occ(const uint8_t* __restrict__ occ, uint32_t W, uint32_t pw, uint32_t r0, uint32_t r1,
                           uint32_t* __restrict__ packed) {
  const int lane = threadIdx.x & 31;
  const uint32_t r = r0 + blockIdx.y;
  const uint32_t w0 = (blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * 32;
  if (r >= r1 || w0 >= pw) return;  // warp-uniform
  const uint8_t* row = occ + (size_t)r * W;
  uint32_t mine = 0;
#pragma unroll 8
  for (int k = 0; k < 32; ++k) {
    const uint32_t c = (w0 + k) * 32 + lane;
    const uint32_t obst = __ballot_sync(0xffffffffu, c < W && row[c] != 0);
    if (lane == k) mine = obst;
  }
  if (w0 + lane < pw) packed[(size_t)r * pw + w0 + lane] = mine;
}
}  // namespace

// Host occupancy rows [0, H) (W bytes each) -> d_occ (dense bytes) and ctx->d_pack (packed words, pw per
// row, kept for the free plane).  Enqueued on ctx->stream; returns once every chunk is packed and its copy
// enqueued (the staging buffer stays in use until the stream reaches the copies: callers synchronise).
am_status upload_occupancy_packed(am_ctx* ctx, const uint8_t* occ, uint32_t W, uint32_t H, uint8_t* d_occ) {
  const uint32_t pw = (W + 31) / 32;
  const size_t bytes = (size_t)pw * H * 4;
  if (ctx->h_pack_cap < bytes) {
    if (ctx->h_pack) cudaFreeHost(ctx->h_pack);
    ctx->h_pack = nullptr;
    ctx->h_pack_cap = 0;
    CK(cudaHostAlloc(&ctx->h_pack, bytes, cudaHostAllocDefault));
    ctx->h_pack_cap = bytes;
  }
  if (ctx->d_pack_cap < bytes) {
    am::dfree(ctx, ctx->d_pack);
    ctx->d_pack = nullptr;
    ctx->d_pack_cap = 0;
    CK(am::dmalloc(ctx, &ctx->d_pack, bytes));
    ctx->d_pack_cap = bytes;
  }
  if (!ctx->hpool) ctx->hpool = new HostPool(pool_workers());
  HostPool& pool = *ctx->hpool;
  const int threads = (int)pool.th.size() + 1;
  // A pinned source lets the copy engine take a share of the rows as raw bytes (packed on the device
  // afterwards) while the host workers pack the rest (AM_RAW_SHARE: the share in percent).  It pays while
  // the packing is instruction-bound (SSE2 / AVX2: 20%); with AVX-512 the workers alone reach the host's
  // memory bandwidth and a raw share only competes for it (default 0).
  uint32_t raw_rows = 0;
  {
    cudaPointerAttributes at{};
    const char* v = getenv("AM_RAW_SHARE");
    const int share = v ? std::max(0, std::min(100, atoi(v))) : pack_isa() == 2 ? 0 : 20;
    if (share && cudaPointerGetAttributes(&at, occ) == cudaSuccess && at.type == cudaMemoryTypeHost)
      raw_rows = (uint32_t)((uint64_t)H * share / 100);
    (void)cudaGetLastError();
  }
  cudaStream_t s = ctx->stream;
  if (raw_rows) {
    if (!ctx->copy_stream) CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    if (!ctx->copy_ev[0]) CK(cudaEventCreateWithFlags(&ctx->copy_ev[0], cudaEventDisableTiming));
    CK(cudaEventRecord(ctx->copy_ev[0], s));  // d_occ / d_pack are free to overwrite (stream order)
    CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_ev[0], 0));
    CK(cudaMemcpyAsync(d_occ, occ, (size_t)raw_rows * W, cudaMemcpyHostToDevice, ctx->copy_stream));
    for (uint32_t r0 = 0; r0 < raw_rows; r0 += 65535) {  // grid.y limit
      const uint32_t r1 = std::min(raw_rows, r0 + 65535);
      const dim3 grid((pw + 32 * 8 - 1) / (32 * 8), r1 - r0);
      k_pack_occ<<<grid, 256, 0, ctx->copy_stream>>>(d_occ, W, pw, r0, r1, ctx->d_pack);
      ++ctx->launches;
      CK(cudaPeekAtLastError());
    }
    CK(cudaEventRecord(ctx->copy_ev[0], ctx->copy_stream));
    ctx->h2d_bytes += (size_t)raw_rows * W;
  }
  const uint32_t HP = H - raw_rows;  // rows the host workers pack: [raw_rows, H)
  const uint32_t chunks = std::max(1u, std::min<uint32_t>(std::max(HP, 1u), (uint32_t)threads * 4));
  const uint32_t rows_per = (std::max(HP, 1u) + chunks - 1) / chunks;
  const uint32_t nch = HP ? (HP + rows_per - 1) / rows_per : 0;
  std::vector<std::atomic<int>> ready(nch);
  for (auto& a : ready) a.store(0);
  uint32_t* hp = ctx->h_pack;
  pool.start((int)nch, [&](int k) {
    const uint32_t r0 = raw_rows + (uint32_t)k * rows_per, r1 = std::min(H, r0 + rows_per);
    pack_rows(occ, W, r0, r1, pw, hp + (size_t)r0 * pw);
    ready[k].store(1, std::memory_order_release);
  });
  am_status st = AM_OK;
  for (uint32_t k = 0; k < nch; ++k) {
    // the calling thread packs too, then enqueues the chunks in order as they complete
    while (!ready[k].load(std::memory_order_acquire)) {
      const int j = pool.next.fetch_add(1);
      if (j < (int)nch) {
        const uint32_t r0 = raw_rows + (uint32_t)j * rows_per, r1 = std::min(H, r0 + rows_per);
        pack_rows(occ, W, r0, r1, pw, hp + (size_t)r0 * pw);
        ready[j].store(1, std::memory_order_release);
      } else {
        std::this_thread::yield();
      }
    }
    if (st) continue;
    const uint32_t r0 = raw_rows + k * rows_per, r1 = std::min(H, r0 + rows_per);
    cudaError_t e = cudaMemcpyAsync(ctx->d_pack + (size_t)r0 * pw, hp + (size_t)r0 * pw, (size_t)(r1 - r0) * pw * 4,
                                    cudaMemcpyHostToDevice, s);
    if (!e) {
      const dim3 grid((pw + 32 * 8 - 1) / (32 * 8), r1 - r0);
      k_unpack_occ<<<grid, 256, 0, s>>>(ctx->d_pack, W, pw, r0, r1, d_occ);
      ++ctx->launches;
      e = cudaPeekAtLastError();
    }
    if (e) st = fail(ctx, AM_ECUDA, "occupancy upload: %s", cudaGetErrorString(e));
  }
  pool.wait();  // `ready` and the job live on this frame
  if (raw_rows && !st) {
    const cudaError_t e = cudaStreamWaitEvent(s, ctx->copy_ev[0], 0);  // the raw share is copied and packed
    if (e) st = fail(ctx, AM_ECUDA, "occupancy upload: %s", cudaGetErrorString(e));
  }
  ctx->h2d_bytes += (size_t)(H - raw_rows) * pw * 4;
  ctx->pack_rows = H;
  ctx->pack_w = W;
  return st;
}

}  // namespace am
