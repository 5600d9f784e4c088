// Spread vs clustered item reads: each warp reads 48 rows x 256 B at a 46 KB
// row pitch (one active-tile item) starting at a base that is either packed
// (neighbouring items) or spread over a 2 GB buffer.  Separates address-spread
// (TLB / DRAM page) cost from the compute of the tile kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tlb_probe tools/tlb_probe.cu && /tmp/tlb_probe
#include <cstdio>
#include <cstdint>

__global__ void items(const uint4* __restrict__ buf, size_t pitch16, const size_t* __restrict__ base, int n, uint4* out) {
  const int w = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= n) return;
  const uint4* p = buf + base[w] + (lane & 15);
  uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll 8
  for (int r = 0; r < 48; ++r) {
    const uint4 v = __ldcg(p + r * pitch16);
    acc.x ^= v.x; acc.y += v.y;
  }
  if (acc.x == 0x12345 && acc.y == 7) out[w] = acc;
}

int main() {
  const size_t bytes = 2ull << 30, pitch = 23232 * 2, pitch16 = pitch / 16;
  uint4* buf; uint4* out; size_t* d_base;
  cudaMalloc(&buf, bytes); cudaMalloc(&out, 1 << 20); cudaMemset(buf, 1, bytes);
  const int ns[] = {1, 296, 1184, 4736};
  size_t* h = new size_t[8192];
  cudaMalloc(&d_base, 8192 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const size_t rows = bytes / pitch - 64;
  for (int mode = 0; mode < 3; ++mode) {
    for (int k = 0; k < 4; ++k) {
      const int n = ns[k];
      for (int i = 0; i < n; ++i) {
        size_t row, col;
        if (mode == 0) { row = (i / 207) * 32; col = (i % 207) * 224; }                   // adjacent items
        else if (mode == 1) { uint64_t x = (uint64_t)i * 7919; row = ((x / 207) * 32) % (rows / 2); col = (x % 207) * 224; }  // spread ~1 GB
        else { uint64_t x = (uint64_t)i * 2654435761u; row = (x % (rows - 48)); col = ((x >> 20) % 207) * 224; }  // random rows
        h[i] = (row * pitch + col) / 16;
      }
      cudaMemcpy(d_base, h, n * 8, cudaMemcpyHostToDevice);
      items<<<(n + 3) / 4, 128>>>(buf, pitch16, d_base, n, out);
      cudaEventRecord(a);
      for (int r = 0; r < 20; ++r) items<<<(n + 3) / 4, 128>>>(buf, pitch16, d_base, n, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("%-9s items %5d: %8.2f us/launch\n", mode == 0 ? "adjacent" : mode == 1 ? "spread" : "random", n, ms * 1000 / 20);
    }
  }
  return 0;
}
