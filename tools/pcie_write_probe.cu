// Posted-write bandwidth from the GPU into pinned (device-mapped) host memory vs the copy engine:
// 47 MB (the C4 paths) written by W warps in 256 B (8 B / lane) or 512 B (16 B / lane) warp stores.
#include <cuda_runtime.h>
#include <cstdio>
template <typename T>
__global__ void k_write(T* out, size_t n_per_warp, int stride_warps) {
  const size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const size_t nw = (size_t)gridDim.x * blockDim.x / 32;
  for (size_t i = 0; i < n_per_warp; ++i) {
    const size_t chunk = stride_warps ? i * nw + w : w * n_per_warp + i;  // interleaved or contiguous per warp
    T v{};
    out[chunk * 32 + lane] = v;
  }
}
int main() {
  const size_t bytes = 47395968;
  void* h; cudaHostAlloc(&h, bytes * 2, cudaHostAllocMapped);
  void* d; cudaMalloc(&d, bytes * 2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("copy engine D2H: %.3f ms %.1f GB/s\n", ms, bytes / ms / 1e6);
  }
  for (int warps : {296, 592, 1184, 2368, 4736}) {
    for (int wide = 0; wide < 2; ++wide) {
      for (int inter = 0; inter < 2; ++inter) {
        const size_t chunk_bytes = wide ? 512 : 256;
        const size_t chunks = bytes / chunk_bytes, per = chunks / warps;
        const int blocks = warps / 4;
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(a);
          if (wide) k_write<uint4><<<blocks, 128>>>((uint4*)h, per, inter);
          else k_write<uint2><<<blocks, 128>>>((uint2*)h, per, inter);
          cudaEventRecord(b); cudaEventSynchronize(b);
          cudaEventElapsedTime(&ms, a, b);
        }
        printf("warps %5d %s %s: %.3f ms %.1f GB/s\n", warps, wide ? "16B/lane" : " 8B/lane",
               inter ? "interleaved" : "contiguous ", ms, per * warps * chunk_bytes / ms / 1e6);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
