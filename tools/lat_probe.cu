// Dependent-chain latency of the stencil's instructions on one warp (cycles per op).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat_probe tools/lat_probe.cu && /tmp/lat_probe
#include <cstdio>
#include <cstdint>

template <int OP>
__global__ void chain(uint32_t* out, long long* cyc, uint32_t seed, int n) {
  uint32_t x = seed + threadIdx.x, y = seed * 3, z = seed * 7;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (OP == 0) x = __vimax3_u16x2(x, y, z);
      if (OP == 1) x = __shfl_down_sync(0xffffffffu, x, 1) ^ y;
      if (OP == 2) x = (x & 0x7FFF7FFFu) | z;
      if (OP == 3) x = __shfl_down_sync(0xffffffffu, x, 1);
      if (OP == 4) { x = __vimax3_u16x2(x, y, z); x = __shfl_down_sync(0xffffffffu, x, 1); x = __vimax3_u16x2(x, y, z) & (z | 0x7FFF7FFFu); }
      if (OP == 5) x = x + y;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  uint32_t* o; long long* c;
  cudaMalloc(&o, 1024); cudaMalloc(&c, 8);
  const char* names[] = {"VIMNMX3 chain", "SHFL+LOP3 chain", "LOP3 chain", "SHFL chain", "layer chain (max3,shfl,max3&mask)", "IADD chain"};
  const int n = 1000;
  for (int op = 0; op < 6; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: chain<0><<<1, 32>>>(o, c, 5, n); break;
        case 1: chain<1><<<1, 32>>>(o, c, 5, n); break;
        case 2: chain<2><<<1, 32>>>(o, c, 5, n); break;
        case 3: chain<3><<<1, 32>>>(o, c, 5, n); break;
        case 4: chain<4><<<1, 32>>>(o, c, 5, n); break;
        case 5: chain<5><<<1, 32>>>(o, c, 5, n); break;
      }
      cudaDeviceSynchronize();
    }
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %.2f cycles per link\n", names[op], (double)h / (n * 16));
  }
  return 0;
}
