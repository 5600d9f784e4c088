// ipc_probe.cu -- measures issue throughput (warp-instructions / cycle / SM) of the
// integer ops the stencil is built from, on the real B200.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ipc tools/ipc_probe.cu && /tmp/ipc
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

#define ILP 8
template <int OP>
__global__ void probe(uint32_t* out, int iters, long long* cyc) {
  uint32_t r[ILP];
  for (int i = 0; i < ILP; ++i) r[i] = threadIdx.x * 2654435761u + i * 97u;
  uint32_t a = blockIdx.x | 0x01000100u, b = 0x00FF00FFu ^ threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      const uint32_t n1 = r[(i + 1) % ILP], n2 = r[(i + 3) % ILP];
      if (OP == 0) r[i] = __vimax3_u16x2(r[i], n1, n2);
      if (OP == 1) r[i] = __vmaxu2(r[i], n1);
      if (OP == 2) { __half2 h = *reinterpret_cast<__half2*>(&r[i]); __half2 g = *reinterpret_cast<const __half2*>(&n1); h = __hmax2(h, g); r[i] = *reinterpret_cast<uint32_t*>(&h); }
      if (OP == 3) r[i] = (r[i] & (n1 | 0x7FFF7FFFu)) ^ n2;
      if (OP == 4) r[i] = r[i] + n1 + n2;
      if (OP == 5) r[i] = __byte_perm(r[i], n1, 0x5410);
      if (OP == 6) r[i] = r[i] * n1 + n2;
      if (OP == 7) r[i] = __shfl_down_sync(0xffffffffu, r[i], 1) + a;
      if (OP == 8) r[i] = __vimax3_u32(r[i], n1, n2);
      if (OP == 9) r[i] = __viaddmax_u16x2(r[i], n1, n2);
      // pipe-sharing probes: two different ops alternate; 4/clk/SM => separate pipes
      if (OP == 10) {
        if (i & 1) r[i] = __vimax3_u16x2(r[i], n1, n2);
        else { __half2 h = *reinterpret_cast<__half2*>(&r[i]); __half2 g = *reinterpret_cast<const __half2*>(&n1); h = __hmax2(h, g); r[i] = *reinterpret_cast<uint32_t*>(&h); }
      }
      if (OP == 11) r[i] = (i & 1) ? __vimax3_u16x2(r[i], n1, n2) : r[i] * n1 + n2;
      if (OP == 12) r[i] = (i & 1) ? __vimax3_u16x2(r[i], n1, n2) : (r[i] & (n1 | 0x7FFF7FFFu));
      if (OP == 13) {
        if (i & 1) r[i] = r[i] * n1 + n2;
        else { __half2 h = *reinterpret_cast<__half2*>(&r[i]); __half2 g = *reinterpret_cast<const __half2*>(&n1); h = __hmax2(h, g); r[i] = *reinterpret_cast<uint32_t*>(&h); }
      }
      if (OP == 14) r[i] = (i & 1) ? __vimax3_u16x2(r[i], n1, n2) : __byte_perm(r[i], n1, 0x5410);
      if (OP == 15) {
        if (i & 1) r[i] = __vimax3_u16x2(r[i], n1, n2);
        else { __half2 h = *reinterpret_cast<__half2*>(&r[i]); __half2 g = *reinterpret_cast<const __half2*>(&n1); h = __hfma2(h, g, h); r[i] = *reinterpret_cast<uint32_t*>(&h); }
      }
      if (OP == 16) r[i] = (r[i] & (n1 | 0x7FFF7FFFu));
      if (OP == 17) { float f = __uint_as_float(r[i]); f = fmaxf(f, __uint_as_float(n1)); r[i] = __float_as_uint(f); }
      if (OP == 18) { if (i & 1) r[i] = __vimax3_u16x2(r[i], n1, n2); else { float f = __uint_as_float(r[i]); f = fmaxf(f, __uint_as_float(n1)); r[i] = __float_as_uint(f); } }
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < ILP; ++i) s ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps_per_sm) {
  int sms = 148, threads = 32 * warps_per_sm, iters = 4096;
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, sms * threads * 4);
  cudaMalloc(&cyc, sms * 8);
  probe<OP><<<sms, threads>>>(out, 16, cyc);
  probe<OP><<<sms, threads>>>(out, iters, cyc);
  long long h[148];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double mean = 0; for (int i = 0; i < sms; ++i) mean += h[i]; mean /= sms;
  double winst = (double)iters * ILP * warps_per_sm;
  printf("%-22s warps/SM=%2d  warp-instr/clk/SM = %.3f\n", name, warps_per_sm, winst / mean);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {16}) {
    run<10>("VIMNMX3 + HMNMX2", w);
    run<11>("VIMNMX3 + IMAD", w);
    run<12>("VIMNMX3 + LOP3", w);
    run<13>("IMAD + HMNMX2", w);
    run<14>("VIMNMX3 + PRMT", w);
    run<15>("VIMNMX3 + HFMA2", w);
    run<16>("LOP3 (single and)", w);
    run<17>("FMNMX", w);
    run<18>("VIMNMX3 + FMNMX", w);
  }
  for (int w : {8}) {
    run<0>("VIMNMX3.U16x2", w);
    run<1>("VIMNMX.U16x2", w);
    run<2>("HMNMX2", w);
    run<3>("LOP3", w);
    run<4>("IADD3", w);
    run<5>("PRMT", w);
    run<6>("IMAD", w);
    run<7>("SHFL", w);
    run<8>("VIMNMX3.U32", w);
    run<9>("VIADDMNMX.U16x2", w);
  }
  return 0;
}
