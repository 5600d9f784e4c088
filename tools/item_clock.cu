// Per-iteration clock of one active-tile work item (2 tiles, one warp alone on the GPU).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include \
//        -DAM_DEBUG_CLOCK -o /tmp/item_clock tools/item_clock.cu && /tmp/item_clock
#include "../paper_2004_00540_b200/csrc/stencil.cu"

#include <vector>

int main() {
  using namespace am;
  const uint32_t W = 4096, H = 4096;
  Geo g = make_geo(W, H, 148 * 12);
  const size_t cells = (size_t)g.rows * g.pitch;
  uint16_t *f0, *f1;
  uint8_t *srcmask, *rowsrc;
  uint32_t *state, *list, *count, *flag;
  uint16_t* front;
  cudaMalloc(&f0, cells * 2); cudaMalloc(&f1, cells * 2);
  cudaMalloc(&srcmask, cells); cudaMalloc(&rowsrc, g.rows);
  cudaMalloc(&state, g.ntiles() * 4); cudaMalloc(&front, g.ntiles() * 2);
  cudaMalloc(&list, 64); cudaMalloc(&count, 4); cudaMalloc(&flag, 8);
  cudaMemset(f0, 0x80, cells * 2);  // every cell free-uncovered-ish (0x8080)
  cudaMemset(f1, 0, cells * 2);
  cudaMemset(srcmask, 0, cells); cudaMemset(rowsrc, 0, g.rows);
  cudaMemset(state, 0, g.ntiles() * 4); cudaMemset(flag, 0xFF, 4); cudaMemset(flag + 1, 0, 4);
  uint32_t h_list[2] = {(5u << 16) | 20u, (9u << 16) | 40u}, n = 2;
  cudaMemcpy(list, h_list, 8, cudaMemcpyHostToDevice);
  cudaMemcpy(count, &n, 4, cudaMemcpyHostToDevice);
  FlagSink sink{flag, flag + 1, nullptr};
  for (int rep = 0; rep < 3; ++rep) {
    launch_block_tiles(g, 16, 1, f0, f1, srcmask, rowsrc, list, count, front, state, 0, sink, 0);
    cudaDeviceSynchronize();
    long long c[64];
    cudaMemcpyFromSymbol(c, am_dbg_clock, sizeof c);
    const int iters = (kTileRows + 2 * kK) / 2;
    printf("rep %d: %s; total %lld cycles; prologue+iter1 %lld; iterations:", rep, cudaGetErrorString(cudaGetLastError()),
           c[iters] - c[0], c[1] - c[0]);
    for (int i = 1; i < iters; ++i) printf(" %lld", c[i + 1] - c[i]);
    printf("\n");
  }
  return 0;
}
