#include <cuda_runtime.h>
#include <cstdio>
__global__ void body(cudaGraphConditionalHandle h, unsigned* cnt) {
  if (threadIdx.x == 0 && blockIdx.x == 0) { unsigned v = ++*cnt; if (v >= 100) cudaGraphSetConditional(h, 0); }
}
int main() {
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h; cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
  cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
  cudaGraphNode_t cn; cudaGraphAddNode(&cn, g, nullptr, 0, &cp);
  cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
  unsigned* cnt; cudaMalloc(&cnt, 4); cudaMemset(cnt, 0, 4);
  cudaGraphNodeParams kp = {cudaGraphNodeTypeKernel};
  void* args[] = {&h, &cnt};
  kp.kernel.func = (void*)body; kp.kernel.gridDim = dim3(592); kp.kernel.blockDim = dim3(128); kp.kernel.kernelParams = args;
  cudaGraphNode_t kn; cudaGraphAddNode(&kn, bodyg, nullptr, 0, &kp);
  cudaGraphExec_t ex; cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
  printf("inst %s\n", cudaGetErrorString(e));
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(cnt, 0, 4);
    cudaEventRecord(a, s); cudaGraphLaunch(ex, s); cudaEventRecord(b, s); cudaStreamSynchronize(s);
    float ms; cudaEventElapsedTime(&ms, a, b); unsigned hc; cudaMemcpy(&hc, cnt, 4, cudaMemcpyDeviceToHost);
    printf("100 iterations: %.3f ms (%.2f us each), cnt %u, err %s\n", ms, ms * 10, hc, cudaGetErrorString(cudaGetLastError()));
  }
}
