#include <cuda_runtime.h>
#include <cstdio>
__global__ void body(cudaGraphConditionalHandle h, int* k, int n) {
  if (threadIdx.x == 0) { int v = ++(*k); cudaGraphSetConditional(h, v < n ? 1 : 0); }
}
int main() {
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
  cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
  cudaGraphNode_t cn; cudaGraphAddNode(&cn, g, nullptr, 0, &cp);
  cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
  int* k; cudaMalloc(&k, 4); cudaMemset(k, 0, 4);
  int n = 1000;
  void* args[] = {&h, &k, &n};
  cudaKernelNodeParams kp = {}; kp.func = (void*)body; kp.gridDim = 1; kp.blockDim = 32; kp.kernelParams = args;
  cudaGraphNode_t kn; cudaGraphAddKernelNode(&kn, bodyg, nullptr, 0, &kp);
  cudaGraphExec_t ge; cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
  printf("inst %s\n", cudaGetErrorString(e));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); e = cudaGraphLaunch(ge, 0); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int hk; cudaMemcpy(&hk, k, 4, cudaMemcpyDeviceToHost);
  printf("launch %s k=%d  %.2f us per iteration\n", cudaGetErrorString(e), hk, ms * 1e3 / hk);
  return 0;
}
