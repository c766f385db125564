// Does programmatic dependent launch shorten a chain of small dependent kernels captured in a
// CUDA graph?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 pdl_graph.cu -o pdl_graph
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step(const double* in, double* out, int n, int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i] * 1.0000001 + 1.0;
}

int main() {
  const int n = 64 * 256, K = 24;
  double *a, *b;
  cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8);
  cudaMemset(a, 0, n * 8); cudaMemset(b, 0, n * 8);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int k = 0; k < K; ++k) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(64); cfg.blockDim = dim3(256); cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = pdl;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, step, (const double*)((k & 1) ? b : a), (k & 1) ? a : b, n, pdl);
    }
    cudaStreamEndCapture(s, &g);
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return 1; }
    for (int w = 0; w < 10; ++w) cudaGraphLaunch(ge, s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 200; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    printf("pdl=%d: %.3f us per kernel (graph of %d dependent kernels)\n", pdl, 1000.0 * ms / (200.0 * K), K);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
