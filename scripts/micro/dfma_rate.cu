// DFMA issue-rate microbenchmark (FP64 vector pipe) on B200, to size the ULV factor's
// DFMA GEMMs against the FP64 peak.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
template <int NACC>
__global__ void k(double* out, int iters) {
  double acc[NACC];
  double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out;
  cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int threads : {256, 512, 1024}) {
    for (int blocks_per_sm : {1, 2, 4}) {
      if (threads * blocks_per_sm > 2048) continue;
      const int grid = 148 * blocks_per_sm;
      k<8><<<grid, threads>>>(out, 100);
      cudaEventRecord(e0);
      k<8><<<grid, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fl = 2.0 * 8 * (double)iters * grid * threads;
      printf("DFMA threads=%d blocks/SM=%d: %.2f TFLOP/s\n", threads, blocks_per_sm, fl / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
