// DMMA.8x8x4 issue-rate microbenchmark: how many warps per SMSP and independent accumulator
// chains are needed to saturate the FP64 tensor pipe on B200 (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NACC, bool LDSB>
__global__ void k(double* out, int iters) {
  __shared__ double sb[64 * 36];
  for (int i = threadIdx.x; i < 64 * 36; i += blockDim.x) sb[i] = 1e-3 * i;
  __syncthreads();
  double acc[NACC][2];
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      double bv = LDSB ? sb[((it & 7) * 4 + (lane & 3)) * 36 + i * 8 % 32 + (lane >> 2)] : b;
      dmma(acc[i][0], acc[i][1], a, bv);
    }
  }
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NACC, bool LDSB>
void run(int warps_per_cta, int ctas_per_sm) {
  int nsm = 148, iters = 2000;
  double* o;
  cudaMalloc(&o, 148 * 32 * 1024 * 8);
  int grid = nsm * ctas_per_sm, thr = 32 * warps_per_cta;
  k<NACC, LDSB><<<grid, thr>>>(o, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<NACC, LDSB><<<grid, thr>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 256 * NACC * (double)iters * grid * warps_per_cta;
  printf("NACC=%2d LDSB=%d warps/CTA=%2d CTAs/SM=%d -> %.2f TFLOP/s (err=%s)\n", NACC, (int)LDSB,
         warps_per_cta, ctas_per_sm, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
}
int main() {
  run<8, false>(4, 1); run<8, false>(8, 1); run<8, false>(16, 1); run<8, false>(32, 1);
  run<16, false>(8, 1); run<16, false>(16, 1);
  run<34, false>(8, 1); run<34, false>(16, 1);
  run<34, true>(8, 1); run<34, true>(16, 1);
  run<17, true>(8, 1); run<17, true>(16, 1);
  run<4, false>(16, 1); run<2, false>(16, 1); run<1, false>(32, 1);
  return 0;
}
