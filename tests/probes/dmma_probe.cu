// Probe: fp64 throughput of B200 through (a) mma.sync.m8n8k4.f64 (DMMA) and (b) plain DFMA, to choose the inner
// product of the LDL' Schur-complement kernel.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3 + 1.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out, int iters) {
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = i;
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3 + 1.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(a, b, c[i]);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 256 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int blocks_per_sm = 1; blocks_per_sm <= 8; blocks_per_sm *= 2) {
    const int grid = 148 * blocks_per_sm, iters = 20000;
    float ms;
    k_dmma<<<grid, 256>>>(out, 100);
    cudaEventRecord(e0);
    k_dmma<<<grid, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl_mma = (double)grid * 8 /*warps*/ * iters * 8 /*mma*/ * 512.0;
    printf("DMMA  %d CTA/SM: %.2f ms  %.2f TFLOP/s\n", blocks_per_sm, ms, fl_mma / ms / 1e9);
    k_dfma<<<grid, 256>>>(out, 100);
    cudaEventRecord(e0);
    k_dfma<<<grid, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl_fma = (double)grid * 256 * iters * 16 * 2.0;
    printf("DFMA  %d CTA/SM: %.2f ms  %.2f TFLOP/s\n", blocks_per_sm, ms, fl_fma / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
