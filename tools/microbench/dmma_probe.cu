// FP64 tensor (mma.sync m8n8k4 f64, DMMA) vs DFMA issue rate on one B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 2) dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0;
  for (int t = 0; t < iters; ++t) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void __launch_bounds__(256, 2) dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double d[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) d[i] = i;
  for (int t = 0; t < iters; ++t) {
#pragma unroll
    for (int i = 0; i < 16; ++i) d[i] = fma(a, b, d[i]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += d[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out;
  cudaMalloc(&out, 148 * 2 * 256 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, blocks = 148 * 2, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    dmma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // each mma.sync m8n8k4: 8*8*4 = 256 FMA = 512 flop per warp instruction
    const double flop = double(blocks) * (threads / 32) * iters * 8 * 512.0;
    printf("DMMA m8n8k4: %.1f TFLOP/s\n", flop / ms / 1e9);
    dfma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double f2 = double(blocks) * threads * iters * 16 * 2.0;
    printf("DFMA: %.1f TFLOP/s\n", f2 / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
