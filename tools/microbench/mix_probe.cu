// Probe: FADD (fma pipe) + 3-input min on float bit patterns (alu pipe) vs VIADDMNMX.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define N 32
template <int V>
__global__ void __launch_bounds__(256, 2) k(uint32_t* sink, long long* cyc, int iters, uint32_t seed) {
  uint32_t acc[N]; float x[N];
#pragma unroll
  for (int i = 0; i < N; ++i) { acc[i] = 0x7f000000u - i; x[i] = float((seed * (i + 1) + threadIdx.x) & 0xFFFFF); }
  float y = float(seed & 0xFFF), y2 = y + 3.f;
  uint32_t yi = seed, yi2 = seed + 7;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (V == 0) acc[i] = min(acc[i], __float_as_uint(x[i]) + yi);                   // VIADDMNMX
      if (V == 1) acc[i] = min(min(acc[i], __float_as_uint(x[i] + y)), __float_as_uint(x[i] + y2));  // 2 FADD + VIMNMX3
      if (V == 2) acc[i] = __float_as_uint(fminf(fminf(__uint_as_float(acc[i]), x[i] + y), x[i] + y2));  // FMNMX form
    }
    y += 1.f; y2 += 1.f; yi += 3; yi2 += 5;
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) s ^= acc[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  const int blocks = 296, threads = 256, iters = 20000;
  uint32_t* sink; long long* cyc; cudaMalloc(&sink, blocks * threads * 4); cudaMalloc(&cyc, blocks * 8);
  long long h[296];
  const char* names[] = {"viaddmnmx (1 instr/term)", "2xFADD + VIMNMX3 (1.5 instr/term)", "2xFADD + FMNMX3?"};
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      if (v == 0) k<0><<<blocks, threads>>>(sink, cyc, iters, 7);
      if (v == 1) k<1><<<blocks, threads>>>(sink, cyc, iters, 7);
      if (v == 2) k<2><<<blocks, threads>>>(sink, cyc, iters, 7);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0; for (int b = 0; b < blocks; ++b) mx = h[b] > mx ? h[b] : mx;
    double terms = double(iters) * N * (v == 0 ? 1 : 2) * threads * 2;  // per SM (2 CTAs)
    printf("%-36s %.1f terms/clk/SM\n", names[v], terms / mx);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
