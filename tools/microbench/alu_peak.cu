// ALU-pipe throughput microbenchmark for the semiring inner-loop instructions on sm_100a.
// Measures per-SM per-clock issue rates (clock64 inside the block) so the result is
// independent of the DVFS clock; prints one line per variant.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NACC 32
#define ITERS 4096

template <int V>
__global__ void __launch_bounds__(256) bench(uint32_t* out, long long* cyc, uint32_t seed) {
  uint32_t acc[NACC], x[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) { acc[i] = seed * (i + 3) + threadIdx.x; x[i] = seed ^ (i * 977 + threadIdx.x); }
  uint32_t y = seed + threadIdx.x, y2 = seed * 7 + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
    if (V == 0) {            // VIADDMNMX: one per term
#pragma unroll
      for (int i = 0; i < NACC; i++) acc[i] = min(acc[i], x[i] + y);
    } else if (V == 1) {     // 2 adds + 3-input min per 2 terms
#pragma unroll
      for (int i = 0; i < NACC; i++) acc[i] = min(min(acc[i], x[i] + y), x[i] + y2);
    } else if (V == 2) {     // signed max-plus
#pragma unroll
      for (int i = 0; i < NACC; i++) acc[i] = (uint32_t)max((int)acc[i], (int)(x[i] + y));
    } else if (V == 3) {     // FFMA
#pragma unroll
      for (int i = 0; i < NACC; i++) acc[i] = __float_as_uint(fmaf(__uint_as_float(x[i]), __uint_as_float(y), __uint_as_float(acc[i])));
    } else if (V == 4) {     // plain IADD3 (alu) dependency-free
#pragma unroll
      for (int i = 0; i < NACC; i++) acc[i] = acc[i] + x[i] + y;
    }
    y += 0x9e3779b9u; y2 += 0x7f4a7c15u;
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// int64 accumulate of int32 products (IMAD.WIDE) and int64 min-plus (reference SEMIRING_MINPLUS dtype)
template <int V>
__global__ void __launch_bounds__(256) bench64(unsigned long long* out, long long* cyc, uint32_t seed) {
  long long acc[NACC / 2]; int x[NACC / 2];
#pragma unroll
  for (int i = 0; i < NACC / 2; i++) { acc[i] = seed * (i + 3) + threadIdx.x; x[i] = seed ^ (i * 977 + threadIdx.x); }
  int y = seed + threadIdx.x;
  long long y64 = (long long)seed * 12345 + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
    if (V == 0) {
#pragma unroll
      for (int i = 0; i < NACC / 2; i++) acc[i] += (long long)x[i] * y;
    } else if (V == 1) {
#pragma unroll
      for (int i = 0; i < NACC / 2; i++) { long long s = (long long)x[i] + y64; acc[i] = acc[i] < s ? acc[i] : s; }
    } else if (V == 2) {
#pragma unroll
      for (int i = 0; i < NACC / 2; i++) acc[i] = __double_as_longlong(fma(__longlong_as_double(x[i] * 0x100000001ll), __longlong_as_double(y64), __longlong_as_double(acc[i])));
    }
    y += 0x3779b9; y64 += 0x7f4a7c15ll;
  }
  long long t1 = clock64();
  unsigned long long s = 0;
#pragma unroll
  for (int i = 0; i < NACC / 2; i++) s ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int blocks = nsm * 4, threads = 256;   // 32 warps/SM
  uint32_t* out; long long* cyc; unsigned long long* out64;
  cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&out64, blocks * threads * 8); cudaMalloc(&cyc, blocks * 8);
  long long* hc = new long long[blocks];
  const char* names[] = {"viaddmnmx_u32_min", "add2_min3_u32", "viaddmnmx_s32_max", "ffma_f32", "iadd3_u32",
                         "imad_wide_i32_i64", "i64_add_min", "dfma_f64"};
  for (int v = 0; v < 8; v++) {
    for (int rep = 0; rep < 2; rep++) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      switch (v) {
        case 0: bench<0><<<blocks, threads>>>(out, cyc, 7); break;
        case 1: bench<1><<<blocks, threads>>>(out, cyc, 7); break;
        case 2: bench<2><<<blocks, threads>>>(out, cyc, 7); break;
        case 3: bench<3><<<blocks, threads>>>(out, cyc, 7); break;
        case 4: bench<4><<<blocks, threads>>>(out, cyc, 7); break;
        case 5: bench64<0><<<blocks, threads>>>(out64, cyc, 7); break;
        case 6: bench64<1><<<blocks, threads>>>(out64, cyc, 7); break;
        case 7: bench64<2><<<blocks, threads>>>(out64, cyc, 7); break;
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(hc, cyc, blocks * 8, cudaMemcpyDeviceToHost);
      long long mx = 0; double mean = 0;
      for (int b = 0; b < blocks; b++) { mx = hc[b] > mx ? hc[b] : mx; mean += hc[b]; }
      mean /= blocks;
      double terms_per_thread = (double)ITERS * (v >= 5 ? NACC / 2 : (v == 1 ? 2 * NACC : NACC));
      // 4 blocks/SM of 256 threads co-resident: per-SM terms per cycle
      double per_sm_clk = terms_per_thread * threads * 4 / (double)mx;
      double total = terms_per_thread * threads * blocks;
      if (rep == 1)
        printf("%-20s terms/clk/SM=%7.2f  (mean-cyc based %7.2f)  wall=%.3f ms  Gterms/s=%.1f  implied_clk_MHz=%.0f\n",
               names[v], per_sm_clk, terms_per_thread * threads * 4 / mean, ms, total / ms / 1e6,
               (double)mx / (ms * 1e3));
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(e));
  return 0;
}
