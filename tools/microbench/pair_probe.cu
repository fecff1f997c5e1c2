// CTA-pair (cta_group::2) probe for sm_100a: TMEM allocation semantics and one
// M=256 x N=256 x K=16 kind::tf32 MMA whose A is split over the two CTAs by M
// and B (given as B^T, K-major) by N, checked against the CPU.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o pair_probe pair_probe.cu -lcuda
//   timeout 60 ./pair_probe
//
// Stage 1 (alloc): warp 1 of BOTH CTAs executes tcgen05.alloc.cta_group::2 for
// 256 columns and reports the address it got -- tells whether the pair
// allocates collectively (same address) or twice.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t cta_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank)); return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t par) {
  uint32_t d; asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(d) : "r"(a), "r"(par) : "memory"); return d;
}
__device__ void mbar_wait(uint64_t* b, uint32_t par, int* err) {
  for (uint32_t t = 0; !mbar_try(smem_u32(b), par); ++t) if (t > (1u << 22)) { *err = 1; return; }
}

extern "C" __global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
alloc_probe(uint32_t* out, int ncols) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&slot)), "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) out[blockIdx.x] = slot;
  cluster_sync();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(slot), "r"(ncols));
}

// ---- stage 2: one pair MMA --------------------------------------------------
// smem (each CTA): A slice 128 x 16 fp32 (K-major, 64B rows, SWIZZLE_64B
// layout written by threads), B^T slice 128 x 16 (rows n0..n0+127), loaded by
// plain stores in the swizzled layout: chunk c of row r at r*64 + ((c ^ ((r>>1)&3))*16).
__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(512 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(4) << 61;
  return d;
}

extern "C" __global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
mma_probe(const float* A /*256 x 16*/, const float* Bt /*256 x 16*/, float* D /*256 x 256*/, int* err, int m_split_b) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 16384 + 64);
  const uint32_t rank = cta_rank();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // fill own slices: A rows rank*128.., B^T rows rank*128.. (N split)
  for (int e = threadIdx.x; e < 128 * 4; e += blockDim.x) {
    const int r = e / 4, c = e % 4;
    const int sw = c ^ ((r >> 1) & 3);
    const float* ga = A + (rank * 128 + r) * 16 + c * 4;
    const float* gb = Bt + ((m_split_b ? rank * 128 : rank * 128) + r) * 16 + c * 4;
    float4 va = *reinterpret_cast<const float4*>(ga), vb = *reinterpret_cast<const float4*>(gb);
    *reinterpret_cast<float4*>(smem + r * 64 + sw * 16) = va;
    *reinterpret_cast<float4*>(smem + 8192 + r * 64 + sw * 16) = vb;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *slot;
  if (rank == 0 && threadIdx.x == 32) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(256 >> 3) << 17) | (uint32_t(256 >> 4) << 24);
    const uint64_t ad = desc_sw64(smem_u32(smem)), bd = desc_sw64(smem_u32(smem + 8192));
    for (int kk = 0; kk < 2; ++kk)
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p; }"
                   :: "r"(tmem), "l"(ad + uint64_t(2 * kk)), "l"(bd + uint64_t(2 * kk)), "r"(idesc), "r"(kk));
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(smem_u32(bar)), "h"((uint16_t)3));
  }
  mbar_wait(bar, 0, err);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // each warp reads its 32 TMEM lanes x 256 columns in 8 chunks of 32
  for (int c = 0; c < 8; ++c) {
    uint32_t v[32];
    const uint32_t ta = tmem + (uint32_t(32 * warp) << 16) + uint32_t(32 * c);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                   "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                   "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int row = rank * 128 + 32 * warp + lane;
    for (int j = 0; j < 32; ++j) D[row * 256 + 32 * c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(256));
}

int main() {
  uint32_t* d_out;
  CK(cudaMalloc(&d_out, 64));
  CK(cudaMemset(d_out, 0xff, 64));
  alloc_probe<<<2, 128>>>(d_out, 256);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  uint32_t h[2];
  CK(cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost));
  printf("alloc cta_group::2 x2 (256 cols): cta0 -> %u, cta1 -> %u\n", h[0], h[1]);
  // stage 2
  std::vector<float> A(256 * 16), Bt(256 * 16), D(256 * 256);
  srand(1);
  for (auto& x : A) x = float(rand() % 17 - 8);   // small integers: exact in tf32 and fp32
  for (auto& x : Bt) x = float(rand() % 17 - 8);
  float *dA, *dB, *dD;
  int* derr;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, Bt.size() * 4));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMalloc(&derr, 4));
  CK(cudaMemset(derr, 0, 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, Bt.data(), Bt.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(mma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 20480 + 1024));
  mma_probe<<<2, 128, 20480 + 1024>>>(dA, dB, dD, derr, 1);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  int err = 0;
  CK(cudaMemcpy(&err, derr, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0, bad_alt = 0;
  for (int i = 0; i < 256; ++i)
    for (int j = 0; j < 256; ++j) {
      double s = 0;
      for (int l = 0; l < 16; ++l) s += double(A[i * 16 + l]) * double(Bt[j * 16 + l]);
      if (fabs(s - D[i * 256 + j]) > 1e-3) {
        if (bad < 5) printf("mismatch D[%d][%d] = %g want %g\n", i, j, D[i * 256 + j], s);
        ++bad;
      }
    }
  (void)bad_alt;
  printf("pair MMA M=256 N=256 K=16: %d mismatches of 65536, barrier timeout=%d\n", bad, err);
  return bad ? 2 : 0;
}
