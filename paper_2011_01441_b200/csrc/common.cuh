// Shared definitions for the sm_100a PACO semiring-MM library.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/paco_b200.h"

namespace paco {

constexpr int kNumSMs = 148;
constexpr int kMaxPieces = PACO_MAX_PIECES;

// One CTA-level PACO piece in TILE units (tile sizes are kernel-specific).
// A piece whose k-range does not cover the whole k extent folds its partial C
// face with an atomic (+) -- exact for the integer / tropical semirings.
struct Piece {
  int32_t ti0, tj0, tl0;  // tile offsets along n, m, k
  int32_t tn, tm, tk;     // extents in tiles
};

struct PieceTable {
  int32_t count;
  int32_t ksplit;  // 1 if any piece covers a strict sub-range of k
  int32_t grid_s;  // count == 0: 0 = PACO plan derived per CTA; s > 0 = tile grid, k split s ways
  int32_t grid_tail;  // tile grid: > 1 = the tiles from grid_head on are split grid_tail ways in k
  int32_t grid_head;
  Piece p[kMaxPieces];
};

// paco_debug_trace()'s device buffer (diagnostics; null when off)
extern long long* g_trace_buffer;

// thread-local error text behind paco_last_error()
void set_error(const char* fmt, ...);

// Developer tuning knobs (CTA-plan overrides, kernel ablations, ...): read from
// the environment ONLY when PACO_DEV_KNOBS=1, so an ordinary user environment
// can never select an unmeasured configuration.  nullptr when unset or gated.
const char* dev_knob(const char* name);
// 2-D row-major tensor map of 4- or 8-byte elements (no swizzle, zero OOB fill)
// over a 16-byte aligned base with a 16-byte row pitch (tc_gemm.cu)
int encode_map_2d(CUtensorMap* map, int elsize, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                  uint32_t box_cols, uint32_t box_rows);

// Live per-kernel timing (paco_kernel_timing): while on, every launch site
// brackets its kernel with a CUDA event pair on the launching stream, so a
// caller can measure the dominant kernel's average duration inside a real
// multi-kernel step (bench.py's roofline).  Off: one relaxed atomic load.
extern std::atomic<int> g_ktime_on;
void ktime_record(int family, cudaStream_t st, bool start);
struct KernelSpan {
  int fam;
  cudaStream_t st;
  bool on;
  KernelSpan(int f, cudaStream_t s) : fam(f), st(s), on(g_ktime_on.load(std::memory_order_relaxed) != 0) {
    if (on) ktime_record(fam, st, true);
  }
  ~KernelSpan() {
    if (on) ktime_record(fam, st, false);
  }
};

#define PACO_CUDA_TRY(expr)                                                     \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) {                                                    \
      ::paco::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr,            \
                        cudaGetErrorString(_e));                                \
      return PACO_ERR_CUDA;                                                     \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async copy with zero fill of the bytes past `src_bytes`.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// CTA-scope mbarrier helpers for the SIMT ring.
__device__ __forceinline__ void mbar_init_cta(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// arrive once this thread's earlier cp.async copies have landed (count not incremented)
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_cta(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}

}  // namespace paco
