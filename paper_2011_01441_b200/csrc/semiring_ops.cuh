// Semiring element algebra for the SIMT (non-tensor-core) PACO kernels.
//
// Each Op mirrors one reference Semiring (matmul.py:34-57) or one of the
// B200-native additions (saturating tropical on 32-bit lanes, fp32):
//   mac(acc, a, b)    one (x) then (+) into the register accumulator
//   finish(acc)       accumulator -> stored C value (tropical: saturate at +-INF)
//   combine(c, x)     the semiring (+) used to fold into existing C (vadd)
//   atomic_combine    the same fold as one global atomic (k-split pieces)
//   atomic_combine_sys  ... at system scope (C in a peer GPU's memory: the owner's
//                     own folds and this GPU's must be atomic w.r.t. each other)
//   bulk_combine      the same fold for a contiguous smem row, done by the TMA
//                     unit in L2 (cp.reduce.async.bulk)
//   zero()            the semiring zero the reference fills temps with
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

#include "common.cuh"

namespace paco {

// TMA bulk reduction smem -> global (SASS UBLKRED): the L2 applies the
// semiring (+) to `bytes` contiguous bytes.  Exact for the integer ops.
#define PACO_BULK_RED(NAME, OPTYPE)                                                    \
  __device__ __forceinline__ static void NAME(void* gdst, uint32_t ssrc, uint32_t bytes) { \
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group." OPTYPE          \
                 " [%0], [%1], %2;\n" ::"l"(gdst), "r"(ssrc), "r"(bytes) : "memory");    \
  }

// (min,+) on 32-bit lanes.  Inputs live in [0, 2^30] (2^30 = INF), so a + b
// <= 2^31 never wraps in u32; min() then a final clamp to 2^30 equals the
// saturating semiring exactly (min commutes with the clamp).  One SASS
// VIADDMNMX.U32 per term.
struct OpMinPlusSat32 {
  using TA = uint32_t;
  using TB = uint32_t;
  using TC = int32_t;
  using Acc = uint32_t;
  static constexpr int kId = PACO_SR_MINPLUS_SAT32;
  __device__ __forceinline__ static Acc identity() { return 0xFFFFFFFFu; }
  __device__ __forceinline__ static Acc mac(Acc acc, TA a, TB b) { return min(acc, a + b); }
  __device__ __forceinline__ static TC finish(Acc acc) {
    return static_cast<TC>(min(acc, static_cast<uint32_t>(PACO_TROPICAL_INF)));
  }
  __device__ __forceinline__ static TC combine(TC c, TC x) { return min(c, x); }
  __device__ __forceinline__ static void atomic_combine(TC* p, TC x) { atomicMin(p, x); }
  __device__ __forceinline__ static void atomic_combine_sys(TC* p, TC x) { atomicMin_system(p, x); }
  PACO_BULK_RED(bulk_combine, "min.s32")
  __host__ __device__ static TC zero() { return PACO_TROPICAL_INF; }
};

// The reference (min,+) semiring (int64, zero 2^62, matmul.py:29,49-50,55) on
// operands that fit [0, 2^31): on that domain a + b <= 2^32 - 2 never wraps in
// u32, so min(acc, a + b) on u32 lanes is the reference's int64 arithmetic
// exactly, with no clamp -- one VIADDMNMX.U32 per term.  C's narrowed image
// saturates at 2^32 - 1 (paco_narrow_i64); paco_widen_u32_i64 restores it.
struct OpMinPlusU32 {
  using TA = uint32_t;
  using TB = uint32_t;
  using TC = uint32_t;
  using Acc = uint32_t;
  static constexpr int kId = PACO_SR_MINPLUS_U32;
  __device__ __forceinline__ static Acc identity() { return 0xFFFFFFFFu; }
  __device__ __forceinline__ static Acc mac(Acc acc, TA a, TB b) { return min(acc, a + b); }
  __device__ __forceinline__ static TC finish(Acc acc) { return acc; }
  __device__ __forceinline__ static TC combine(TC c, TC x) { return min(c, x); }
  __device__ __forceinline__ static void atomic_combine(TC* p, TC x) { atomicMin(p, x); }
  __device__ __forceinline__ static void atomic_combine_sys(TC* p, TC x) { atomicMin_system(p, x); }
  PACO_BULK_RED(bulk_combine, "min.u32")
  __host__ __device__ static TC zero() { return 0xFFFFFFFFu; }
};

// (max,+) on signed 32-bit lanes, -INF = -2^30: sums stay in [-2^31, 2^31).
struct OpMaxPlusSat32 {
  using TA = int32_t;
  using TB = int32_t;
  using TC = int32_t;
  using Acc = int32_t;
  static constexpr int kId = PACO_SR_MAXPLUS_SAT32;
  __device__ __forceinline__ static Acc identity() { return INT32_MIN; }
  __device__ __forceinline__ static Acc mac(Acc acc, TA a, TB b) { return max(acc, a + b); }
  __device__ __forceinline__ static TC finish(Acc acc) { return max(acc, -PACO_TROPICAL_INF); }
  __device__ __forceinline__ static TC combine(TC c, TC x) { return max(c, x); }
  __device__ __forceinline__ static void atomic_combine(TC* p, TC x) { atomicMax(p, x); }
  __device__ __forceinline__ static void atomic_combine_sys(TC* p, TC x) { atomicMax_system(p, x); }
  PACO_BULK_RED(bulk_combine, "max.s32")
  __host__ __device__ static TC zero() { return -PACO_TROPICAL_INF; }
};

struct OpF32 {
  using TA = float;
  using TB = float;
  using TC = float;
  using Acc = float;
  static constexpr int kId = PACO_SR_F32;
  __device__ __forceinline__ static Acc identity() { return 0.f; }
  __device__ __forceinline__ static Acc mac(Acc acc, TA a, TB b) { return fmaf(a, b, acc); }
  __device__ __forceinline__ static TC finish(Acc acc) { return acc; }
  __device__ __forceinline__ static TC combine(TC c, TC x) { return c + x; }
  __device__ __forceinline__ static void atomic_combine(TC* p, TC x) { atomicAdd(p, x); }
  __device__ __forceinline__ static void atomic_combine_sys(TC* p, TC x) { atomicAdd_system(p, x); }
  PACO_BULK_RED(bulk_combine, "add.f32")
  __host__ __device__ static TC zero() { return 0.f; }
};

struct OpF64 {
  using TA = double;
  using TB = double;
  using TC = double;
  using Acc = double;
  static constexpr int kId = PACO_SR_F64;
  __device__ __forceinline__ static Acc identity() { return 0.0; }
  __device__ __forceinline__ static Acc mac(Acc acc, TA a, TB b) { return fma(a, b, acc); }
  __device__ __forceinline__ static TC finish(Acc acc) { return acc; }
  __device__ __forceinline__ static TC combine(TC c, TC x) { return c + x; }
  __device__ __forceinline__ static void atomic_combine(TC* p, TC x) { atomicAdd(p, x); }
  __device__ __forceinline__ static void atomic_combine_sys(TC* p, TC x) { atomicAdd_system(p, x); }
  PACO_BULK_RED(bulk_combine, "add.f64")
  __host__ __device__ static TC zero() { return 0.0; }
};

// int64 ring with two's-complement wrap (what NumPy int64 does).
struct OpIntI64 {
  using TA = int64_t;
  using TB = int64_t;
  using TC = int64_t;
  using Acc = uint64_t;
  static constexpr int kId = PACO_SR_INT_I64;
  __device__ __forceinline__ static Acc identity() { return 0ull; }
  __device__ __forceinline__ static Acc mac(Acc acc, TA a, TB b) {
    return acc + static_cast<uint64_t>(a) * static_cast<uint64_t>(b);
  }
  __device__ __forceinline__ static TC finish(Acc acc) { return static_cast<TC>(acc); }
  __device__ __forceinline__ static TC combine(TC c, TC x) {
    return static_cast<TC>(static_cast<uint64_t>(c) + static_cast<uint64_t>(x));
  }
  __device__ __forceinline__ static void atomic_combine(TC* p, TC x) {
    atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(x));
  }
  __device__ __forceinline__ static void atomic_combine_sys(TC* p, TC x) {
    atomicAdd_system(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(x));
  }
  PACO_BULK_RED(bulk_combine, "add.u64")
  __host__ __device__ static TC zero() { return 0; }
};

// int32 x int32 -> int64 accumulate (IMAD.WIDE); cfg1's configuration.
struct OpIntI32I64 {
  using TA = int32_t;
  using TB = int32_t;
  using TC = int64_t;
  using Acc = uint64_t;
  static constexpr int kId = PACO_SR_INT_I32_I64;
  __device__ __forceinline__ static Acc identity() { return 0ull; }
  __device__ __forceinline__ static Acc mac(Acc acc, TA a, TB b) {
    return acc + static_cast<uint64_t>(static_cast<int64_t>(a) * static_cast<int64_t>(b));
  }
  __device__ __forceinline__ static TC finish(Acc acc) { return static_cast<TC>(acc); }
  __device__ __forceinline__ static TC combine(TC c, TC x) {
    return static_cast<TC>(static_cast<uint64_t>(c) + static_cast<uint64_t>(x));
  }
  __device__ __forceinline__ static void atomic_combine(TC* p, TC x) {
    atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(x));
  }
  __device__ __forceinline__ static void atomic_combine_sys(TC* p, TC x) {
    atomicAdd_system(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(x));
  }
  PACO_BULK_RED(bulk_combine, "add.u64")
  __host__ __device__ static TC zero() { return 0; }
};

// The reference (min,+) semiring verbatim: int64, zero = 2^62, NON-saturating
// wrapping add (matmul.py:29,49-50,55).
struct OpMinPlusI64 {
  using TA = int64_t;
  using TB = int64_t;
  using TC = int64_t;
  using Acc = int64_t;
  static constexpr int kId = PACO_SR_MINPLUS_I64;
  __device__ __forceinline__ static Acc identity() { return INT64_MAX; }
  __device__ __forceinline__ static Acc mac(Acc acc, TA a, TB b) {
    const Acc s = static_cast<Acc>(static_cast<uint64_t>(a) + static_cast<uint64_t>(b));
    return s < acc ? s : acc;
  }
  __device__ __forceinline__ static TC finish(Acc acc) { return acc; }
  __device__ __forceinline__ static TC combine(TC c, TC x) { return x < c ? x : c; }
  __device__ __forceinline__ static void atomic_combine(TC* p, TC x) {
    atomicMin(reinterpret_cast<long long*>(p), static_cast<long long>(x));
  }
  __device__ __forceinline__ static void atomic_combine_sys(TC* p, TC x) {
    atomicMin_system(reinterpret_cast<long long*>(p), static_cast<long long>(x));
  }
  PACO_BULK_RED(bulk_combine, "min.s64")
  __host__ __device__ static TC zero() { return static_cast<TC>(1) << 62; }
};

// bf16 x bf16 -> fp32: only its elementwise pieces (fold/fill/naive) use this;
// the product kernel is the tcgen05 one.
struct OpBF16F32 {
  using TA = __nv_bfloat16;
  using TB = __nv_bfloat16;
  using TC = float;
  using Acc = float;
  static constexpr int kId = PACO_SR_BF16_F32;
  __device__ __forceinline__ static Acc identity() { return 0.f; }
  __device__ __forceinline__ static Acc mac(Acc acc, TA a, TB b) {
    return fmaf(__bfloat162float(a), __bfloat162float(b), acc);
  }
  __device__ __forceinline__ static TC finish(Acc acc) { return acc; }
  __device__ __forceinline__ static TC combine(TC c, TC x) { return c + x; }
  __device__ __forceinline__ static void atomic_combine(TC* p, TC x) { atomicAdd(p, x); }
  __device__ __forceinline__ static void atomic_combine_sys(TC* p, TC x) { atomicAdd_system(p, x); }
  PACO_BULK_RED(bulk_combine, "add.f32")
  __host__ __device__ static TC zero() { return 0.f; }
};

// Dispatch a functor templated on the Op for a runtime semiring id.
template <class F>
int dispatch_op(int sr, F&& f) {
  switch (sr) {
    case PACO_SR_INT_I64: return f(OpIntI64{});
    case PACO_SR_INT_I32_I64: return f(OpIntI32I64{});
    case PACO_SR_F64: return f(OpF64{});
    case PACO_SR_MINPLUS_I64: return f(OpMinPlusI64{});
    case PACO_SR_MINPLUS_SAT32: return f(OpMinPlusSat32{});
    case PACO_SR_MAXPLUS_SAT32: return f(OpMaxPlusSat32{});
    case PACO_SR_MINPLUS_U32: return f(OpMinPlusU32{});
    case PACO_SR_F32:
    case PACO_SR_F32_TC: return f(OpF32{});
    case PACO_SR_BF16_F32: return f(OpBF16F32{});
    default: set_error("unknown semiring id %d", sr); return PACO_ERR_ARG;
  }
}

}  // namespace paco
