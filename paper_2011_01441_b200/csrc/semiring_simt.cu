// Register-blocked SIMT semiring MM for sm_100a (tropical / integer / fp32 / fp64).
//
// Replaces the reference's recursive mm_seq + 32^3 NumPy leaves
// (matmul.py:342-397, block kernels 45-50) with one launch:
//   * grid = the CTA-level plan.  Default: the tile grid -- one CTA per 128x128
//     C tile and k range, the k extent split s ways by a cost model (whole
//     SM-waves x per-visit cost, grid_plan; the partial last wave's tiles
//     split in k on their own); measured faster than the
//     balanced PACO cuboid plan (MM-1-Piece over tile units,
//     plan_pieces_balanced), which stays available (PACO_MM_PACO_PLAN) and
//     for explicit piece tables;
//   * each CTA walks the C tiles of its piece; per tile it streams its k range
//     through a STAGES-deep cp.async ring (16 B; an unpredicated fast path for
//     interior tiles, zero-filled predicated loads at the edges) synchronised
//     by split arrive/wait mbarriers (full: copies landed, empty: stage read);
//   * a 16x16 thread grid holds TMxTN register accumulators per thread, fed by
//     128-bit LDS from padded, bank-conflict-free shared tiles;
//   * epilogue: C (+)= acc through TMA bulk copies / bulk reductions
//     (cp.reduce.async.bulk min/max/add, exact and order-free for the
//     integer/tropical semirings when pieces split k), or per-element stores /
//     atomics at ragged edges.
// The tropical inner loop is one VIADDMNMX per term (checked in SASS).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "cta_plan.cuh"
#include "semiring_ops.cuh"

namespace paco {

// 8192^3 (min,+) with 1/2/3/4/5/8 waves of 296: 37.5/35.2/34.6/34.3/35.1/35.6 ms
constexpr int kDefaultWaves = 4;
#ifndef PACO_SIMT_WIDE_TILE
#define PACO_SIMT_WIDE_TILE 128
#endif
#ifndef PACO_SIMT_MBAR
#define PACO_SIMT_MBAR 1
#endif
constexpr bool kMbarPipe = PACO_SIMT_MBAR != 0;  // split arrive/wait stage ring (vs __syncthreads)
constexpr double kDefaultKw = 1.0;
constexpr int kMaxKSplit = 64;
constexpr double kVisitK = 64.0;  // per-visit cost in k elements (re-fitted with the mbarrier ring)

// Device buffer of 10 x (grid size) int64 set by paco_debug_trace(); when
// non-null every CTA of the next launches records smid and start/end times.
long long* g_trace_buffer = nullptr;

#ifndef PACO_SIMT_BK
#define PACO_SIMT_BK 32  // 32-bit ops: k depth of a ring stage (16: six stages of the same total size)
#endif
#ifndef PACO_SIMT_NSPAN
#define PACO_SIMT_NSPAN 1  // 32-bit ops: C tile width in units of 128 columns (2 = 128x256 tiles,
                           // 1 CTA/SM: measured 34.7 vs 34.4 ms on 8192^3 min-plus -- kept at 1)
#endif

template <class Op>
struct SimtCfg {
  static constexpr bool kWide = sizeof(typename Op::Acc) == 8;
  // 64-bit accumulators: 128x128 tiles too (8x8 per thread = 128 registers of
  // accumulators, one CTA per SM) -- 64x64 tiles left DFMA at 38 % of its issue
  // rate (smem-bound: 2 loaded values per term pair)
  static constexpr int BM = kWide ? PACO_SIMT_WIDE_TILE : 128;
  static constexpr int BN = kWide ? PACO_SIMT_WIDE_TILE : 128 * PACO_SIMT_NSPAN;
  static constexpr int BK = kWide ? 16 : PACO_SIMT_BK;
  static constexpr int GM = BM / 64;  // 4-row groups per thread along m
  static constexpr int GN = BN / 64;
  static constexpr int TM = 4 * GM;
  static constexpr int TN = 4 * GN;
  static constexpr int THREADS = 256;
  static constexpr int STAGES = kWide ? 4 : (PACO_SIMT_NSPAN > 1 ? 4 : (PACO_SIMT_BK == 16 ? 6 : 3));
  static constexpr int MIN_BLOCKS = (!kWide && PACO_SIMT_NSPAN > 1) || (kWide && BM > 64) ? 1 : 2;
  static constexpr int VA = 16 / sizeof(typename Op::TA);  // elements per 16 B chunk
  static constexpr int VB = 16 / sizeof(typename Op::TB);
  static constexpr int KQ = VA;          // k quantum of piece boundaries
  static constexpr int LDA_S = BK + VA;  // padded smem row (k-major rows of A)
  static constexpr int LDB_S = BN;
  static constexpr int A_STAGE = BM * LDA_S;
  static constexpr int B_STAGE = BK * LDB_S;
  static constexpr int A_CPR = BK / VA;             // 16 B chunks per A tile row
  static constexpr int A_RPP = THREADS / A_CPR;     // A rows covered per pass
  static constexpr int A_PASSES = BM / A_RPP;
  static constexpr int B_CPR = BN / VB;
  static constexpr int B_RPP = THREADS / B_CPR;
  static constexpr int B_PASSES = BK / B_RPP;
  static constexpr size_t SMEM =
      size_t(STAGES) * (A_STAGE * sizeof(typename Op::TA) + B_STAGE * sizeof(typename Op::TB));
  // TMA stage loads (32-bit operands): A as one [BM rows][LDA_S k] box -- the box's
  // inner extent IS the padded smem row, so the bank-conflict-free layout comes for
  // free (the 4 extra k per row are read and ignored) -- and B as one [BK][BN] box
  static constexpr bool kTmaOk = !kWide && sizeof(typename Op::TA) == 4 && sizeof(typename Op::TB) == 4 &&
                                 LDA_S * 4 % 16 == 0 && BN <= 256;
  static constexpr uint32_t TMA_BYTES = uint32_t(BM * LDA_S * 4 + BK * BN * 4);
  static_assert(A_RPP * A_CPR == THREADS && A_PASSES * A_RPP == BM, "A load mapping");
  static_assert(B_RPP * B_CPR == THREADS && B_PASSES * B_RPP == BK, "B load mapping");
};

template <class T>
struct Vec4 {
  T v[4];
};

template <class T>
__device__ __forceinline__ Vec4<T> lds4(const T* p) {
  Vec4<T> r;
  if constexpr (sizeof(T) == 4) {
    const uint4 x = *reinterpret_cast<const uint4*>(p);
    memcpy(&r, &x, 16);
  } else {
    const ulonglong2 x = reinterpret_cast<const ulonglong2*>(p)[0];
    const ulonglong2 y = reinterpret_cast<const ulonglong2*>(p)[1];
    memcpy(&r.v[0], &x, 16);
    memcpy(&r.v[2], &y, 16);
  }
  return r;
}

struct MMArgs {
  const void* A;
  const void* B;
  void* C;
  int64_t lda, ldb, ldc;
  int64_t n, m, k;
  int32_t kq;  // k quantum of the piece table
  int32_t overwrite;
  long long* trace;  // optional per-CTA [smid, start ns, end ns, stages] (diagnostics)
  int32_t bulk_ok;   // C is 16 B aligned with ldc*sizeof(TC) % 16 == 0: TMA bulk epilogue
  int32_t all_atomic;  // every piece folds atomically (other kernels fold into the same C)
  double kw;           // virtual k weight of the CTA plan (cta_plan.cuh)
  int32_t sys_atomic;  // C is peer memory (PACO_MM_REMOTE): element folds at system scope
};

struct BatchTable {
  int32_t count;
  int32_t grid_s[PACO_MAX_BATCH];
  int32_t grid_tail[PACO_MAX_BATCH];  // tail split (plan_grid_piece)
  int32_t grid_head[PACO_MAX_BATCH];
  int64_t first[PACO_MAX_BATCH + 1];  // CTA prefix sums
  MMArgs args[PACO_MAX_BATCH];
};

// Stage one (C tile, k tile) of A and B into shared memory.  kVec: 16 B
// chunks; interior tiles skip every bound check.
template <class Op, bool kVec>
__device__ __forceinline__ void load_stage(const MMArgs& a, typename Op::TA* As, typename Op::TB* Bs,
                                           int64_t row0, int64_t col0, int64_t k0, int64_t kend) {
  using C = SimtCfg<Op>;
  using TA = typename Op::TA;
  using TB = typename Op::TB;
  const TA* A = static_cast<const TA*>(a.A);
  const TB* B = static_cast<const TB*>(a.B);
  const int tid = threadIdx.x;
  if constexpr (kVec) {
    const int ar = tid / C::A_CPR, ak = (tid % C::A_CPR) * C::VA;
    const int br = tid / C::B_CPR, bc = (tid % C::B_CPR) * C::VB;
    TA* sa = As + ar * C::LDA_S + ak;
    TB* sb = Bs + br * C::LDB_S + bc;
    const bool interior = (row0 + C::BM <= a.n) && (col0 + C::BN <= a.m) && (k0 + C::BK <= kend);
    if (interior) {
      const TA* ga = A + (row0 + ar) * a.lda + (k0 + ak);
      const TB* gb = B + (k0 + br) * a.ldb + (col0 + bc);
#pragma unroll
      for (int i = 0; i < C::A_PASSES; ++i)
        cp_async16(sa + i * C::A_RPP * C::LDA_S, ga + i * C::A_RPP * a.lda, 16);
#pragma unroll
      for (int i = 0; i < C::B_PASSES; ++i)
        cp_async16(sb + i * C::B_RPP * C::LDB_S, gb + i * C::B_RPP * a.ldb, 16);
    } else {
#pragma unroll
      for (int i = 0; i < C::A_PASSES; ++i) {
        const int64_t gr = row0 + ar + i * C::A_RPP, gk = k0 + ak;
        int bytes = 0;
        const TA* src = A;
        if (gr < a.n && gk < kend) {
          bytes = int((kend - gk < C::VA ? kend - gk : C::VA) * sizeof(TA));
          src = A + gr * a.lda + gk;
        }
        cp_async16(sa + i * C::A_RPP * C::LDA_S, src, bytes);
      }
#pragma unroll
      for (int i = 0; i < C::B_PASSES; ++i) {
        const int64_t gk = k0 + br + i * C::B_RPP, gc = col0 + bc;
        int bytes = 0;
        const TB* src = B;
        if (gk < kend && gc < a.m) {
          bytes = int((a.m - gc < C::VB ? a.m - gc : C::VB) * sizeof(TB));
          src = B + gk * a.ldb + gc;
        }
        cp_async16(sb + i * C::B_RPP * C::LDB_S, src, bytes);
      }
    }
  } else {
    // element-granular path for views that are not 16 B aligned
    constexpr int A_ITERS = C::BM * C::BK / C::THREADS;
#pragma unroll 4
    for (int it = 0; it < A_ITERS; ++it) {
      const int c = tid + it * C::THREADS;
      const int r = c / C::BK, kc = c % C::BK;
      const int64_t gr = row0 + r, gk = k0 + kc;
      const bool ok = gr < a.n && gk < kend;
      const TA* src = ok ? A + gr * a.lda + gk : A;
      if constexpr (sizeof(TA) == 4)
        cp_async4(As + r * C::LDA_S + kc, src, ok ? 4 : 0);
      else
        cp_async8(As + r * C::LDA_S + kc, src, ok ? 8 : 0);
    }
    constexpr int B_ITERS = C::BK * C::BN / C::THREADS;
#pragma unroll 4
    for (int it = 0; it < B_ITERS; ++it) {
      const int c = tid + it * C::THREADS;
      const int r = c / C::BN, nc = c % C::BN;
      const int64_t gk = k0 + r, gc = col0 + nc;
      const bool ok = gk < kend && gc < a.m;
      const TB* src = ok ? B + gk * a.ldb + gc : B;
      if constexpr (sizeof(TB) == 4)
        cp_async4(Bs + r * C::LDB_S + nc, src, ok ? 4 : 0);
      else
        cp_async8(Bs + r * C::LDB_S + nc, src, ok ? 8 : 0);
    }
  }
}

// Four k steps of the register-blocked product: 2*GM + 2*GN LDS.128 feed
// TM*TN*4 semiring MACs.
template <class Op>
__device__ __forceinline__ void mac_k4(typename Op::Acc (&acc)[SimtCfg<Op>::TM][SimtCfg<Op>::TN],
                                       const typename Op::TA* a_base, const typename Op::TB* b_base,
                                       int kk) {
  using C = SimtCfg<Op>;
  using TA = typename Op::TA;
  using TB = typename Op::TB;
  TA a[C::TM][4];
#pragma unroll
  for (int g = 0; g < C::GM; ++g)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const Vec4<TA> v = lds4(a_base + (g * 64 + r) * C::LDA_S + kk);
#pragma unroll
      for (int q = 0; q < 4; ++q) a[g * 4 + r][q] = v.v[q];
    }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    TB b[C::TN];
#pragma unroll
    for (int g = 0; g < C::GN; ++g) {
      const Vec4<TB> v = lds4(b_base + (kk + q) * C::LDB_S + g * 64);
#pragma unroll
      for (int e = 0; e < 4; ++e) b[g * 4 + e] = v.v[e];
    }
#pragma unroll
    for (int i = 0; i < C::TM; ++i)
#pragma unroll
      for (int j = 0; j < C::TN; ++j) acc[i][j] = Op::mac(acc[i][j], a[i][q], b[j]);
  }
}

// acc (+)= A_stage (x) B_stage over the first `kvalid` k of the stage.
template <class Op>
__device__ __forceinline__ void compute_stage(typename Op::Acc (&acc)[SimtCfg<Op>::TM][SimtCfg<Op>::TN],
                                              const typename Op::TA* As, const typename Op::TB* Bs,
                                              int kvalid) {
  using C = SimtCfg<Op>;
  using TA = typename Op::TA;
  using TB = typename Op::TB;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const TA* a_base = As + (ty * 4) * C::LDA_S;
  const TB* b_base = Bs + tx * 4;
  if (kvalid == C::BK) {
#pragma unroll
    for (int kk = 0; kk < C::BK; kk += 4) mac_k4<Op>(acc, a_base, b_base, kk);
    return;
  }
  int kk = 0;
  for (; kk + 4 <= kvalid; kk += 4) mac_k4<Op>(acc, a_base, b_base, kk);
  for (; kk < kvalid; ++kk) {  // only at a global k end that is not a multiple of 4
    TA a[C::TM];
    TB b[C::TN];
#pragma unroll
    for (int g = 0; g < C::GM; ++g)
#pragma unroll
      for (int r = 0; r < 4; ++r) a[g * 4 + r] = a_base[(g * 64 + r) * C::LDA_S + kk];
#pragma unroll
    for (int g = 0; g < C::GN; ++g)
#pragma unroll
      for (int e = 0; e < 4; ++e) b[g * 4 + e] = b_base[kk * C::LDB_S + g * 64 + e];
#pragma unroll
    for (int i = 0; i < C::TM; ++i)
#pragma unroll
      for (int j = 0; j < C::TN; ++j) acc[i][j] = Op::mac(acc[i][j], a[i], b[j]);
  }
}

template <class Op>
__device__ __forceinline__ void epilogue(const MMArgs& a,
                                         typename Op::Acc (&acc)[SimtCfg<Op>::TM][SimtCfg<Op>::TN],
                                         int64_t row0, int64_t col0, bool atomic) {
  using C = SimtCfg<Op>;
  using TC = typename Op::TC;
  TC* Cp = static_cast<TC*>(a.C);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const bool rmw = !atomic && !a.overwrite;
#pragma unroll
  for (int i = 0; i < C::TM; ++i) {
    const int64_t gr = row0 + (i / 4) * 64 + ty * 4 + (i % 4);
    if (gr >= a.n) continue;
    TC* crow = Cp + gr * a.ldc;
    // read-modify-write: issue the row's TN loads before any store, so they
    // are in flight together (one memory round trip per row, not per element)
    TC old[C::TN];
#pragma unroll
    for (int j = 0; j < C::TN; ++j) {
      const int64_t gc = col0 + (j / 4) * 64 + tx * 4 + (j % 4);
      old[j] = (rmw && gc < a.m) ? crow[gc] : TC(0);
    }
#pragma unroll
    for (int j = 0; j < C::TN; ++j) {
      const int64_t gc = col0 + (j / 4) * 64 + tx * 4 + (j % 4);
      if (gc >= a.m) continue;
      const TC v = Op::finish(acc[i][j]);
      if (atomic && a.sys_atomic)
        Op::atomic_combine_sys(crow + gc, v);
      else if (atomic)
        Op::atomic_combine(crow + gc, v);
      else if (a.overwrite)
        crow[gc] = v;
      else
        crow[gc] = Op::combine(old[j], v);
    }
  }
}

// Epilogue through the TMA unit: the finished tile is staged in the stage
// buffer that was just consumed (A part: 32 rows, B part: 32 rows of 512 B),
// 64 rows per round, and each row is folded into C by one
// cp.reduce.async.bulk (semiring (+) applied in L2) -- or stored with
// cp.async.bulk when overwriting.  Exact and order-free for k-split pieces.
template <class Op>
__device__ __forceinline__ void epilogue_bulk(const MMArgs& a,
                                              typename Op::Acc (&acc)[SimtCfg<Op>::TM][SimtCfg<Op>::TN],
                                              int64_t row0, int64_t col0, void* bufA, void* bufB,
                                              uint32_t bytes) {
  using C = SimtCfg<Op>;
  using TC = typename Op::TC;
  static_assert(C::BM == 128 && sizeof(TC) == 4, "bulk epilogue layout");
  // rows per round: the B stage buffer holds BK rows of the C tile, the padded
  // A buffer A_STAGE / BN more
  constexpr int ROOM = C::BK + C::A_STAGE / C::BN;
  static_assert(ROOM >= 32, "bulk epilogue staging room");
  constexpr int RPR = ROOM >= 64 ? 64 : 32;
  constexpr int ROUNDS = C::BM / RPR;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  TC* Cp = static_cast<TC*>(a.C);
  auto row_buf = [&](int lr) -> TC* {
    return lr < C::BK ? static_cast<TC*>(bufB) + lr * C::BN : static_cast<TC*>(bufA) + (lr - C::BK) * C::BN;
  };
  __syncthreads();  // every warp is done reading the stage buffer
#pragma unroll
  for (int h = 0; h < ROUNDS; ++h) {
    const int g = (h * RPR) / 64;                    // the thread's 64-row group in this round
    const int lr0 = 64 * g + ty * 4 - RPR * h;      // first local row of this thread
    if (lr0 >= 0 && lr0 < RPR) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        TC* dst = row_buf(lr0 + r);
#pragma unroll
        for (int gn = 0; gn < C::GN; ++gn) {
          TC v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) v[e] = Op::finish(acc[4 * g + r][4 * gn + e]);
          uint4 bits;
          memcpy(&bits, v, 16);  // bit copy (TC may be float)
          *reinterpret_cast<uint4*>(dst + gn * 64 + tx * 4) = bits;
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (lane == 0) {
#pragma unroll 1
      for (int q = 0; q < RPR / 8; ++q) {
        const int lr = warp * (RPR / 8) + q;
        const int64_t gr = row0 + RPR * h + lr;
        if (gr < a.n) {
          const void* src = row_buf(lr);
          TC* gdst = Cp + gr * a.ldc + col0;
          if (a.overwrite)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
                         "r"(smem_u32(src)), "r"(bytes) : "memory");
          else
            Op::bulk_combine(gdst, smem_u32(src), bytes);
        }
      }
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
    __syncthreads();  // smem free again (next round / the next cp.async stage)
  }
}

// Bulk epilogue for 8-byte C elements (64-bit tiles, 128 x 128, 1 KB rows):
// RPR rows per round are staged in shared memory and each row is folded into
// C by one cp.reduce.async.bulk (or stored by cp.async.bulk when overwriting)
// -- coalesced, order-free, no per-element atomics or load round trips.
// kWhole: the CTA's last tile, when every pipeline stage is free -- the whole
// stage area holds 64 (32-bit inputs) or 128 (64-bit inputs) rows, 2 or 1
// rounds; otherwise 16 rows per round in the just-consumed stage (8 in its B
// part, 8 in its A part).
template <class Op, bool kWhole>
__device__ __forceinline__ void epilogue_bulk_wide(const MMArgs& a,
                                                   typename Op::Acc (&acc)[SimtCfg<Op>::TM][SimtCfg<Op>::TN],
                                                   int64_t row0, int64_t col0, void* bufA, void* bufB,
                                                   uint32_t bytes) {
  using C = SimtCfg<Op>;
  using TC = typename Op::TC;
  static_assert(C::BM == 128 && C::BN == 128 && sizeof(TC) == 8, "wide bulk epilogue layout");
  static_assert(C::B_STAGE * sizeof(typename Op::TB) >= 8 * C::BN * sizeof(TC) &&
                C::A_STAGE * sizeof(typename Op::TA) >= 8 * C::BN * sizeof(TC), "staging room");
  constexpr int WHOLE_ROWS = int(C::SMEM / (C::BN * sizeof(TC)));
  constexpr int RPR = !kWhole ? 16 : (WHOLE_ROWS >= 128 ? 128 : 64);
  static_assert(!kWhole || WHOLE_ROWS >= 64, "whole-stage staging room");
  constexpr int ROUNDS = C::BM / RPR;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  TC* Cp = static_cast<TC*>(a.C);
  auto row_buf = [&](int lr) -> TC* {
    if constexpr (kWhole) return static_cast<TC*>(bufA) + lr * C::BN;
    return lr < 8 ? static_cast<TC*>(bufB) + lr * C::BN : static_cast<TC*>(bufA) + (lr - 8) * C::BN;
  };
  __syncthreads();  // every warp is done reading the stage buffers
#pragma unroll
  for (int h = 0; h < ROUNDS; ++h) {
#pragma unroll
    for (int g = 0; g < C::GM; ++g) {
      const int lr0 = 64 * g + ty * 4 - RPR * h;  // this thread's first row, local to the round
      if (lr0 >= 0 && lr0 < RPR) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          TC* dst = row_buf(lr0 + r);
#pragma unroll
          for (int gn = 0; gn < C::GN; ++gn) {
            TC v[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = Op::finish(acc[4 * g + r][4 * gn + e]);
            uint4 bits[2];
            memcpy(bits, v, 32);  // bit copy (TC may be double)
            reinterpret_cast<uint4*>(dst + gn * 64 + tx * 4)[0] = bits[0];
            reinterpret_cast<uint4*>(dst + gn * 64 + tx * 4)[1] = bits[1];
          }
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (lane == 0) {
#pragma unroll 1
      for (int q = 0; q < RPR / 8; ++q) {
        const int lr = warp * (RPR / 8) + q;
        const int64_t gr = row0 + RPR * h + lr;
        if (gr < a.n) {
          const void* src = row_buf(lr);
          TC* gdst = Cp + gr * a.ldc + col0;
          if (a.overwrite)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
                         "r"(smem_u32(src)), "r"(bytes) : "memory");
          else
            Op::bulk_combine(gdst, smem_u32(src), bytes);
        }
      }
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
    __syncthreads();  // smem free again
  }
}

// Operand tensor maps of a TMA-loaded launch (simt_mm_kernel<Op, true, true>).
struct SimtMaps {
  CUtensorMap a, b;
};

__device__ __forceinline__ void tma_load_2d_cta(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_cta(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// CTA-scope acq_rel counter bump (the slot-release vote of the TMA ring)
__device__ __forceinline__ uint32_t smem_add_acq_rel(uint32_t* p) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;\n" : "=r"(old) : "r"(smem_u32(p)) : "memory");
  return old;
}

// (ti, tj, kt) walk of one piece: k fastest, then C tile columns, then rows.
struct TileWalk {
  int ti, tj, kt;
  __device__ __forceinline__ void next(int tm, int KT) {
    if (++kt == KT) {
      kt = 0;
      if (++tj == tm) {
        tj = 0;
        ++ti;
      }
    }
  }
};

// One CTA's piece of one problem: the whole pipeline (ring, MACs, epilogue).
template <class Op, bool kVec, bool kTma = false>
__device__ __forceinline__ void simt_mm_body(const MMArgs& args, const Piece pc, const SimtMaps* maps = nullptr) {
  using C = SimtCfg<Op>;
  using TA = typename Op::TA;
  using TB = typename Op::TB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TA* As = reinterpret_cast<TA*>(smem_raw);
  TB* Bs = reinterpret_cast<TB*>(smem_raw + size_t(C::STAGES) * C::A_STAGE * sizeof(TA));

  long long t_start = 0;
  if (args.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  const int64_t kb = int64_t(pc.tl0) * args.kq;
  const int64_t kend = min(args.k, kb + int64_t(pc.tk) * args.kq);
  const bool atomic = args.all_atomic || !(kb == 0 && kend == args.k);
  const int KT = int((kend - kb + C::BK - 1) / C::BK);
  const int total = pc.tn * pc.tm * KT;

  TileWalk ld{0, 0, 0};
  typename Op::Acc acc[C::TM][C::TN];
#pragma unroll
  for (int i = 0; i < C::TM; ++i)
#pragma unroll
    for (int j = 0; j < C::TN; ++j) acc[i][j] = Op::identity();
  TileWalk cw{0, 0, 0};

  if constexpr (kTma) {
    // TMA ring: stage j of the piece's (tile, k tile) walk lands in slot j % STAGES
    // by two tensor copies completing on full[slot].  No thread issues per-element
    // copies or waits for a free slot: each warp votes on freed[slot] after reading
    // it (and after an epilogue staged in it), and the warp casting the slot's
    // last vote refills it with stage j + STAGES -- so a slow warp delays only the
    // refill of the slot it still reads, never another warp's arithmetic.
    static_assert(C::kTmaOk, "TMA stage layout");
    constexpr int NWARPS = C::THREADS / 32;
    static_assert((NWARPS & (NWARPS - 1)) == 0, "vote modulus");
    __shared__ uint64_t full[C::STAGES];
    __shared__ uint32_t freed[C::STAGES];
    const int lane = threadIdx.x % 32;
    auto issue = [&](int j, int slot) {
      const int kt = j % KT, t = j / KT;
      const int tj = t % pc.tm, ti = t / pc.tm;
      const int row0 = (pc.ti0 + ti) * C::BM, col0 = (pc.tj0 + tj) * C::BN;
      const int k0 = int(kb) + kt * C::BK;
      mbar_arrive_expect_tx_cta(&full[slot], C::TMA_BYTES);
      tma_load_2d_cta(As + slot * C::A_STAGE, &maps->a, &full[slot], k0, row0);
      tma_load_2d_cta(Bs + slot * C::B_STAGE, &maps->b, &full[slot], col0, k0);
    };
    if (threadIdx.x == 0) {
      for (int s = 0; s < C::STAGES; ++s) {
        mbar_init_cta(&full[s], 1);
        freed[s] = 0;
      }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      for (int s = 0; s < C::STAGES && s < total; ++s) issue(s, s);
    }
    __syncthreads();
    for (int it = 0; it < total; ++it) {
      const int s = it % C::STAGES;
      mbar_wait_cta(&full[s], uint32_t(it / C::STAGES) & 1);
      const int64_t k0 = kb + int64_t(cw.kt) * C::BK;
      const int kvalid = (kend - k0 < C::BK) ? int(kend - k0) : C::BK;
      compute_stage<Op>(acc, As + s * C::A_STAGE, Bs + s * C::B_STAGE, kvalid);
      if (cw.kt == KT - 1) {
        const int64_t row0 = int64_t(pc.ti0 + cw.ti) * C::BM, col0 = int64_t(pc.tj0 + cw.tj) * C::BN;
        const int64_t cols = (args.m - col0 < C::BN) ? args.m - col0 : C::BN;
        const uint32_t bytes = uint32_t(cols * sizeof(typename Op::TC));
        if (args.bulk_ok && (bytes % 16) == 0)  // stages the tile in slot s (CTA-wide syncs)
          epilogue_bulk<Op>(args, acc, row0, col0, As + s * C::A_STAGE, Bs + s * C::B_STAGE, bytes);
        else
          epilogue<Op>(args, acc, row0, col0, atomic);
#pragma unroll
        for (int i = 0; i < C::TM; ++i)
#pragma unroll
          for (int j = 0; j < C::TN; ++j) acc[i][j] = Op::identity();
      }
      cw.next(pc.tm, KT);
      if (it + C::STAGES < total) {
        __syncwarp();
        if (lane == 0 && (smem_add_acq_rel(&freed[s]) & (NWARPS - 1)) == NWARPS - 1) issue(it + C::STAGES, s);
      }
    }
  } else if constexpr (kMbarPipe) {
    // Split arrive/wait ring: full[s] completes when every thread's cp.async
    // into stage s has landed (cp.async.mbarrier.arrive.noinc); empty[s]
    // when every thread has finished reading it.  A stage is refilled one
    // iteration after it was consumed, so the empty wait is almost never a
    // stall -- unlike a __syncthreads per k step, which makes all 8 warps
    // meet every stage.
    __shared__ uint64_t full[C::STAGES], empty[C::STAGES];
    if (threadIdx.x == 0) {
      for (int s = 0; s < C::STAGES; ++s) {
        mbar_init_cta(&full[s], C::THREADS);
        mbar_init_cta(&empty[s], C::THREADS);
      }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < C::STAGES - 1; ++s) {
      if (s < total) {
        load_stage<Op, kVec>(args, As + s * C::A_STAGE, Bs + s * C::B_STAGE,
                             int64_t(pc.ti0 + ld.ti) * C::BM, int64_t(pc.tj0 + ld.tj) * C::BN,
                             kb + int64_t(ld.kt) * C::BK, kend);
        cp_async_arrive_noinc(&full[s]);
        ld.next(pc.tm, KT);
      }
    }
    for (int it = 0; it < total; ++it) {
      const int s = it % C::STAGES;
      mbar_wait_cta(&full[s], uint32_t(it / C::STAGES) & 1);
      const int64_t k0 = kb + int64_t(cw.kt) * C::BK;
      const int kvalid = (kend - k0 < C::BK) ? int(kend - k0) : C::BK;
      compute_stage<Op>(acc, As + s * C::A_STAGE, Bs + s * C::B_STAGE, kvalid);
      if (cw.kt == KT - 1) {
        const int64_t row0 = int64_t(pc.ti0 + cw.ti) * C::BM, col0 = int64_t(pc.tj0 + cw.tj) * C::BN;
        bool done = false;
        {
          const int64_t cols = (args.m - col0 < C::BN) ? args.m - col0 : C::BN;
          const uint32_t bytes = uint32_t(cols * sizeof(typename Op::TC));
          if (args.bulk_ok && (bytes % 16) == 0) {  // stages the tile in stage s (CTA-wide syncs)
            if constexpr (!C::kWide)
              epilogue_bulk<Op>(args, acc, row0, col0, As + s * C::A_STAGE, Bs + s * C::B_STAGE, bytes);
            else if (it == total - 1)  // last tile: no stage is in use any more
              epilogue_bulk_wide<Op, true>(args, acc, row0, col0, smem_raw, nullptr, bytes);
            else
              epilogue_bulk_wide<Op, false>(args, acc, row0, col0, As + s * C::A_STAGE, Bs + s * C::B_STAGE,
                                            bytes);
            done = true;
          }
        }
        if (!done) epilogue<Op>(args, acc, row0, col0, atomic);
#pragma unroll
        for (int i = 0; i < C::TM; ++i)
#pragma unroll
          for (int j = 0; j < C::TN; ++j) acc[i][j] = Op::identity();
      }
      cw.next(pc.tm, KT);
      mbar_arrive_cta(&empty[s]);
      const int nl = it + C::STAGES - 1;  // refill the stage consumed in the previous iteration
      if (nl < total) {
        const int sl = nl % C::STAGES;
        mbar_wait_cta(&empty[sl], (uint32_t(nl / C::STAGES) & 1) ^ 1);
        load_stage<Op, kVec>(args, As + sl * C::A_STAGE, Bs + sl * C::B_STAGE,
                             int64_t(pc.ti0 + ld.ti) * C::BM, int64_t(pc.tj0 + ld.tj) * C::BN,
                             kb + int64_t(ld.kt) * C::BK, kend);
        cp_async_arrive_noinc(&full[sl]);
        ld.next(pc.tm, KT);
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  } else {
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < total) {
      load_stage<Op, kVec>(args, As + s * C::A_STAGE, Bs + s * C::B_STAGE,
                           int64_t(pc.ti0 + ld.ti) * C::BM, int64_t(pc.tj0 + ld.tj) * C::BN,
                           kb + int64_t(ld.kt) * C::BK, kend);
      ld.next(pc.tm, KT);
    }
    cp_async_commit();
  }

  int s_load = C::STAGES - 1, s_comp = 0;
  for (int it = 0; it < total; ++it) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    if (it + C::STAGES - 1 < total) {
      load_stage<Op, kVec>(args, As + s_load * C::A_STAGE, Bs + s_load * C::B_STAGE,
                           int64_t(pc.ti0 + ld.ti) * C::BM, int64_t(pc.tj0 + ld.tj) * C::BN,
                           kb + int64_t(ld.kt) * C::BK, kend);
      ld.next(pc.tm, KT);
    }
    cp_async_commit();
    s_load = (s_load + 1 == C::STAGES) ? 0 : s_load + 1;

    const int64_t k0 = kb + int64_t(cw.kt) * C::BK;
    const int kvalid = (kend - k0 < C::BK) ? int(kend - k0) : C::BK;
    const int s_cur = s_comp;
    compute_stage<Op>(acc, As + s_cur * C::A_STAGE, Bs + s_cur * C::B_STAGE, kvalid);
    s_comp = (s_comp + 1 == C::STAGES) ? 0 : s_comp + 1;
    if (cw.kt == KT - 1) {
      const int64_t row0 = int64_t(pc.ti0 + cw.ti) * C::BM, col0 = int64_t(pc.tj0 + cw.tj) * C::BN;
      bool done = false;
      {
        const int64_t cols = (args.m - col0 < C::BN) ? args.m - col0 : C::BN;
        const uint32_t bytes = uint32_t(cols * sizeof(typename Op::TC));
        if (args.bulk_ok && (bytes % 16) == 0) {
          if constexpr (!C::kWide)
            epilogue_bulk<Op>(args, acc, row0, col0, As + s_cur * C::A_STAGE, Bs + s_cur * C::B_STAGE, bytes);
          else if (it == total - 1)
            epilogue_bulk_wide<Op, true>(args, acc, row0, col0, smem_raw, nullptr, bytes);
          else
            epilogue_bulk_wide<Op, false>(args, acc, row0, col0, As + s_cur * C::A_STAGE,
                                          Bs + s_cur * C::B_STAGE, bytes);
          done = true;
        }
      }
      if (!done) epilogue<Op>(args, acc, row0, col0, atomic);
#pragma unroll
      for (int i = 0; i < C::TM; ++i)
#pragma unroll
        for (int j = 0; j < C::TN; ++j) acc[i][j] = Op::identity();
    }
    cw.next(pc.tm, KT);
  }
  }
  cp_async_wait<0>();
  if (args.trace && threadIdx.x == 0) {
    long long t_end;
    unsigned smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    long long* tr = args.trace + 10 * blockIdx.x;
    tr[0] = smid;
    tr[1] = t_start;
    tr[2] = t_end;
    tr[3] = total;
    tr[4] = pc.ti0;
    tr[5] = pc.tj0;
    tr[6] = pc.tl0;
    tr[7] = pc.tn;
    tr[8] = pc.tm;
    tr[9] = pc.tk;
  }
}

template <class Op, bool kVec, bool kTma = false>
__global__ void __launch_bounds__(SimtCfg<Op>::THREADS, SimtCfg<Op>::MIN_BLOCKS)
    simt_mm_kernel(const MMArgs args, const __grid_constant__ PieceTable table,
                   const __grid_constant__ SimtMaps maps) {
  using C = SimtCfg<Op>;
  Piece pc;
  if (table.count > 0) {
    pc = table.p[blockIdx.x];
  } else {  // derive this CTA's piece of the default plan (same code as paco_plan_cta)
    UnitBox b;
    if (table.grid_s > 0)
      plan_grid_piece(args.n, args.m, args.k, C::BM, C::BN, C::KQ, table.grid_s, int(blockIdx.x), b,
                      table.grid_tail, table.grid_head);
    else
      plan_piece(args.n, args.m, args.k, C::BM, C::BN, C::KQ, int(gridDim.x), int(blockIdx.x), b, args.kw);
    pc = Piece{int32_t(b.o[0]), int32_t(b.o[1]), int32_t(b.o[2]), int32_t(b.e[0]), int32_t(b.e[1]),
               int32_t(b.e[2])};
  }
  simt_mm_body<Op, kVec, kTma>(args, pc, &maps);
}

// ---------------------------------------------------------------------------
// f64 (+,x) -- the reference's SEMIRING_F64 -- on the FP64 tensor pipe: warp-level
// DMMA (mma.sync m8n8k4 f64).  The SIMT DFMA kernel is shared-memory bound (one
// LDS.128 per 8 DFMAs per thread: 0.65 of the DFMA rate); a DMMA reuses each
// loaded A element across 8 columns and each B element across 8 rows inside the
// tensor unit, so operand traffic falls 4x and the FP64 pipe sets the pace
// (tools/microbench/dmma_probe.cu: 37.2 TFLOP/s DMMA vs 33.7 DFMA).
// Same CTA plan (128 x 128 tiles, pieces, k splits) and C semantics as the SIMT
// kernel; TMA stage ring with the last-vote refill; fragments stored straight
// from registers (atomic adds for k-split pieces).
// ---------------------------------------------------------------------------
#ifndef PACO_DMMA_WN
#define PACO_DMMA_WN 4  // warps along n (x 4 along m): 4 -> 32 x 32 warp tiles, 16 warps (2 -> 32 x 64, 8 warps: 31.4 vs 33.8 TFLOP/s at 4096^3)
#endif
struct DmmaCfg {
  static constexpr int WM = 4, WN = PACO_DMMA_WN, NW = WM * WN;
  static constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4, THREADS = 32 * NW;
  static constexpr int MI = BM / WM / 8, NJ = BN / WN / 8;  // 8 x 8 fragments per warp along m, n
  // padded rows: A k-rows of 20 doubles (160 B), B n-rows of 136 doubles (1088 B) --
  // both fragment loads then take the minimum two wavefronts.  The TMA boxes are
  // [BM][20] and [BK][136]: a box's inner extent is the padded row.
  static constexpr int LDA_S = BK + 4, LDB_S = BN + 8;
  static constexpr int A_STAGE = BM * LDA_S, B_STAGE = BK * LDB_S;  // doubles
  static constexpr uint32_t TMA_BYTES = uint32_t((A_STAGE + B_STAGE) * 8);
  static constexpr size_t SMEM = size_t(STAGES) * TMA_BYTES;
  static_assert(BM == SimtCfg<OpF64>::BM && BN == SimtCfg<OpF64>::BN, "same CTA plan as the SIMT f64 kernel");
};

__device__ __forceinline__ void dmma_m8n8k4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(DmmaCfg::THREADS, 1)
    dmma_f64_kernel(const MMArgs args, const __grid_constant__ PieceTable table, const __grid_constant__ SimtMaps maps) {
  using D = DmmaCfg;
  using S = SimtCfg<OpF64>;
  Piece pc;
  if (table.count > 0) {
    pc = table.p[blockIdx.x];
  } else {
    UnitBox b;
    if (table.grid_s > 0)
      plan_grid_piece(args.n, args.m, args.k, S::BM, S::BN, S::KQ, table.grid_s, int(blockIdx.x), b,
                      table.grid_tail, table.grid_head);
    else
      plan_piece(args.n, args.m, args.k, S::BM, S::BN, S::KQ, int(gridDim.x), int(blockIdx.x), b, args.kw);
    pc = Piece{int32_t(b.o[0]), int32_t(b.o[1]), int32_t(b.o[2]), int32_t(b.e[0]), int32_t(b.e[1]),
               int32_t(b.e[2])};
  }
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* As = reinterpret_cast<double*>(smem_raw);
  double* Bs = As + D::STAGES * D::A_STAGE;
  __shared__ uint64_t full[D::STAGES];
  __shared__ uint32_t freed[D::STAGES];

  const int64_t kb = int64_t(pc.tl0) * args.kq;
  const int64_t kend = min(args.k, kb + int64_t(pc.tk) * args.kq);
  const bool atomic = args.all_atomic || !(kb == 0 && kend == args.k);
  const int KT = int((kend - kb + D::BK - 1) / D::BK);
  const int total = pc.tn * pc.tm * KT;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int wm = warp % D::WM, wn = warp / D::WM;  // warp tile: rows 8 MI wm .., columns 8 NJ wn ..
  const int lr = lane / 4, lc = lane % 4;  // fragment row / column group

  auto issue = [&](int j, int slot) {
    const int kt = j % KT, t = j / KT;
    const int tj = t % pc.tm, ti = t / pc.tm;
    const int k0 = int(kb) + kt * D::BK;
    mbar_arrive_expect_tx_cta(&full[slot], D::TMA_BYTES);
    tma_load_2d_cta(As + slot * D::A_STAGE, &maps.a, &full[slot], k0, (pc.ti0 + ti) * D::BM);
    tma_load_2d_cta(Bs + slot * D::B_STAGE, &maps.b, &full[slot], (pc.tj0 + tj) * D::BN, k0);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < D::STAGES; ++s) {
      mbar_init_cta(&full[s], 1);
      freed[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    for (int s = 0; s < D::STAGES && s < total; ++s) issue(s, s);
  }
  __syncthreads();

  double acc[D::MI][D::NJ][2];
#pragma unroll
  for (int i = 0; i < D::MI; ++i)
#pragma unroll
    for (int j = 0; j < D::NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  TileWalk cw{0, 0, 0};
  for (int it = 0; it < total; ++it) {
    const int s = it % D::STAGES;
    mbar_wait_cta(&full[s], uint32_t(it / D::STAGES) & 1);
    const double* a_s = As + s * D::A_STAGE + (wm * 8 * D::MI + lr) * D::LDA_S + lc;
    const double* b_s = Bs + s * D::B_STAGE + lc * D::LDB_S + wn * 8 * D::NJ + lr;
    const int64_t k0 = kb + int64_t(cw.kt) * D::BK;
    const int kvalid = (kend - k0 < D::BK) ? int(kend - k0) : D::BK;
    if (kvalid == D::BK) {
#pragma unroll
      for (int ks = 0; ks < D::BK / 4; ++ks) {
        double a[D::MI], b[D::NJ];
#pragma unroll
        for (int i = 0; i < D::MI; ++i) a[i] = a_s[i * 8 * D::LDA_S + ks * 4];
#pragma unroll
        for (int j = 0; j < D::NJ; ++j) b[j] = b_s[ks * 4 * D::LDB_S + j * 8];
#pragma unroll
        for (int i = 0; i < D::MI; ++i)
#pragma unroll
          for (int j = 0; j < D::NJ; ++j) dmma_m8n8k4(acc[i][j], a[i], b[j]);
      }
    } else {  // the piece's (or the matrix's) last, partial k block: k >= kvalid contributes 0
      for (int ks = 0; ks * 4 < kvalid; ++ks) {
        const bool ok = ks * 4 + lc < kvalid;
        double a[D::MI], b[D::NJ];
#pragma unroll
        for (int i = 0; i < D::MI; ++i) a[i] = ok ? a_s[i * 8 * D::LDA_S + ks * 4] : 0.0;
#pragma unroll
        for (int j = 0; j < D::NJ; ++j) b[j] = ok ? b_s[ks * 4 * D::LDB_S + j * 8] : 0.0;
#pragma unroll
        for (int i = 0; i < D::MI; ++i)
#pragma unroll
          for (int j = 0; j < D::NJ; ++j) dmma_m8n8k4(acc[i][j], a[i], b[j]);
      }
    }
    if (cw.kt == KT - 1) {
      // fragment (i, j): rows row0 + 32 wm + 8 i + lr, columns col0 + 64 wn + 8 j + 2 lc + {0, 1}
      const int64_t row0 = int64_t(pc.ti0 + cw.ti) * D::BM + wm * 8 * D::MI + lr;
      const int64_t col0 = int64_t(pc.tj0 + cw.tj) * D::BN + wn * 8 * D::NJ + 2 * lc;
      double* Cp = static_cast<double*>(args.C);
      const bool pair_ok = (args.ldc % 2 == 0) && (reinterpret_cast<uintptr_t>(Cp) % 16 == 0);
#pragma unroll
      for (int i = 0; i < D::MI; ++i) {
        const int64_t r = row0 + 8 * i;
        if (r >= args.n) continue;
        double* crow = Cp + r * args.ldc;
#pragma unroll
        for (int j = 0; j < D::NJ; ++j) {
          const int64_t c = col0 + 8 * j;
          if (c >= args.m) continue;
          const bool two = c + 1 < args.m;
          if (atomic) {
            if (args.sys_atomic) {
              OpF64::atomic_combine_sys(crow + c, acc[i][j][0]);
              if (two) OpF64::atomic_combine_sys(crow + c + 1, acc[i][j][1]);
            } else {
              OpF64::atomic_combine(crow + c, acc[i][j][0]);
              if (two) OpF64::atomic_combine(crow + c + 1, acc[i][j][1]);
            }
          } else if (two && pair_ok) {
            double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
            if (!args.overwrite) {
              const double2 o = *reinterpret_cast<const double2*>(crow + c);
              v.x += o.x;
              v.y += o.y;
            }
            *reinterpret_cast<double2*>(crow + c) = v;
          } else {
            crow[c] = args.overwrite ? acc[i][j][0] : crow[c] + acc[i][j][0];
            if (two) crow[c + 1] = args.overwrite ? acc[i][j][1] : crow[c + 1] + acc[i][j][1];
          }
          acc[i][j][0] = acc[i][j][1] = 0.0;
        }
      }
    }
    cw.next(pc.tm, KT);
    if (it + D::STAGES < total) {
      __syncwarp();
      if (lane == 0 && (smem_add_acq_rel(&freed[s]) & uint32_t(D::NW - 1)) == uint32_t(D::NW - 1))
        issue(it + D::STAGES, s);
    }
  }
}

// A batch of independent problems (e.g. every COMPUTE cuboid of a GPU-level
// PACO plan on one device) as ONE launch: CTA ranges [first[q], first[q+1])
// take problem q's tile-grid pieces (k split grid_s[q] ways).
template <class Op, bool kVec>
__global__ void __launch_bounds__(SimtCfg<Op>::THREADS, SimtCfg<Op>::MIN_BLOCKS)
    simt_mm_batch_kernel(const __grid_constant__ BatchTable bt) {
  using C = SimtCfg<Op>;
  int q = 0;
  while (q + 1 < bt.count && int64_t(blockIdx.x) >= bt.first[q + 1]) ++q;
  const MMArgs& args = bt.args[q];
  UnitBox b;
  plan_grid_piece(args.n, args.m, args.k, C::BM, C::BN, C::KQ, bt.grid_s[q], int(blockIdx.x - bt.first[q]), b,
                  bt.grid_tail[q], bt.grid_head[q]);
  const Piece pc{int32_t(b.o[0]), int32_t(b.o[1]), int32_t(b.o[2]), int32_t(b.e[0]), int32_t(b.e[1]),
                 int32_t(b.e[2])};
  simt_mm_body<Op, kVec>(args, pc);
}

// ---------------------------------------------------------------------------
// CTA-level PACO planning (host side).
// ---------------------------------------------------------------------------
namespace {
struct Box {
  int64_t o[3];  // offsets (units)
  int64_t e[3];  // extents (units)
};

int virtual_axis(const double v[3]) {
  if (v[0] >= v[1] && v[0] >= v[2]) return 0;
  return v[1] >= v[2] ? 1 : 2;
}

// Exactly mm_one_piece_partition (matmul.py:250-300) on unit-size cells.
bool one_piece_rec(const Box& b, int lo_w, int hi_w, double v0, double v1, double v2,
                   std::vector<Box>& out) {
  const int cnt = hi_w - lo_w;
  if (cnt == 1) {
    out[lo_w] = b;
    return true;
  }
  const int h = cnt / 2;  // left list is the smaller one
  double v[3] = {v0, v1, v2};
  const int axis = virtual_axis(v);
  const int64_t len = b.e[axis];
  if (len < 2) return false;
  const int64_t left = std::max<int64_t>(1, len * h / cnt);
  Box lo = b, hi = b;
  lo.e[axis] = left;
  hi.o[axis] += left;
  hi.e[axis] = len - left;
  v[axis] /= 2;
  return one_piece_rec(lo, lo_w, lo_w + h, v[0], v[1], v[2], out) &&
         one_piece_rec(hi, lo_w + h, hi_w, v[0], v[1], v[2], out);
}

}  // namespace

bool plan_pieces(int64_t n, int64_t m, int64_t k, int p, std::vector<Box>& out) {
  out.assign(p, Box{});
  Box root{{0, 0, 0}, {n, m, k}};
  return one_piece_rec(root, 0, p, double(n), double(m), double(k), out);
}

// Virtual k weight of the default CTA plan; PACO_CTA_KW overrides it.
double plan_kw() {
  static double kw = -1.0;
  if (kw < 0.0) {
    const char* e = dev_knob("PACO_CTA_KW");
    kw = e ? atof(e) : kDefaultKw;
  }
  return kw;
}

bool plan_pieces_balanced(int64_t n, int64_t m, int64_t k, int bm, int bn, int kq, int p,
                          std::vector<Box>& out) {
  out.assign(p, Box{});
  for (int i = 0; i < p; ++i) {
    UnitBox b;
    if (!plan_piece(n, m, k, bm, bn, kq, p, i, b, plan_kw())) return false;
    for (int d = 0; d < 3; ++d) {
      out[i].o[d] = b.o[d];
      out[i].e[d] = b.e[d];
    }
  }
  return true;
}

// Default CTA-level plan size: 148 SMs x resident CTAs x waves (the later
// waves are dispatched to whichever SM frees a slot first).  PACO_CTA_PIECES
// overrides it (tuning / experiments).
int default_pieces(int ctas_per_sm) {
  static int env = -1;
  if (env < 0) {
    const char* e = dev_knob("PACO_CTA_PIECES");
    env = e ? atoi(e) : 0;
  }
  return env > 0 ? env : kNumSMs * ctas_per_sm * kDefaultWaves;
}

// Resolve the CTA plan: an explicit table (pieces != NULL), or the default
// plan derived on device (t.count = 0).  Returns the grid size in *grid.
// k split of the default tile-grid plan: whole SM-waves of equal pieces
// (ceil(tiles*s/148)), each piece k/s of work plus a fixed per-visit cost
// (ring fill, epilogue, fold) worth kVisitK k elements of MACs.  Measured on B200:
// lone CTAs run an SM at nearly full ALU rate, so only SM-level waves count.
// PACO_CTA_KSPLIT overrides s.
struct GridPlan {
  int s;         // k split of every tile
  int tail;      // > 1: tiles from `head` on are split `tail` ways instead
  int64_t head;  // whole-tile pieces before the tail
  int64_t ctas;
};

GridPlan grid_plan(const int64_t units[3], int kq) {
  static int env = -1, env_tail = -2;
  if (env < 0) {
    const char* e = dev_knob("PACO_CTA_KSPLIT");
    env = e ? atoi(e) : 0;
    const char* t = dev_knob("PACO_CTA_TAIL");  // 0/1: no tail split; > 1: forced
    env_tail = t ? atoi(t) : -1;
  }
  const int64_t tiles = units[0] * units[1];
  const int64_t smax = units[2] < kMaxKSplit ? units[2] : kMaxKSplit;
  const double kk = double(units[2] * kq);
  int64_t best = 1;
  if (env > 0) {
    best = env < smax ? env : smax;
  } else {
    double best_cost = 1e300;
    for (int64_t s = 1; s <= smax; ++s) {
      const double waves = double((tiles * s + kNumSMs - 1) / kNumSMs);
      const double cost = waves * (kk / double(s) + kVisitK);
      if (cost < best_cost * (1.0 - 1e-9)) {
        best_cost = cost;
        best = s;
      }
    }
  }
  GridPlan g{int(best), 0, tiles * best, tiles * best};
  // Tail split of the partial last SM-wave (whole tiles only): the rem tiles
  // left after the full waves cost one wave of full-k visits; split into t k
  // parts they cost ceil(rem * t / 148) waves of k/t visits.
  const int64_t rem = tiles % kNumSMs;
  if (best != 1 || rem == 0 || tiles < kNumSMs || env_tail == 0 || env_tail == 1) return g;
  int64_t tail = 1;
  double tail_cost = kk + kVisitK;
  if (env_tail > 1) {
    tail = env_tail < smax ? env_tail : smax;
  } else {
    for (int64_t t = 2; t <= smax; ++t) {
      const double c = double((rem * t + kNumSMs - 1) / kNumSMs) * (kk / double(t) + kVisitK);
      if (c < tail_cost * (1.0 - 1e-9)) {
        tail_cost = c;
        tail = t;
      }
    }
  }
  if (tail > 1) {
    g.tail = int(tail);
    g.head = tiles - rem;
    g.ctas = g.head + rem * tail;
  }
  return g;
}

int fill_table(PieceTable& t, int* grid, int64_t n, int64_t m, int64_t k, int bm, int bn, int kq,
               const int32_t* pieces, int n_pieces, int default_p, int flags) {
  const int64_t units[3] = {(n + bm - 1) / bm, (m + bn - 1) / bn, (k + kq - 1) / kq};
  t.ksplit = 0;
  t.grid_s = 0;
  t.grid_tail = 0;
  t.grid_head = 0;
  if (pieces && n_pieces > 0) {
    if (n_pieces > kMaxPieces) {
      set_error("n_pieces=%d exceeds PACO_MAX_PIECES=%d", n_pieces, kMaxPieces);
      return PACO_ERR_ARG;
    }
    t.count = n_pieces;
    for (int i = 0; i < n_pieces; ++i) {
      const int32_t* q = pieces + 6 * i;
      if (q[3] < 1 || q[4] < 1 || q[5] < 1 || q[0] < 0 || q[1] < 0 || q[2] < 0 ||
          q[0] + q[3] > units[0] || q[1] + q[4] > units[1] || q[2] + q[5] > units[2]) {
        set_error("piece %d (%d,%d,%d,%d,%d,%d) is empty or outside the %lldx%lldx%lld unit grid", i,
                  q[0], q[1], q[2], q[3], q[4], q[5], (long long)units[0], (long long)units[1],
                  (long long)units[2]);
        return PACO_ERR_ARG;
      }
      t.p[i] = Piece{q[0], q[1], q[2], q[3], q[4], q[5]};
      t.ksplit |= (q[5] != units[2]);
    }
    *grid = n_pieces;
    return PACO_OK;
  }
  if (!(flags & PACO_MM_PACO_PLAN)) {
    const GridPlan g = grid_plan(units, kq);
    t.count = 0;
    t.grid_s = g.s;
    t.grid_tail = g.tail;
    t.grid_head = int32_t(g.head);
    t.ksplit = g.s > 1 || g.tail > 1;
    *grid = int(g.ctas);
    return PACO_OK;
  }
  // default: the largest feasible p <= default_p, cached per shape
  struct Key {
    int64_t n, m, k;
    int bm, bn, kq, p;
  };
  static thread_local Key last{-1, -1, -1, 0, 0, 0, 0};
  static thread_local int last_p = 0, last_ksplit = 0;
  const int64_t cells = units[0] * units[1] * units[2];
  int p = int(std::min<int64_t>(default_p, cells));
  if (!(last.n == n && last.m == m && last.k == k && last.bm == bm && last.bn == bn && last.kq == kq &&
        last.p == p)) {
    std::vector<Box> boxes;
    int q = p;
    while (q > 1 && !plan_pieces_balanced(n, m, k, bm, bn, kq, q, boxes)) --q;
    if (q <= 1) {
      q = 1;
      plan_pieces_balanced(n, m, k, bm, bn, kq, 1, boxes);
    }
    int ks = 0;
    for (const Box& b : boxes) ks |= (b.e[2] != units[2]);
    last = Key{n, m, k, bm, bn, kq, p};
    last_p = q;
    last_ksplit = ks;
  }
  t.count = 0;
  t.ksplit = last_ksplit;
  *grid = last_p;
  return PACO_OK;
}

// Operands whose view is not 16-byte aligned take the element-granular load
// path (4-8 B cp.async per element), which costs a compute-bound product ~25 %
// (a GPU-level cuboid at column offset 5461 of a 16384-wide B: 63 vs 51 ms).
// Above kRepackTerms the view is first copied into aligned stream-ordered
// scratch (n*k + k*m elements -- noise next to n*m*k terms).
constexpr double kRepackTerms = double(1 << 26);

struct SimtScratch {
  cudaStream_t st = nullptr;
  std::vector<void*> bufs;
  ~SimtScratch() {
    for (void* p : bufs) cudaFreeAsync(p, st);
  }
};

bool aligned16(const void* p, int64_t ld, size_t es) {
  return reinterpret_cast<uintptr_t>(p) % 16 == 0 && (ld * int64_t(es)) % 16 == 0;
}

int repack16(SimtScratch& sc, cudaStream_t st, const void** p, int64_t* ld, int64_t rows, int64_t cols,
             size_t es) {
  if (aligned16(*p, *ld, es) || rows <= 0 || cols <= 0) return PACO_OK;
  const int64_t q = int64_t(16 / es), ld2 = (cols + q - 1) / q * q;
  void* dst = nullptr;
  {  // keep freed scratch cached in the device's default pool
    static std::mutex mu;
    static bool ready[64] = {};
    int dev = 0;
    PACO_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    PACO_CUDA_TRY(cudaStreamIsCapturing(st, &cs));
    if (!ready[dev & 63] && cs == cudaStreamCaptureStatusNone) {  // no pool changes inside a capture
      cudaMemPool_t pool;
      PACO_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
      uint64_t keep = UINT64_MAX;
      PACO_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
      ready[dev & 63] = true;
    }
  }
  sc.st = st;
  PACO_CUDA_TRY(cudaMallocAsync(&dst, size_t(rows) * size_t(ld2) * es, st));
  sc.bufs.push_back(dst);
  PACO_CUDA_TRY(cudaMemcpy2DAsync(dst, size_t(ld2) * es, *p, size_t(*ld) * es, size_t(cols) * es, size_t(rows),
                                  cudaMemcpyDeviceToDevice, st));
  *p = dst;
  *ld = ld2;
  return PACO_OK;
}

template <class Op>
int launch_simt(int device, cudaStream_t stream, const void* A, int64_t lda, const void* B,
                int64_t ldb, void* C, int64_t ldc, int64_t n, int64_t m, int64_t k,
                const int32_t* pieces, int n_pieces, int flags) {
  using Cfg = SimtCfg<Op>;
  SimtScratch sc;  // freed (stream-ordered) after the launch
  if (double(n) * double(m) * double(k) >= kRepackTerms) {
    int rc0 = repack16(sc, stream, &A, &lda, n, k, sizeof(typename Op::TA));
    if (!rc0) rc0 = repack16(sc, stream, &B, &ldb, k, m, sizeof(typename Op::TB));
    if (rc0) return rc0;
  }
  static PieceTable table;  // ~15 KB; copied into the launch's parameter buffer
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int grid = 0;
  int rc = fill_table(table, &grid, n, m, k, Cfg::BM, Cfg::BN, Cfg::KQ, pieces, n_pieces,
                      default_pieces(Cfg::MIN_BLOCKS), flags);
  if (rc) return rc;
  MMArgs args{A, B, C, lda, ldb, ldc, n, m, k, Cfg::KQ, (flags & PACO_MM_OVERWRITE) ? 1 : 0,
              g_trace_buffer,
              (reinterpret_cast<uintptr_t>(C) % 16 == 0 && (ldc * sizeof(typename Op::TC)) % 16 == 0 &&
               !(flags & PACO_MM_REMOTE)) ? 1 : 0,
              (flags & (PACO_MM_ATOMIC | PACO_MM_REMOTE)) ? 1 : 0, plan_kw()};
  args.sys_atomic = (flags & (PACO_MM_REMOTE | PACO_MM_SYS)) ? 1 : 0;
  if (args.overwrite && (flags & (PACO_MM_ATOMIC | PACO_MM_REMOTE))) {
    set_error("PACO_MM_OVERWRITE cannot be combined with atomic / remote folding");
    return PACO_ERR_ARG;
  }
  if (args.overwrite && table.ksplit) {
    // atomics fold into C, so C must first hold the semiring zero
    rc = paco_fill(device, stream, Op::kId, C, ldc, n, m);
    if (rc) return rc;
    args.overwrite = 0;
  }
  const bool vec = (reinterpret_cast<uintptr_t>(A) % 16 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0) &&
                   ((lda * sizeof(typename Op::TA)) % 16 == 0) && ((ldb * sizeof(typename Op::TB)) % 16 == 0);
  static SimtMaps maps;
  bool tma = false;
  if constexpr (Cfg::kTmaOk) {
    // TMA stage loads for aligned operands whose coordinates fit the tensor-map
    // int32 range (PACO_SIMT_TMA=0: per-thread cp.async ring)
    static const bool on = !dev_knob("PACO_SIMT_TMA") || atoi(dev_knob("PACO_SIMT_TMA")) != 0;
    tma = on && vec && n < INT32_MAX && m < INT32_MAX && k < INT32_MAX - 64;
    if (tma) {
      rc = encode_map_2d(&maps.a, 4, A, n, k, lda, Cfg::LDA_S, Cfg::BM);
      if (!rc) rc = encode_map_2d(&maps.b, 4, B, k, m, ldb, Cfg::BN, Cfg::BK);
      if (rc) return rc;
    }
  }
  if constexpr (Op::kId == PACO_SR_F64) {
    // the FP64 tensor pipe (PACO_SIMT_DMMA=0: the DFMA kernel)
    static const bool dmma = !dev_knob("PACO_SIMT_DMMA") || atoi(dev_knob("PACO_SIMT_DMMA")) != 0;
    if (dmma && vec && n < INT32_MAX && m < INT32_MAX && k < INT32_MAX - 64) {
      rc = encode_map_2d(&maps.a, 8, A, n, k, lda, DmmaCfg::LDA_S, DmmaCfg::BM);
      if (!rc) rc = encode_map_2d(&maps.b, 8, B, k, m, ldb, DmmaCfg::LDB_S, DmmaCfg::BK);
      if (rc) return rc;
      PACO_CUDA_TRY(cudaFuncSetAttribute(dmma_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(DmmaCfg::SMEM)));
      {
        KernelSpan ks(PACO_KT_SIMT_MM, stream);
        dmma_f64_kernel<<<grid, DmmaCfg::THREADS, DmmaCfg::SMEM, stream>>>(args, table, maps);
      }
      PACO_CUDA_TRY(cudaGetLastError());
      return PACO_OK;
    }
  }
  auto kern = tma   ? simt_mm_kernel<Op, true, Cfg::kTmaOk>
              : vec ? simt_mm_kernel<Op, true>
                    : simt_mm_kernel<Op, false>;
  PACO_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM)));
  {
    KernelSpan ks(PACO_KT_SIMT_MM, stream);
    kern<<<grid, Cfg::THREADS, Cfg::SMEM, stream>>>(args, table, maps);
  }
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
}

// f64 batch problems of at least this many terms run alone on the DMMA kernel
constexpr double kDmmaAloneTerms = double(1 << 30);  // ~60 us of DMMA work: a whole-GPU plan of its own

template <class Op>
int launch_simt_batch(int device, cudaStream_t stream, int count, const paco_mm_problem* pr) {
  using Cfg = SimtCfg<Op>;
  if constexpr (Op::kId == PACO_SR_F64) {
    // f64 problems big enough to fill the GPU on their own go to the FP64 tensor
    // pipe one launch each (each gets its own all-SM tile-grid plan, so running
    // them back to back loses nothing); the rest stay in one DFMA batch launch
    static const bool dmma = !dev_knob("PACO_SIMT_DMMA") || atoi(dev_knob("PACO_SIMT_DMMA")) != 0;
    if (dmma) {
      paco_mm_problem rest[PACO_MAX_BATCH];
      int nrest = 0;
      for (int q = 0; q < count; ++q) {
        const paco_mm_problem& P = pr[q];
        const bool big = double(P.n) * double(P.m) * double(P.k) >= kDmmaAloneTerms && !(P.flags & PACO_MM_REMOTE) &&
                         !((P.flags & PACO_MM_OVERWRITE) && (P.flags & PACO_MM_ATOMIC));
        if (big) {
          const int rc = launch_simt<Op>(device, stream, P.A, P.lda, P.B, P.ldb, P.C, P.ldc, P.n, P.m, P.k, nullptr,
                                         0, P.flags);
          if (rc) return rc;
        } else {
          rest[nrest++] = P;
        }
      }
      if (nrest < count) {
        if (nrest == 0) return PACO_OK;
        pr = rest;
        count = nrest;
      }
    }
  }
  SimtScratch sc;
  static BatchTable bt;  // ~7.5 KB; copied into the launch's parameter buffer
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  bool vec = true;
  int64_t total = 0;
  int c = 0;
  for (int q = 0; q < count; ++q) {
    const paco_mm_problem& P = pr[q];
    if (P.flags & PACO_MM_REMOTE) {
      set_error("paco_mm_batch: PACO_MM_REMOTE is not supported in a batch");
      return PACO_ERR_UNSUPPORTED;
    }
    if ((P.flags & PACO_MM_OVERWRITE) && (P.flags & PACO_MM_ATOMIC)) {
      set_error("paco_mm_batch: problem %d combines OVERWRITE with ATOMIC", q);
      return PACO_ERR_ARG;
    }
    if (P.n <= 0 || P.m <= 0) continue;
    if (P.k <= 0) {
      if (P.flags & PACO_MM_OVERWRITE) {
        const int rc = paco_fill(device, stream, Op::kId, P.C, P.ldc, P.n, P.m);
        if (rc) return rc;
      }
      continue;
    }
    const void *pa = P.A, *pb = P.B;
    int64_t plda = P.lda, pldb = P.ldb;
    if (double(P.n) * double(P.m) * double(P.k) >= kRepackTerms) {
      int rc0 = repack16(sc, stream, &pa, &plda, P.n, P.k, sizeof(typename Op::TA));
      if (!rc0) rc0 = repack16(sc, stream, &pb, &pldb, P.k, P.m, sizeof(typename Op::TB));
      if (rc0) return rc0;
    }
    const int64_t units[3] = {(P.n + Cfg::BM - 1) / Cfg::BM, (P.m + Cfg::BN - 1) / Cfg::BN,
                              (P.k + Cfg::KQ - 1) / Cfg::KQ};
    const GridPlan g = grid_plan(units, Cfg::KQ);
    const int s = g.s;
    const int64_t ctas = g.ctas;
    MMArgs a{pa, pb, P.C, plda, pldb, P.ldc, P.n, P.m, P.k, Cfg::KQ, (P.flags & PACO_MM_OVERWRITE) ? 1 : 0,
             g_trace_buffer,
             (reinterpret_cast<uintptr_t>(P.C) % 16 == 0 && (P.ldc * sizeof(typename Op::TC)) % 16 == 0) ? 1 : 0,
             (P.flags & PACO_MM_ATOMIC) ? 1 : 0, plan_kw()};
    a.sys_atomic = (P.flags & PACO_MM_SYS) ? 1 : 0;
    if (a.overwrite && (s > 1 || g.tail > 1)) {  // k-split pieces fold into C: it must hold the semiring zero first
      const int rc = paco_fill(device, stream, Op::kId, P.C, P.ldc, P.n, P.m);
      if (rc) return rc;
      a.overwrite = 0;
    }
    vec = vec && aligned16(pa, plda, sizeof(typename Op::TA)) && aligned16(pb, pldb, sizeof(typename Op::TB));
    bt.args[c] = a;
    bt.grid_s[c] = s;
    bt.grid_tail[c] = g.tail;
    bt.grid_head[c] = int32_t(g.head);
    bt.first[c] = total;
    total += ctas;
    ++c;
  }
  bt.count = c;
  bt.first[c] = total;
  if (c == 0) return PACO_OK;
  if (total > INT32_MAX) {
    set_error("paco_mm_batch: %lld CTAs exceed the grid limit", (long long)total);
    return PACO_ERR_ARG;
  }
  auto kern = vec ? simt_mm_batch_kernel<Op, true> : simt_mm_batch_kernel<Op, false>;
  PACO_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM)));
  {
    KernelSpan ks(PACO_KT_SIMT_MM, stream);
    kern<<<unsigned(total), Cfg::THREADS, Cfg::SMEM, stream>>>(bt);
  }
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
}

int launch_mm_simt_batch(int sr, int device, cudaStream_t stream, int count, const paco_mm_problem* problems) {
  return dispatch_op(sr, [&](auto op) -> int {
    using Op = decltype(op);
    if constexpr (Op::kId == PACO_SR_BF16_F32) {
      set_error("paco_mm_batch: bf16 goes through the tcgen05 kernel");
      return PACO_ERR_UNSUPPORTED;
    } else {
      return launch_simt_batch<Op>(device, stream, count, problems);
    }
  });
}

int launch_mm_simt(int sr, int device, cudaStream_t stream, const void* A, int64_t lda, const void* B,
                   int64_t ldb, void* C, int64_t ldc, int64_t n, int64_t m, int64_t k,
                   const int32_t* pieces, int n_pieces, int flags) {
  return dispatch_op(sr, [&](auto op) -> int {
    using Op = decltype(op);
    if constexpr (Op::kId == PACO_SR_BF16_F32) {
      set_error("bf16 goes through the tcgen05 kernel");
      return PACO_ERR_UNSUPPORTED;
    } else {
      return launch_simt<Op>(device, stream, A, lda, B, ldb, C, ldc, n, m, k, pieces, n_pieces, flags);
    }
  });
}

int simt_tile_shape(int sr, int* bm, int* bn, int* bk, int* cps) {
  return dispatch_op(sr, [&](auto op) -> int {
    using Cfg = SimtCfg<decltype(op)>;
    *bm = Cfg::BM;
    *bn = Cfg::BN;
    *bk = Cfg::KQ;
    *cps = Cfg::MIN_BLOCKS;
    return PACO_OK;
  });
}

}  // namespace paco

extern "C" int paco_debug_trace(void* device_buffer) {
  paco::g_trace_buffer = static_cast<long long*>(device_buffer);
  return PACO_OK;
}

extern "C" int paco_plan_one_piece(int64_t n, int64_t m, int64_t k, int p, int64_t* out) {
  using namespace paco;
  if (p < 1 || !out || n < 1 || m < 1 || k < 1) {
    set_error("paco_plan_one_piece: need extents >= 1, p >= 1 and an output buffer");
    return PACO_ERR_ARG;
  }
  std::vector<Box> boxes;
  if (!plan_pieces(n, m, k, p, boxes)) {
    set_error("extents too small to give every worker a nonempty piece");
    return PACO_ERR_ARG;
  }
  for (int i = 0; i < p; ++i)
    for (int d = 0; d < 3; ++d) {
      out[6 * i + d] = boxes[i].o[d];
      out[6 * i + 3 + d] = boxes[i].e[d];
    }
  return PACO_OK;
}

extern "C" int paco_cta_grid(int semiring, int64_t n, int64_t m, int64_t k, int* ksplit, int64_t* ctas) {
  using namespace paco;
  int bm, bn, kq, cps;
  int rc = paco_mm_tile_shape(semiring, &bm, &bn, &kq, &cps);
  if (rc) return rc;
  if (n < 1 || m < 1 || k < 1 || !ksplit || !ctas) {
    set_error("paco_cta_grid: need extents >= 1 and output pointers");
    return PACO_ERR_ARG;
  }
  const int64_t units[3] = {(n + bm - 1) / bm, (m + bn - 1) / bn, (k + kq - 1) / kq};
  const GridPlan g = grid_plan(units, kq);
  *ksplit = g.s;
  *ctas = g.ctas;
  return PACO_OK;
}

extern "C" int paco_cta_grid_tail(int semiring, int64_t n, int64_t m, int64_t k, int* tail, int64_t* head) {
  using namespace paco;
  int bm, bn, kq, cps;
  int rc = paco_mm_tile_shape(semiring, &bm, &bn, &kq, &cps);
  if (rc) return rc;
  if (n < 1 || m < 1 || k < 1 || !tail || !head) {
    set_error("paco_cta_grid_tail: need extents >= 1 and output pointers");
    return PACO_ERR_ARG;
  }
  const int64_t units[3] = {(n + bm - 1) / bm, (m + bn - 1) / bn, (k + kq - 1) / kq};
  const GridPlan g = grid_plan(units, kq);
  *tail = g.tail;
  *head = g.head;
  return PACO_OK;
}

extern "C" int paco_plan_cta(int semiring, int64_t n, int64_t m, int64_t k, int p, int32_t* out) {
  using namespace paco;
  int bm, bn, kq, cps;
  int rc = paco_mm_tile_shape(semiring, &bm, &bn, &kq, &cps);
  if (rc) return rc;
  if (p < 1 || !out || n < 1 || m < 1 || k < 1) {
    set_error("paco_plan_cta: need extents >= 1, p >= 1 and an output buffer");
    return PACO_ERR_ARG;
  }
  std::vector<Box> boxes;
  if (!plan_pieces_balanced(n, m, k, bm, bn, kq, p, boxes)) {
    set_error("extents too small to give every worker a nonempty piece");
    return PACO_ERR_ARG;
  }
  for (int i = 0; i < p; ++i)
    for (int d = 0; d < 3; ++d) {
      out[6 * i + d] = int32_t(boxes[i].o[d]);
      out[6 * i + 3 + d] = int32_t(boxes[i].e[d]);
    }
  return PACO_OK;
}
