// Register-blocked SIMT semiring MM for sm_100a (tropical / integer / fp32 / fp64).
//
// Replaces the reference's recursive mm_seq + 32^3 NumPy leaves
// (matmul.py:342-397, block kernels 45-50) with one persistent launch:
//   * grid = the CTA-level PACO plan: one CTA per MM-1-Piece cuboid over the
//     tile grid (148 SMs x resident CTAs), see plan_pieces() below;
//   * each CTA walks the C tiles of its cuboid; per tile it streams its k
//     range through a STAGES-deep cp.async ring (16 B, zero-filled at edges);
//   * a 16x16 thread grid holds TMxTN register accumulators per thread, fed by
//     128-bit LDS from padded, bank-conflict-free shared tiles;
//   * epilogue: C (+)= acc, or one global atomic (+) per element for pieces
//     that split k (exact for the integer/tropical semirings, order-free).
// The tropical inner loop is one VIADDMNMX per term (checked in SASS).
#include <algorithm>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "semiring_ops.cuh"

namespace paco {

template <class Op>
struct SimtCfg {
  static constexpr bool kWide = sizeof(typename Op::Acc) == 8;
  static constexpr int BM = kWide ? 64 : 128;
  static constexpr int BN = kWide ? 64 : 128;
  static constexpr int BK = kWide ? 16 : 32;
  static constexpr int GM = BM / 64;  // 4-row groups per thread along m
  static constexpr int GN = BN / 64;
  static constexpr int TM = 4 * GM;
  static constexpr int TN = 4 * GN;
  static constexpr int THREADS = 256;
  static constexpr int STAGES = kWide ? 4 : 3;
  static constexpr int MIN_BLOCKS = kWide ? 2 : 2;
  static constexpr int VA = 16 / sizeof(typename Op::TA);  // elements per 16 B chunk
  static constexpr int VB = 16 / sizeof(typename Op::TB);
  static constexpr int LDA_S = BK + VA;  // padded smem row (k-major rows of A)
  static constexpr int LDB_S = BN;
  static constexpr int A_STAGE = BM * LDA_S;
  static constexpr int B_STAGE = BK * LDB_S;
  static constexpr size_t SMEM =
      size_t(STAGES) * (A_STAGE * sizeof(typename Op::TA) + B_STAGE * sizeof(typename Op::TB));
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
  int32_t k_tiles;  // total k tiles of the problem
  int32_t overwrite;
};

// Stage one (tile, k-tile) pair of A and B into shared memory.
template <class Op, bool kVec>
__device__ __forceinline__ void load_stage(const MMArgs& a, typename Op::TA* As, typename Op::TB* Bs,
                                           int64_t row0, int64_t col0, int64_t k0) {
  using C = SimtCfg<Op>;
  using TA = typename Op::TA;
  using TB = typename Op::TB;
  const TA* A = static_cast<const TA*>(a.A);
  const TB* B = static_cast<const TB*>(a.B);
  const int tid = threadIdx.x;
  if constexpr (kVec) {
    constexpr int A_CHUNKS_ROW = C::BK / C::VA;
    constexpr int A_ITERS = C::BM * A_CHUNKS_ROW / C::THREADS;
#pragma unroll
    for (int it = 0; it < A_ITERS; ++it) {
      const int c = tid + it * C::THREADS;
      const int r = c / A_CHUNKS_ROW, kc = (c % A_CHUNKS_ROW) * C::VA;
      const int64_t gr = row0 + r, gk = k0 + kc;
      int bytes = 0;
      const TA* src = A;
      if (gr < a.n && gk < a.k) {
        bytes = int((a.k - gk < C::VA ? a.k - gk : C::VA) * sizeof(TA));
        src = A + gr * a.lda + gk;
      }
      cp_async16(As + r * C::LDA_S + kc, src, bytes);
    }
    constexpr int B_CHUNKS_ROW = C::BN / C::VB;
    constexpr int B_ITERS = C::BK * B_CHUNKS_ROW / C::THREADS;
#pragma unroll
    for (int it = 0; it < B_ITERS; ++it) {
      const int c = tid + it * C::THREADS;
      const int r = c / B_CHUNKS_ROW, nc = (c % B_CHUNKS_ROW) * C::VB;
      const int64_t gk = k0 + r, gc = col0 + nc;
      int bytes = 0;
      const TB* src = B;
      if (gk < a.k && gc < a.m) {
        bytes = int((a.m - gc < C::VB ? a.m - gc : C::VB) * sizeof(TB));
        src = B + gk * a.ldb + gc;
      }
      cp_async16(Bs + r * C::LDB_S + nc, src, bytes);
    }
  } else {
    // element-granular path for views that are not 16 B aligned
    constexpr int A_ITERS = C::BM * C::BK / C::THREADS;
#pragma unroll 4
    for (int it = 0; it < A_ITERS; ++it) {
      const int c = tid + it * C::THREADS;
      const int r = c / C::BK, kc = c % C::BK;
      const int64_t gr = row0 + r, gk = k0 + kc;
      const bool ok = gr < a.n && gk < a.k;
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
      const bool ok = gk < a.k && gc < a.m;
      const TB* src = ok ? B + gk * a.ldb + gc : B;
      if constexpr (sizeof(TB) == 4)
        cp_async4(Bs + r * C::LDB_S + nc, src, ok ? 4 : 0);
      else
        cp_async8(Bs + r * C::LDB_S + nc, src, ok ? 8 : 0);
    }
  }
}

// acc[i][j] = acc (+) A[row_i][k] (x) B[k][col_j] over `kvalid` k of the stage.
template <class Op, bool kFull>
__device__ __forceinline__ void compute_stage(typename Op::Acc (&acc)[SimtCfg<Op>::TM][SimtCfg<Op>::TN],
                                              const typename Op::TA* As, const typename Op::TB* Bs,
                                              int kvalid) {
  using C = SimtCfg<Op>;
  using TA = typename Op::TA;
  using TB = typename Op::TB;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const TA* a_base = As + (ty * 4) * C::LDA_S;
  const TB* b_base = Bs + tx * 4;
  if constexpr (kFull) {
#pragma unroll
    for (int kk = 0; kk < C::BK; kk += 4) {
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
  } else {
    for (int kk = 0; kk < kvalid; ++kk) {
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
}

template <class Op>
__device__ __forceinline__ void epilogue(const MMArgs& a,
                                         typename Op::Acc (&acc)[SimtCfg<Op>::TM][SimtCfg<Op>::TN],
                                         int64_t row0, int64_t col0, bool atomic) {
  using C = SimtCfg<Op>;
  using TC = typename Op::TC;
  TC* Cp = static_cast<TC*>(a.C);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
#pragma unroll
  for (int i = 0; i < C::TM; ++i) {
    const int64_t gr = row0 + (i / 4) * 64 + ty * 4 + (i % 4);
    if (gr >= a.n) continue;
    TC* crow = Cp + gr * a.ldc;
#pragma unroll
    for (int j = 0; j < C::TN; ++j) {
      const int64_t gc = col0 + (j / 4) * 64 + tx * 4 + (j % 4);
      if (gc >= a.m) continue;
      const TC v = Op::finish(acc[i][j]);
      if (atomic)
        Op::atomic_combine(crow + gc, v);
      else if (a.overwrite)
        crow[gc] = v;
      else
        crow[gc] = Op::combine(crow[gc], v);
    }
  }
}

template <class Op, bool kVec>
__global__ void __launch_bounds__(SimtCfg<Op>::THREADS, SimtCfg<Op>::MIN_BLOCKS)
    simt_mm_kernel(const MMArgs args, const __grid_constant__ PieceTable table) {
  using C = SimtCfg<Op>;
  using TA = typename Op::TA;
  using TB = typename Op::TB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TA* As = reinterpret_cast<TA*>(smem_raw);
  TB* Bs = reinterpret_cast<TB*>(smem_raw + size_t(C::STAGES) * C::A_STAGE * sizeof(TA));

  const Piece pc = table.p[blockIdx.x];
  const bool atomic = pc.tk != args.k_tiles;
  const int KT = pc.tk;
  const int total = pc.tn * pc.tm * KT;

  auto coords = [&](int it, int64_t& row0, int64_t& col0, int64_t& k0) {
    const int tile = it / KT, kt = it - tile * KT;
    const int ti = tile / pc.tm, tj = tile - ti * pc.tm;
    row0 = int64_t(pc.ti0 + ti) * C::BM;
    col0 = int64_t(pc.tj0 + tj) * C::BN;
    k0 = int64_t(pc.tl0 + kt) * C::BK;
  };

#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < total) {
      int64_t r0, c0, k0;
      coords(s, r0, c0, k0);
      load_stage<Op, kVec>(args, As + s * C::A_STAGE, Bs + s * C::B_STAGE, r0, c0, k0);
    }
    cp_async_commit();
  }

  typename Op::Acc acc[C::TM][C::TN];
#pragma unroll
  for (int i = 0; i < C::TM; ++i)
#pragma unroll
    for (int j = 0; j < C::TN; ++j) acc[i][j] = Op::identity();

  for (int it = 0; it < total; ++it) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    {
      const int nxt = it + C::STAGES - 1;
      if (nxt < total) {
        int64_t r0, c0, k0;
        coords(nxt, r0, c0, k0);
        const int s = nxt % C::STAGES;
        load_stage<Op, kVec>(args, As + s * C::A_STAGE, Bs + s * C::B_STAGE, r0, c0, k0);
      }
      cp_async_commit();
    }
    int64_t r0, c0, k0;
    coords(it, r0, c0, k0);
    const int s = it % C::STAGES;
    const int64_t krem = args.k - k0;
    if (krem >= C::BK)
      compute_stage<Op, true>(acc, As + s * C::A_STAGE, Bs + s * C::B_STAGE, C::BK);
    else
      compute_stage<Op, false>(acc, As + s * C::A_STAGE, Bs + s * C::B_STAGE, int(krem));
    if ((it + 1) % KT == 0) {
      epilogue<Op>(args, acc, r0, c0, atomic);
#pragma unroll
      for (int i = 0; i < C::TM; ++i)
#pragma unroll
        for (int j = 0; j < C::TN; ++j) acc[i][j] = Op::identity();
    }
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// CTA-level PACO: MM-1-Piece over the tile grid (host side).
//
// Same recursion as mm_one_piece_partition (matmul.py:250-300): the worker
// list splits floor(p/2):ceil(p/2); the cut axis is the longest axis of an
// evenly-halved virtual cuboid (ties n -> m -> k); the real length is split
// max(1, len*a // (a+b)).  Here the virtual cuboid is in ELEMENTS while the
// real cut is in TILES, so pieces stay cube-like in the iteration space and
// every cut lands on a tile boundary.  With unit tiles it is exactly the
// reference rule (paco_plan_one_piece, pinned by the CPU tests).
// ---------------------------------------------------------------------------
namespace {
struct Box {
  int64_t o[3];  // offsets (tiles)
  int64_t e[3];  // extents (tiles)
};

bool one_piece_rec(const Box& b, int lo_w, int hi_w, double vn, double vm, double vk,
                   std::vector<Box>& out) {
  const int cnt = hi_w - lo_w;
  if (cnt == 1) {
    out[lo_w] = b;
    return true;
  }
  const int h = cnt / 2;  // left list is the smaller one
  int axis;
  if (vn >= vm && vn >= vk)
    axis = 0;
  else
    axis = vm >= vk ? 1 : 2;
  const int64_t len = b.e[axis];
  if (len < 2) return false;
  const int64_t left = std::max<int64_t>(1, len * h / cnt);
  Box lo = b, hi = b;
  lo.e[axis] = left;
  hi.o[axis] += left;
  hi.e[axis] = len - left;
  double v[3] = {vn, vm, vk};
  v[axis] /= 2;
  return one_piece_rec(lo, lo_w, lo_w + h, v[0], v[1], v[2], out) &&
         one_piece_rec(hi, lo_w + h, hi_w, v[0], v[1], v[2], out);
}
}  // namespace

// Tile-quantised MM-1-Piece plan; returns false when p pieces do not fit.
bool plan_pieces(int64_t n, int64_t m, int64_t k, int bm, int bn, int bk, int p, std::vector<Box>& out) {
  out.assign(p, Box{});
  Box root{{0, 0, 0}, {(n + bm - 1) / bm, (m + bn - 1) / bn, (k + bk - 1) / bk}};
  return one_piece_rec(root, 0, p, double(n), double(m), double(k), out);
}

int fill_table(PieceTable& t, int64_t n, int64_t m, int64_t k, int bm, int bn, int bk, int k_tiles,
               const int32_t* pieces, int n_pieces, int default_p) {
  if (pieces && n_pieces > 0) {
    if (n_pieces > kMaxPieces) {
      set_error("n_pieces=%d exceeds PACO_MAX_PIECES=%d", n_pieces, kMaxPieces);
      return PACO_ERR_ARG;
    }
    t.count = n_pieces;
    for (int i = 0; i < n_pieces; ++i) {
      const int32_t* q = pieces + 6 * i;
      t.p[i] = Piece{q[0], q[1], q[2], q[3], q[4], q[5]};
      if (q[3] < 1 || q[4] < 1 || q[5] < 1) {
        set_error("piece %d has an empty extent", i);
        return PACO_ERR_ARG;
      }
    }
  } else {
    const int64_t tiles = ((n + bm - 1) / bm) * ((m + bn - 1) / bn) * int64_t(k_tiles);
    int p = int(std::min<int64_t>(std::min(default_p, kMaxPieces), tiles));
    std::vector<Box> boxes;
    while (p > 1 && !plan_pieces(n, m, k, bm, bn, bk, p, boxes)) --p;
    if (p <= 1) plan_pieces(n, m, k, bm, bn, bk, 1, boxes);
    t.count = p;
    for (int i = 0; i < p; ++i) {
      const Box& b = boxes[i];
      t.p[i] = Piece{int32_t(b.o[0]), int32_t(b.o[1]), int32_t(b.o[2]),
                     int32_t(b.e[0]), int32_t(b.e[1]), int32_t(b.e[2])};
    }
  }
  t.ksplit = 0;
  for (int i = 0; i < t.count; ++i) t.ksplit |= (t.p[i].tk != k_tiles);
  return PACO_OK;
}

template <class Op>
int launch_simt(int device, cudaStream_t stream, const void* A, int64_t lda, const void* B,
                int64_t ldb, void* C, int64_t ldc, int64_t n, int64_t m, int64_t k,
                const int32_t* pieces, int n_pieces, int flags) {
  using Cfg = SimtCfg<Op>;
  static PieceTable table;  // large; guarded by the mutex below
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  const int k_tiles = int((k + Cfg::BK - 1) / Cfg::BK);
  int rc = fill_table(table, n, m, k, Cfg::BM, Cfg::BN, Cfg::BK, k_tiles, pieces, n_pieces,
                      kNumSMs * Cfg::MIN_BLOCKS);
  if (rc) return rc;
  MMArgs args{A, B, C, lda, ldb, ldc, n, m, k, k_tiles, (flags & PACO_MM_OVERWRITE) ? 1 : 0};
  if (args.overwrite && table.ksplit) {
    // atomics fold into C, so C must first hold the semiring zero
    rc = paco_fill(device, stream, Op::kId, C, ldc, n, m);
    if (rc) return rc;
    args.overwrite = 0;
  }
  const bool vec = (reinterpret_cast<uintptr_t>(A) % 16 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0) &&
                   ((lda * sizeof(typename Op::TA)) % 16 == 0) && ((ldb * sizeof(typename Op::TB)) % 16 == 0);
  auto kern = vec ? simt_mm_kernel<Op, true> : simt_mm_kernel<Op, false>;
  PACO_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM)));
  kern<<<table.count, Cfg::THREADS, Cfg::SMEM, stream>>>(args, table);
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
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
    *bk = Cfg::BK;
    *cps = Cfg::MIN_BLOCKS;
    return PACO_OK;
  });
}

}  // namespace paco

extern "C" int paco_plan_one_piece(int64_t n, int64_t m, int64_t k, int p, int64_t* out) {
  using namespace paco;
  if (p < 1 || !out || n < 1 || m < 1 || k < 1) {
    set_error("paco_plan_one_piece: need extents >= 1, p >= 1 and an output buffer");
    return PACO_ERR_ARG;
  }
  std::vector<Box> boxes;
  if (!plan_pieces(n, m, k, 1, 1, 1, p, boxes)) {
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
