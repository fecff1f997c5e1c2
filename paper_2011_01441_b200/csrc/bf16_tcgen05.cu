// bf16 x bf16 -> fp32 (+,x) MM on the 5th-generation tensor cores (cfg3).
//
// Replaces SEMIRING_F64.block_mm / _int_block (matmul.py:45-46,54) for the
// dense bf16 case.  One persistent CTA per SM, warp-specialised:
//   warp 0      TMA producer: A tile [128 x 64] (K-major) and B tile
//               [64 x 256] (N-major, as the caller stores it) per k block,
//               128B-swizzled, into a 4-stage smem ring; when K fits the ring
//               (K <= 256) B stays resident across consecutive tiles of the
//               same column block;
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma.kind::f16
//               (M=128, N=256, K=16) into a double-buffered TMEM accumulator
//               (2 x 256 fp32 columns) and commits to mbarriers;
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 -> registers -> swizzled smem
//               staging -> TMA tensor store (C = AB) or TMA reduce-add
//               (C += AB), overlapping the next tile's MMAs.
// The CTA-level plan is the 1-D MM-1-Piece split of the column-block-major
// tile sequence over the 148 CTAs (floor(p/2):ceil(p/2) halving of a 1-D
// range == contiguous ranges of floor/ceil(T/p) tiles), which keeps each
// CTA on one B column block.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace paco {

namespace tc {

constexpr int BM = 128, BN = 256, BK = 64, UMMA_K = 16;
constexpr int STAGES = 4;
constexpr int THREADS = 192;  // 6 warps
constexpr int A_BYTES = BM * BK * 2;        // 16 KB
constexpr int B_BYTES = BN * BK * 2;        // 32 KB
constexpr int EPI_BUF = 32 * 32 * 4;        // 4 KB: 32 rows x 32 fp32 (128 B)
constexpr int SMEM_A = 0;
constexpr int SMEM_B = SMEM_A + STAGES * A_BYTES;
constexpr int SMEM_EPI = SMEM_B + STAGES * B_BYTES;
constexpr int SMEM_BAR = SMEM_EPI + 4 * 2 * EPI_BUF;
constexpr int SMEM_TOTAL = SMEM_BAR + 256;
constexpr int SMEM_ALLOC = SMEM_TOTAL + 1024;  // runtime 1024-B alignment slack
constexpr uint32_t TMEM_COLS = 512;

// instruction descriptor: F32 accumulate, BF16 A/B, A K-major, B MN-major
// (bit 16), N=256, M=128
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(BN >> 3) << 17) |
                            (uint32_t(BM >> 4) << 24);

__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  // K-major, 128B swizzle: rows of 128 B, 8-row groups 1024 B apart (SBO),
  // LBO unused (1), version 1 (sm_100), layout type 2 = SWIZZLE_128B.
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

// MN-major (N contiguous), 128B swizzle, canonical ((8,n),(8,k)):((1,LBO),(8,SBO))
// in 16 B units: 64 N-elements per 128 B row, rows = k; 8-row (1024 B) atoms
// step along k by SBO; 64-wide N chunks (one TMA box of BK rows each) step by LBO.
__device__ __forceinline__ uint64_t smem_desc_mn_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((BK * 128) >> 4) << 16;  // LBO: next 64-wide N chunk
  d |= uint64_t(1024 >> 4) << 32;        // SBO: next 8 k-rows
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// Bounded wait: traps instead of hanging the GPU if a phase never completes.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  for (uint32_t tries = 0;; ++tries) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) return;
    if (tries > (1u << 24)) __trap();
  }
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

struct TcArgs {
  int64_t n, m, k;   // C is n x m
  int32_t a_col0;    // column offset of A inside its aligned tensor map
  int32_t b_col0;    // column offset of B inside its aligned tensor map
  int32_t c_col0;    // column offset of C inside its aligned tensor map
  int32_t overwrite;
  int32_t tiles_rb;  // row blocks
  int32_t tiles_nb;  // column blocks
  int32_t kblocks;
};

__global__ void __launch_bounds__(THREADS, 1)
    bf16_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_c, const TcArgs args) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SMEM_BAR);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  // CTA-level plan: contiguous range of the column-block-major tile sequence
  const int64_t T = int64_t(args.tiles_rb) * args.tiles_nb;
  const int64_t t_begin = T * blockIdx.x / gridDim.x, t_end = T * (blockIdx.x + 1) / gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_c)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      const bool can_keep_b = args.kblocks == STAGES;
      int resident_nb = -1;
      uint32_t it = 0;
      for (int64_t t = t_begin; t < t_end; ++t) {
        const int nb = int(t / args.tiles_rb), rb = int(t % args.tiles_rb);
        const bool keep_b = can_keep_b && nb == resident_nb;
        for (int kb = 0; kb < args.kblocks; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          mbar_expect_tx(&full[s], keep_b ? A_BYTES : A_BYTES + B_BYTES);
          tma_load_2d(smem + SMEM_A + s * A_BYTES, &map_a, &full[s], args.a_col0 + kb * BK, rb * BM);
          if (!keep_b) {
            // B is k x m row-major (N contiguous): 4 boxes of [64 k rows][64 n]
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(smem + SMEM_B + s * B_BYTES + j * (BK * 128), &map_b, &full[s],
                          args.b_col0 + nb * BN + 64 * j, kb * BK);
          }
        }
        resident_nb = can_keep_b ? nb : -1;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      uint32_t it = 0;
      int tile = 0;
      for (int64_t t = t_begin; t < t_end; ++t, ++tile) {
        const int a = tile & 1;
        const uint32_t use = uint32_t(tile >> 1);
        mbar_wait(&tempty[a], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + uint32_t(a * BN);
        for (int kb = 0; kb < args.kblocks; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint64_t ad = smem_desc_sw128(smem_u32(smem + SMEM_A + s * A_BYTES));
          const uint64_t bd = smem_desc_mn_sw128(smem_u32(smem + SMEM_B + s * B_BYTES));
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; ++kk) {
            // A (K-major): +32 B inside the 128 B swizzle row = +2 units;
            // B (MN-major): +16 k rows = 2 atoms of 1024 B = +128 units
            umma_bf16(d_tmem, ad + uint64_t(2 * kk), bd + uint64_t(128 * kk), (kb | kk) != 0);
          }
          umma_commit(&empty[s]);  // stage is free once these MMAs complete
        }
        umma_commit(&tfull[a]);    // accumulator ready for the epilogue
      }
    }
  } else {
    // ---------------- epilogue warps ----------------
    const int q = warp % 4;  // TMEM lane quadrant this warp may access
    unsigned char* stage0 = smem + SMEM_EPI + q * 2 * EPI_BUF;
    int tile = 0;
    uint32_t nstore = 0;
    for (int64_t t = t_begin; t < t_end; ++t, ++tile) {
      const int nb = int(t / args.tiles_rb), rb = int(t % args.tiles_rb);
      const int a = tile & 1;
      const uint32_t use = uint32_t(tile >> 1);
      mbar_wait(&tfull[a], use & 1);
      tc_fence_after();
      const int row0 = rb * BM + 32 * q;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        const uint32_t taddr = tmem_base + (uint32_t(32 * q) << 16) + uint32_t(a * BN + 32 * c);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (c == BN / 32 - 1) {
          // all of this warp's TMEM reads for the tile are done: release the buffer
          tc_fence_before();
          if (lane == 0) mbar_arrive(&tempty[a]);
        }
        const int col0 = nb * BN + 32 * c;
        if (col0 >= args.m) continue;  // warp-uniform: nothing left to store
        unsigned char* buf = stage0 + (nstore & 1) * EPI_BUF;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
        __syncwarp();
        // 128B-swizzled [32 rows][32 fp32] staging: 16 B chunk j of row r at (j ^ r%8)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint4 w = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          *reinterpret_cast<uint4*>(buf + lane * 128 + ((j ^ (lane & 7)) * 16)) = w;
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if (row0 < args.n) {
            if (args.overwrite)
              tma_store_2d(&map_c, buf, args.c_col0 + col0, row0);
            else
              tma_reduce_add_2d(&map_c, buf, args.c_col0 + col0, row0);
          }
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
        ++nstore;
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(TMEM_COLS));
}

}  // namespace tc

namespace {
PFN_cuTensorMapEncodeTiled_v12000 get_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D row-major tensor map over an aligned base; `col_off` returns how many
// elements the view starts after that base (added to column coordinates).
int make_map(CUtensorMap* map, CUtensorMapDataType dt, int elsize, const void* ptr, int64_t rows,
             int64_t cols, int64_t ld, uint32_t box_cols, uint32_t box_rows, int32_t* col_off) {
  auto enc = get_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled is unavailable from the driver");
    return PACO_ERR_CUDA;
  }
  const uintptr_t p = reinterpret_cast<uintptr_t>(ptr);
  const uintptr_t base = p & ~uintptr_t(15);
  if ((p - base) % elsize != 0 || (ld * elsize) % 16 != 0) {  // callers repack first
    set_error("internal: tensor map needs a 16-byte row pitch (ld*%d %% 16 == 0)", elsize);
    return PACO_ERR_UNSUPPORTED;
  }
  *col_off = int32_t((p - base) / elsize);
  cuuint64_t dims[2] = {cuuint64_t(cols + *col_off), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld * elsize)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, dt, 2, reinterpret_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) for %lldx%lld ld=%lld", int(r), (long long)rows,
              (long long)cols, (long long)ld);
    return PACO_ERR_CUDA;
  }
  return PACO_OK;
}

// Per-device scratch for operands whose row pitch is not a multiple of 16 B
// (TMA needs it): they are repacked with a padded pitch.  Grown on demand.
struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
};
std::mutex g_scratch_mu;
Scratch g_scratch[64][3];

int scratch(int device, int slot, size_t bytes, cudaStream_t st, void** out) {
  std::lock_guard<std::mutex> lock(g_scratch_mu);
  Scratch& w = g_scratch[device & 63][slot];
  if (w.bytes < bytes) {
    if (w.ptr) {
      PACO_CUDA_TRY(cudaStreamSynchronize(st));
      PACO_CUDA_TRY(cudaFree(w.ptr));
      w = Scratch{};
    }
    PACO_CUDA_TRY(cudaMalloc(&w.ptr, bytes));
    w.bytes = bytes;
  }
  *out = w.ptr;
  return PACO_OK;
}

bool pitch_ok(const void* p, int64_t ld, int elsize) {
  return (reinterpret_cast<uintptr_t>(p) % elsize == 0) && (ld * elsize) % 16 == 0;
}
}  // namespace

int launch_mm_bf16_tc(int device, cudaStream_t stream, const void* A, int64_t lda, const void* B, int64_t ldb,
                      void* C, int64_t ldc, int64_t n, int64_t m, int64_t k, const int32_t* pieces,
                      int n_pieces, int flags) {
  if (pieces && n_pieces > 0) {
    set_error("the tcgen05 bf16 kernel takes its own CTA plan (pass pieces=NULL)");
    return PACO_ERR_UNSUPPORTED;
  }
  if (n > INT32_MAX || m > INT32_MAX || k > INT32_MAX) {
    set_error("tcgen05 bf16 path: extents must fit int32");
    return PACO_ERR_ARG;
  }
  CUtensorMap ma, mb, mc;
  int rc;
  int32_t a_off = 0, b_off = 0, c_off = 0;
  // operands with a row pitch TMA cannot take are repacked into padded scratch
  if (!pitch_ok(A, lda, 2)) {
    const int64_t ld2 = (k + 7) / 8 * 8;
    void* p;
    if ((rc = scratch(device, 0, size_t(n) * ld2 * 2, stream, &p))) return rc;
    PACO_CUDA_TRY(cudaMemcpy2DAsync(p, ld2 * 2, A, lda * 2, k * 2, n, cudaMemcpyDeviceToDevice, stream));
    A = p;
    lda = ld2;
  }
  if (!pitch_ok(B, ldb, 2)) {
    const int64_t ld2 = (m + 7) / 8 * 8;
    void* p;
    if ((rc = scratch(device, 1, size_t(k) * ld2 * 2, stream, &p))) return rc;
    PACO_CUDA_TRY(cudaMemcpy2DAsync(p, ld2 * 2, B, ldb * 2, m * 2, k, cudaMemcpyDeviceToDevice, stream));
    B = p;
    ldb = ld2;
  }
  void* c_user = nullptr;
  int64_t ldc_user = ldc;
  if (!pitch_ok(C, ldc, 4)) {
    const int64_t ld2 = (m + 3) / 4 * 4;
    void* p;
    if ((rc = scratch(device, 2, size_t(n) * ld2 * 4, stream, &p))) return rc;
    if (!(flags & PACO_MM_OVERWRITE))
      PACO_CUDA_TRY(cudaMemcpy2DAsync(p, ld2 * 4, C, ldc * 4, m * 4, n, cudaMemcpyDeviceToDevice, stream));
    c_user = C;
    C = p;
    ldc = ld2;
  }
  if ((rc = make_map(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, A, n, k, lda, tc::BK, tc::BM, &a_off))) return rc;
  if ((rc = make_map(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, k, m, ldb, 64, tc::BK, &b_off))) return rc;
  if ((rc = make_map(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, C, n, m, ldc, 32, 32, &c_off))) return rc;
  tc::TcArgs args;
  args.n = n;
  args.m = m;
  args.k = k;
  args.a_col0 = a_off;
  args.b_col0 = b_off;
  args.c_col0 = c_off;
  args.overwrite = (flags & PACO_MM_OVERWRITE) ? 1 : 0;
  args.tiles_rb = int32_t((n + tc::BM - 1) / tc::BM);
  args.tiles_nb = int32_t((m + tc::BN - 1) / tc::BN);
  args.kblocks = int32_t((k + tc::BK - 1) / tc::BK);
  const int64_t tiles = int64_t(args.tiles_rb) * args.tiles_nb;
  const int grid = int(tiles < kNumSMs ? tiles : kNumSMs);
  PACO_CUDA_TRY(cudaFuncSetAttribute(tc::bf16_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_ALLOC));
  tc::bf16_tc_kernel<<<grid, tc::THREADS, tc::SMEM_ALLOC, stream>>>(ma, mb, mc, args);
  PACO_CUDA_TRY(cudaGetLastError());
  if (c_user)
    PACO_CUDA_TRY(cudaMemcpy2DAsync(c_user, ldc_user * 4, C, ldc * 4, m * 4, n, cudaMemcpyDeviceToDevice, stream));
  return PACO_OK;
}

int bf16_tile_shape(int* bm, int* bn, int* bk, int* cps) {
  *bm = tc::BM;
  *bn = tc::BN;
  *bk = tc::BK;
  *cps = 1;
  return PACO_OK;
}

}  // namespace paco
