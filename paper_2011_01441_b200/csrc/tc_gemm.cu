// (+,x) MM on the 5th-generation tensor cores: bf16 x bf16 -> fp32 (cfg3) and
// fp32 x fp32 -> fp32 as 3xTF32 (Strassen leaves, cfg5).
//
// Replaces SEMIRING_F64.block_mm / _int_block (matmul.py:45-46,54) for the
// dense floating-point case.  One persistent CTA per SM, warp-specialised:
//   warp 0      TMA producer: claims tiles from a global counter (dynamic
//               schedule, see claim_tile) and loads A tiles [128 x 64]
//               (K-major) and B tiles [64 x 256] (N-major, as the caller
//               stores it), 128B-swizzled, into a smem ring; with K <= 256
//               (cfg3) the CTA's whole B column block stays resident and only
//               A streams;
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma.kind::f16
//               (M=128, N=256, K=16) into a double-buffered TMEM accumulator
//               (2 x 256 fp32 columns) and commits to mbarriers;
//   warps 2..   epilogue: tcgen05.ld 32x32b.x64 -> registers -> swizzled smem
//               staging -> TMA tensor store (C = AB) or TMA reduce-add
//               (C += AB), overlapping the next tile's MMAs.
//
// 3xTF32: every fp32 operand x is split (by split_tf32_kernel) into
// hi = tf32_rn(x) and lo = tf32_rn(x - hi) (|x - hi - lo| <= 2^-22 |x|; a
// truncated split leaves lo's low bits to the MMA's truncation: 20x the
// error); C += Ahi*Bhi + Ahi*Blo + Alo*Bhi with kind::tf32 MMAs accumulating
// in fp32 TMEM -- ~fp32 accuracy (the dropped Alo*Blo term is < 2^-22
// relative) at tensor-core rate.  The split writes B
// transposed (K-major): kind::tf32 with an MN-major B descriptor returned
// zeros on this toolchain/hardware, K-major both sides is exact.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <atomic>
#include <vector>

#include "common.cuh"

#ifndef PACO_TC_EARLY_ABLATE
#define PACO_TC_EARLY_ABLATE 0
#endif
#ifndef PACO_EXIT_WAIT_READ
#define PACO_EXIT_WAIT_READ 1
#endif
namespace paco {

#ifndef PACO_RES_AST
#define PACO_RES_AST 5
#define PACO_RES_EB 1
#define PACO_RES_EC 16
#endif
#ifndef PACO_EPI_RING
#define PACO_EPI_RING 1
#endif

namespace tc {

#define PACO_TC_ARGS(...) __VA_ARGS__
constexpr int BM = 128;
// warp 0: TMA producer, warp 1: MMA issuer, warps 2..: epilogue (Kind::EPI_WARPS)

// bf16 inputs, one MMA pass; N=256 tiles, 64-deep k blocks (128 B rows);
// ST stages of 48 KB, EW epilogue warps (EW = 8: 2 per TMEM lane quadrant,
// half the columns each) with EB staging buffers each.
template <int ST, int EB, int EW, int EC = 32>
struct KindBF16T {
  static constexpr int BN = 256, BK = 64, UMMA_K = 16, STAGES = ST, ELEM = 2, NOPS = 1, PASSES = 1;
  static constexpr int RING_BYTES = ST * 48 * 1024, EPI_WARPS = EW, EPI_BUFS = EB, KB_MAX = 0, EPI_COLS = EC;
  static constexpr int SWZ = 128;  // operand swizzle (bytes per K-major row)
  static constexpr bool B_KMAJOR = false, B_RES = false, FUSED = false;
  static constexpr int CONV_WARPS = 0, RAW_STAGES = 0, NT = 0, RAW_BYTES = 0;
  // F32 accumulate, BF16 A/B (format 1), A K-major, B MN-major (bit 16)
  static constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                                    (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
  static constexpr CUtensorMapDataType DT = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
};
// streaming default: 4 stages of 48 KB + 8 warps x 2 x 2 KB staging (16-column
// boxes) -- 8192^3 bf16 1000 -> 936 us vs 3 stages / 32-column boxes
#ifndef PACO_BF16_ST
#define PACO_BF16_ST 4
#define PACO_BF16_EB 2
#define PACO_BF16_EC 16
#endif
using KindBF16 = KindBF16T<PACO_BF16_ST, PACO_BF16_EB, 8, PACO_BF16_EC>;
// fp32 inputs as 3xTF32 (hi/lo operand tiles), N=128 tiles, 32-deep k blocks.
// BK_ = 32: 128-byte K-major rows (SWIZZLE_128B); BK_ = 16: 64-byte rows
// (SWIZZLE_64B) -- half the bytes per stage, so twice the stages in the ring.
template <int BN_, int ST, int BK_ = 32>
struct KindTF32x3T {
  static constexpr int BN = BN_, BK = BK_, UMMA_K = 8, STAGES = ST, ELEM = 4, NOPS = 2, PASSES = 3;
  static constexpr int RING_BYTES = ST * 2 * (128 + BN_) * BK * 4, EPI_WARPS = 4, EPI_BUFS = 2, KB_MAX = 0,
                       EPI_COLS = 32, SWZ = BK_ * 4;
  static constexpr bool B_KMAJOR = true, B_RES = false, FUSED = false;  // B^T tiles (the split writes B transposed)
  static constexpr int CONV_WARPS = 0, RAW_STAGES = 0, NT = 0, RAW_BYTES = 0;
  // F32 accumulate, TF32 A/B (format 2), both K-major
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                                    (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
  static constexpr CUtensorMapDataType DT = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
};
using KindTF32x3 = KindTF32x3T<128, 3>;
// Wide: N = 256 tiles, 16-deep k blocks (64-byte rows, SWIZZLE_64B) so four
// 48 KB stages fit beside the epilogue buffers -- measured best of
// {<256,2,32>, <256,4,16>, <128,6,16>} on cfg5 (36.9 / 34.6 / 48.1 ms).
using KindTF32x3W = KindTF32x3T<256, 4, 16>;
// (MN-major B -- bit 16 of the descriptor -- is what the bf16 kind uses; with
// kind::tf32 it returned all-zero products here, hence the transposed split.)

// 3xTF32 with the operand formation fused into the kernel (Strassen leaves):
// each operand is a signed sum of NT_ <= 2 raw fp32 K-major views (S_r of A,
// T_r^T of B^T).  The producer TMA-loads the raw term
// tiles straight into the hi / lo slots of an operand stage; CW converter
// warps then form x = (+/-)t0 (+/-) t1 and split it IN PLACE into
// hi = tf32_rn(x), lo = tf32_rn(x - hi) -- raw and operand tiles share one
// 64B-swizzled box layout, so every 16-byte chunk is read and rewritten by one
// thread at one position.  So the ring keeps the split path's bytes in flight
// (ST stages of 48 KB) while the separate split launches and their HBM round
// trip of hi/lo pairs disappear.
template <int ST, int NT_, int CW = 4>
struct KindTF32x3FT {
  static constexpr int BN = 256, BK = 16, UMMA_K = 8, STAGES = ST, ELEM = 4, NOPS = 2, PASSES = 3;
  static constexpr int EPI_WARPS = 4, EPI_BUFS = 2, KB_MAX = 0, EPI_COLS = 16, SWZ = 64;
  static constexpr bool B_KMAJOR = true, B_RES = false, FUSED = true;
  static constexpr int CONV_WARPS = CW, RAW_STAGES = 0, NT = NT_, RAW_BYTES = 0;
  static_assert(NT_ >= 1 && NT_ <= NOPS, "raw terms live in the hi / lo slots");
  static constexpr int RING_BYTES = ST * 2 * (128 + BN) * BK * 4;
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                                    (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
  static constexpr CUtensorMapDataType DT = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
};
#ifndef PACO_TF32F_ST
#define PACO_TF32F_ST 4
#define PACO_TF32F_CW 8
#endif
using KindTF32x3F = KindTF32x3FT<PACO_TF32F_ST, 2, PACO_TF32F_CW>;

// bf16 with K <= KB_MAX * BK: the CTA's whole B column block (K x 256, 128 KB)
// stays resident in shared memory across its consecutive tiles of that block,
// so per tile only A (64 KB) is loaded -- the streaming kind re-reads B's
// 128 KB from L2 for every 128 KB of C it writes, which puts cfg3 on the L2
// throughput cap instead of HBM.  A ring of AST stages, EB staging buffers
// per epilogue warp.
template <int AST, int EB, int EW = 8, int EC = 32, int BN_ = 256>
struct KindBF16Res {
  static constexpr int BN = BN_, BK = 64, UMMA_K = 16, STAGES = AST, ELEM = 2, NOPS = 1, PASSES = 1;
  static constexpr int KB_MAX = 4, EPI_WARPS = EW, EPI_BUFS = EB, EPI_COLS = EC, SWZ = 128;
  static constexpr int RING_BYTES = KB_MAX * BN * BK * 2 + AST * 128 * BK * 2;
  static constexpr bool B_KMAJOR = false, B_RES = true, FUSED = false;
  static constexpr int CONV_WARPS = 0, RAW_STAGES = 0, NT = 0, RAW_BYTES = 0;
  // F32 accumulate, BF16 A/B, A K-major, B MN-major, N = BN
  static constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                                    (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
  static constexpr CUtensorMapDataType DT = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
};

template <class K>
struct Layout {
  static constexpr int BOX_N = 128 / K::ELEM;                 // elements per 128 B row
  static constexpr int A_BYTES = BM * K::BK * K::ELEM;        // one operand tile
  static constexpr int B_BYTES = K::BN * K::BK * K::ELEM;
  static constexpr int B_REGION = K::KB_MAX * B_BYTES;         // resident B (B_RES kinds)
  static constexpr int STAGE_BYTES = K::B_RES ? A_BYTES : K::NOPS * (A_BYTES + B_BYTES);
  static constexpr int SMEM_EPI = K::RING_BYTES;
  static constexpr int EPI_BUF = 32 * K::EPI_COLS * 4;        // one C store box: 32 rows x EPI_COLS fp32
  static constexpr int SMEM_BAR = SMEM_EPI + K::EPI_WARPS * K::EPI_BUFS * EPI_BUF;
  static constexpr int THREADS = 64 + 32 * (K::EPI_WARPS + K::CONV_WARPS);
  static_assert(B_REGION + K::STAGES * STAGE_BYTES + K::RAW_BYTES <= K::RING_BYTES, "stage ring");
  static constexpr int SMEM_ALLOC = SMEM_BAR + 512 + 1024;    // + runtime 1024-B alignment slack
  static constexpr uint32_t TMEM_COLS = 2 * K::BN;            // double-buffered accumulator
  static_assert(SMEM_ALLOC <= 232448, "shared memory budget");
  __device__ static int a_off(int stage, int op) { return B_REGION + stage * STAGE_BYTES + op * A_BYTES; }
  __device__ static int b_off(int stage, int op) { return stage * STAGE_BYTES + K::NOPS * A_BYTES + op * B_BYTES; }
  __device__ static int b_res_off(int kb) { return kb * B_BYTES; }
};

// K-major, 64B swizzle: 64-byte rows, 8-row groups 512 B apart, layout type 4.
__device__ __forceinline__ uint64_t smem_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(512 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(4) << 61;
  return d;
}

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
// in 16 B units: 128 B of N per row, rows = k; 8-row (1024 B) atoms step along
// k by SBO; 128-byte-wide N chunks (one TMA box of BK rows each) step by LBO.
__device__ __forceinline__ uint64_t smem_desc_mn_sw128(uint32_t saddr, int bk) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((bk * 128) >> 4) << 16;  // LBO: next 128-byte-wide N chunk (one TMA box)
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
// Relaxed: no release fence, so an in-flight global atomic (the producer's
// tile claim) does not stall it; the TMA's complete_tx orders the data.
__device__ __forceinline__ void mbar_expect_tx_relaxed(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
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

// Round to the nearest tf32 (10 mantissa bits; the result's low 13 bits are 0).
__device__ __forceinline__ float round_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);  // .x = a (low half)
  return *reinterpret_cast<const uint32_t*>(&v);
}

// The same rounding on the integer ALU (cvt.rna.tf32 issues on the narrow XU
// pipe): add half an ulp of tf32 to the magnitude bits and clear the 13 low
// bits -- round half away from zero, as .rna; carries roll into the exponent
// exactly like a rounding up (finite inputs).
__device__ __forceinline__ uint32_t round_tf32_bits(uint32_t b) { return (b + 0x1000u) & 0xFFFFE000u; }

// 16-byte shared-memory accesses by 32-bit shared address (the generic
// LD.E / ST.E the compiler emits for computed smem pointers cost a translation)
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

template <class K>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  if constexpr (K::ELEM == 2)
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(K::IDESC), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(K::IDESC), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

struct TcArgs {
  int64_t n, m, k;   // every problem's C is n x m
  int32_t count;     // problems in the batch (same shape; tiles of all share one queue)
  int32_t overwrite;
  int32_t tiles_rb;  // row blocks
  int32_t tiles_nb;  // column blocks
  int32_t kblocks;
  int32_t ablate;    // diagnostics: 1 = no C stores, 2 = no MMAs, 4 = no smem staging, 8 = no A loads,
                     // 16 = no resident-B loads
  long long* trace;  // diagnostics (paco_debug_trace): per CTA x 16 tiles x 6 globaltimer stamps
  int32_t* sched;    // per-group tile counters + a CTA-done counter at [groups]
                     // (zero at launch; the last CTA to finish zeroes them again)
  int32_t groups;    // CTA c serves group c % groups: column blocks g, g + groups, ...
  int32_t early;     // operands are not written by the previous launch on the stream (run_tc): the
                     // producer loads its first tile and the MMAs run before griddepcontrol.wait
};

// slot 15 of each CTA: (entry, after setup, exit)
__device__ __forceinline__ void tc_stamp(const TcArgs& a, int64_t tile, int field) {
  if (a.trace && tile < 16) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[(int64_t(blockIdx.x) * 16 + tile) * 6 + field] = t;
  }
}

// CTA-level schedule: dynamic.  The producer of each CTA claims the next tile
// of its group with an atomic counter and hands it to the MMA and epilogue
// warps through a small smem queue, so CTAs that get less HBM/L2 bandwidth
// simply take fewer tiles (a static split left the slowest CTA ~10 % behind
// the median).  groups = 1 (streaming B): tiles in row-block-major order, so
// the CTAs running at any moment write whole rows of C (HBM page locality)
// and share A row blocks in L2.  groups > 1 (resident B): group g walks column
// blocks g, g + groups, ... and inside one all row blocks, so a CTA never
// reloads its B, and the groups advance through the row blocks in step.
// A batch (count > 1, groups = 1) puts every problem's tiles in one queue:
// id = problem * tiles_rb * tiles_nb + nb * tiles_rb + rb.
// The first tile of every CTA is static (its rank in its group) so 148
// simultaneous atomics on one counter do not delay the start (~2 us measured);
// later claims are atomics, issued one tile ahead by the producer.
// Streaming kinds walk row-block bands of kRowBand: inside a band, column by
// column, the band's row blocks in turn -- the ~148 tiles in flight then touch
// kRowBand A row blocks and ~148/kRowBand B column blocks, an L2-sized working
// set; a plain row-major walk re-streamed the whole of B from HBM every ~2-5
// row blocks once A and B outgrow the 126 MB L2 (8192^3: +7 %).
constexpr int32_t kRowBand = 8;

__device__ __forceinline__ int32_t tile_of(const TcArgs& a, int g, int32_t t) {
  if (a.groups == 1) {
    const int32_t tpp = a.tiles_rb * a.tiles_nb;
    if (t >= tpp * a.count) return -1;
    const int32_t u = t % tpp;
    const int32_t band = u / (kRowBand * a.tiles_nb), r0 = band * kRowBand;
    const int32_t rows = a.tiles_rb - r0 < kRowBand ? a.tiles_rb - r0 : kRowBand;
    const int32_t v = u - r0 * a.tiles_nb;  // position inside the band
    const int32_t nb = v / rows, rb = r0 + v % rows;
    return (t / tpp) * tpp + nb * a.tiles_rb + rb;
  }
  const int32_t nb = g + (t / a.tiles_rb) * a.groups;
  if (nb >= a.tiles_nb) return -1;
  return nb * a.tiles_rb + t % a.tiles_rb;
}

__device__ __forceinline__ int32_t claim_tile(const TcArgs& a, bool first) {
  const int g = int(blockIdx.x % uint32_t(a.groups));
  const int32_t in_group = int32_t((gridDim.x - g + a.groups - 1) / a.groups);
  const int32_t t = first ? int32_t(blockIdx.x / a.groups) : in_group + atomicAdd(&a.sched[g], 1);
  return tile_of(a, g, t);
}
// Split form for the producer: issue the claim now (atomic result in flight),
// turn it into a tile id only when it is needed (the next publish), so the
// ~1 us round trip of 148 contending atomics never delays the current tile's
// TMA loads.
__device__ __forceinline__ int32_t claim_issue(const TcArgs& a) {
  return atomicAdd(&a.sched[blockIdx.x % uint32_t(a.groups)], 1);
}
__device__ __forceinline__ int32_t claim_resolve(const TcArgs& a, int32_t raw) {
  const int g = int(blockIdx.x % uint32_t(a.groups));
  const int32_t in_group = int32_t((gridDim.x - g + a.groups - 1) / a.groups);
  return tile_of(a, g, in_group + raw);
}

// One problem: operand maps (hi/lo for 3xTF32), the output map, and the column
// offset of each view inside its 16-byte aligned map base.
struct TcProb {
  CUtensorMap a[2], b[2], c;
  CUtensorMap cx[3];  // further destinations of the same product (reduce-add only)
  int32_t a_col0[2], b_col0[2], c_col0, cx_col0[3];
  int32_t ndst;  // 1 + number of cx maps in use
  uint32_t neg;  // bit d: destination d receives -AB
  int32_t nta, ntb;      // fused kinds: raw terms of A (maps a[0..nta)) and of B^T (b[0..ntb))
  uint32_t sga, sgb;     // bit t: term t enters with coefficient -1
  CUtensorMap a2, b2;    // tf32 + 2 x bf16 format: a[0] = hi (fp32), a[1] = bf16(hi), a2 = bf16(x - hi)
  int32_t a2_col0, b2_col0;
};
#ifndef PACO_TC_MAXBATCH
#define PACO_TC_MAXBATCH 8
#endif
constexpr int kMaxBatch = PACO_TC_MAXBATCH;
struct TcMaps {
  TcProb p[kMaxBatch];
};

template <class K>
__global__ void __launch_bounds__(Layout<K>::THREADS, 1) tc_gemm_kernel(const __grid_constant__ TcMaps maps, const TcArgs args) {
  using L = Layout<K>;
  constexpr int STAGES = K::STAGES, BN = K::BN, BK = K::BK;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int MAXR = 16;  // barrier slots for the stage / A ring
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::SMEM_BAR);
  uint64_t* empty = full + MAXR;
  uint64_t* tfull = empty + MAXR;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;   // resident B k block landed (B_RES; one per k block)
  uint64_t* bempty = bfull + 4;   // MMAs reading the resident B completed (B_RES)
  constexpr int QD = 4;           // tile queue depth
  uint64_t* qfull = bempty + 1;   // tile id published by the producer
  uint64_t* qempty = qfull + QD;  // ... and read by the MMA warp + every epilogue (+ converter) warp
  uint64_t* rfull = qempty + QD;  // fused kinds: raw term tiles landed in a stage (TMA)
  int32_t* qid = reinterpret_cast<int32_t*>(rfull + 4);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qid + QD);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) tc_stamp(args, 15, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], K::FUSED ? K::CONV_WARPS : 1);  // fused: one arrival per converter warp
      mbar_init(&empty[s], 1);
    }
    if (K::FUSED)
      for (int s = 0; s < STAGES; ++s) mbar_init(&rfull[s], 1);  // raw terms landed in stage s
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], K::EPI_WARPS);
    }
    for (int kb = 0; kb < 4; ++kb) mbar_init(&bfull[kb], 1);
    mbar_init(bempty, 1);
    for (int j = 0; j < QD; ++j) {
      mbar_init(&qfull[j], 1);
      mbar_init(&qempty[j], 1 + K::EPI_WARPS + K::CONV_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int q = 0; q < args.count; ++q) {
      for (int o = 0; o < K::NOPS; ++o) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&maps.p[q].a[o])) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&maps.p[q].b[o])) : "memory");
      }
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&maps.p[q].c)) : "memory");
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: the set-up above (barriers, TMEM, tensor-map
  // prefetch) overlaps the previous kernel on the stream; every global access
  // (operand loads, tile claims, C stores) comes after its grid has completed.
  // The next launch may start as soon as SMs free up (one CTA per SM: only
  // SMs whose CTA has exited take one of its CTAs).
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  // early (resident-B kinds): the producer's first-tile loads and the MMA warp
  // (TMEM and shared memory only) run ahead of the wait; tile claims and every
  // C store still come after the previous grid has completed
  const bool early = K::B_RES && args.early;
  if (!(early && warp <= 1)) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (threadIdx.x == 0) tc_stamp(args, 15, 1);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      {
        uint32_t it = 0, bloads = 0;
        int loaded_nb = -1;
        const int32_t first_id = claim_tile(args, true);
        int32_t raw = 0;
        for (int64_t i = 0;; ++i) {
          const int32_t id = i == 0 ? first_id : claim_resolve(args, raw);
          if (i == 0) tc_stamp(args, 15, 3);
          const int qs = int(i % QD);
          mbar_wait(&qempty[qs], (uint32_t(i / QD) & 1) ^ 1);
          qid[qs] = id;
          mbar_arrive(&qfull[qs]);
          if (id < 0) {
            if (early && i == 0) asm volatile("griddepcontrol.wait;\n" ::: "memory");
            break;
          }
          const bool late_claim = early && i == 0;  // the first claim waits for the previous grid
          if (!late_claim) raw = claim_issue(args);  // one tile ahead; resolved (waited for) at the next publish
          const int tpp = args.tiles_rb * args.tiles_nb, lid = id % tpp;
          const int nb = lid / args.tiles_rb, rb = lid % args.tiles_rb;
          const TcProb& P = maps.p[id / tpp];
          if constexpr (K::B_RES) {
            if (nb != loaded_nb) {  // (re)load the resident B column block
              if (bloads > 0) mbar_wait(bempty, (bloads - 1) & 1);
              for (int kb = 0; kb < args.kblocks; ++kb) {  // per k block: the first MMA starts early
                if (args.ablate & 16) {  // diagnostics: the resident B "lands" with no bytes
                  mbar_arrive(&bfull[kb]);
                  continue;
                }
                mbar_expect_tx_relaxed(&bfull[kb], L::B_BYTES);
#pragma unroll
                for (int j = 0; j < BN / L::BOX_N; ++j)
                  tma_load_2d(smem + L::b_res_off(kb) + j * (BK * 128), &P.b[0], &bfull[kb],
                              P.b_col0[0] + nb * BN + L::BOX_N * j, kb * BK);
              }
              loaded_nb = nb;
              ++bloads;
              if (i == 0) tc_stamp(args, 15, 4);
            }
          }
          if constexpr (K::FUSED) {
            // raw fp32 term tiles into the stage's hi / lo slots; the converter
            // warps form and split them in place (rfull -> full)
            const uint32_t bytes = uint32_t(P.nta * L::A_BYTES + P.ntb * L::B_BYTES);
            for (int kb = 0; kb < args.kblocks; ++kb, ++it) {
              const int s = it % STAGES;
              mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
              if (kb == 0 && i < 15) tc_stamp(args, i, 0);
              mbar_expect_tx_relaxed(&rfull[s], bytes);
#pragma unroll
              for (int t = 0; t < K::NT; ++t) {
                if (t < P.nta) tma_load_2d(smem + L::a_off(s, t), &P.a[t], &rfull[s], P.a_col0[t] + kb * BK, rb * BM);
                if (t < P.ntb) tma_load_2d(smem + L::b_off(s, t), &P.b[t], &rfull[s], P.b_col0[t] + kb * BK, nb * BN);
              }
            }
            continue;
          }
          for (int kb = 0; kb < args.kblocks; ++kb, ++it) {
            const int s = it % STAGES;
            mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
            if (kb == 0 && i < 15) tc_stamp(args, i, 0);
            if (kb == args.kblocks - 1 && i < 15) tc_stamp(args, i, 1);
            if constexpr (K::B_RES) {
              if (args.ablate & 8) {  // diagnostics: the stage "lands" with no bytes
                mbar_arrive(&full[s]);
                continue;
              }
              mbar_expect_tx_relaxed(&full[s], L::A_BYTES);
              tma_load_2d(smem + L::a_off(s, 0), &P.a[0], &full[s], P.a_col0[0] + kb * BK, rb * BM);
              continue;
            }
            mbar_expect_tx_relaxed(&full[s], K::NOPS * (L::A_BYTES + L::B_BYTES));
#pragma unroll
            for (int o = 0; o < K::NOPS; ++o) {
              tma_load_2d(smem + L::a_off(s, o), &P.a[o], &full[s], P.a_col0[o] + kb * BK, rb * BM);
              if constexpr (K::B_KMAJOR) {
                // B^T (m x k, K contiguous): one box of [BN rows][BK k]
                tma_load_2d(smem + L::b_off(s, o), &P.b[o], &full[s], P.b_col0[o] + kb * BK, nb * BN);
              } else {
                // B is k x m row-major (N contiguous): boxes of [BK k rows][128 B of n]
#pragma unroll
                for (int j = 0; j < BN / L::BOX_N; ++j)
                  tma_load_2d(smem + L::b_off(s, o) + j * (BK * 128), &P.b[o], &full[s],
                              P.b_col0[o] + nb * BN + L::BOX_N * j, kb * BK);
              }
            }
          }
          if (late_claim) {
            asm volatile("griddepcontrol.wait;\n" ::: "memory");
            raw = claim_issue(args);
          }
        }
        // every claim of this CTA has returned (the last one said "no tile"): the
        // last CTA to get here re-zeroes the counters for the next launch on this
        // stream (no memset per launch; that launch claims only after
        // griddepcontrol.wait, i.e. after this grid completed).  Done here, not at
        // exit, so the atomic's round trip is off the CTA's exit path.
        if (atomicAdd(&args.sched[args.groups], 1) == int32_t(gridDim.x) - 1) {
          for (int g = 0; g < args.groups; ++g) args.sched[g] = 0;
          args.sched[args.groups] = 0;
          __threadfence();
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      uint32_t it = 0, buses = 0;
      int tile = 0, cur_nb = -1;
      bool new_b = false;  // first tile on a freshly loaded B: wait per k block
      for (int64_t i = 0;; ++i, ++tile) {
        const int qs = int(i % QD);
        mbar_wait(&qfull[qs], uint32_t(i / QD) & 1);
        const int32_t id = qid[qs];
        mbar_arrive(&qempty[qs]);
        if (id < 0) break;
        const int a = tile & 1;
        const uint32_t use = uint32_t(tile >> 1);
        if constexpr (K::B_RES) {  // count == 1
          const int nb = id / args.tiles_rb;
          if (nb != cur_nb) {
            if (cur_nb >= 0) umma_commit(bempty);  // the old B is free once its MMAs complete
            new_b = true;
            ++buses;
            cur_nb = nb;
          }
        }
        mbar_wait(&tempty[a], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + uint32_t(a * BN);
        for (int kb = 0; kb < args.kblocks; ++kb, ++it) {
          const int s = it % STAGES;
          if (K::B_RES && new_b) mbar_wait(&bfull[kb], (buses - 1) & 1);
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          if (kb == 0 && i < 15) tc_stamp(args, i, 2);
          uint64_t ad[K::NOPS], bd[K::NOPS];
#pragma unroll
          for (int o = 0; o < K::NOPS; ++o) {
            const int aoff = L::a_off(s, o), boff = K::B_RES ? L::b_res_off(kb) : L::b_off(s, o);
            if constexpr (K::SWZ == 64) {
              ad[o] = smem_desc_sw64(smem_u32(smem + aoff));
              bd[o] = smem_desc_sw64(smem_u32(smem + boff));  // B^T, K-major
            } else {
              ad[o] = smem_desc_sw128(smem_u32(smem + aoff));
              bd[o] = K::B_KMAJOR ? smem_desc_sw128(smem_u32(smem + boff)) : smem_desc_mn_sw128(smem_u32(smem + boff), BK);
            }
          }
#pragma unroll
          for (int kk = 0; kk < BK / K::UMMA_K; ++kk) {
            // A (K-major): +UMMA_K*ELEM = 32 B inside the 128 B swizzle row = +2 units;
            // B (MN-major): +UMMA_K k rows of 128 B = +8*UMMA_K units
            const uint64_t a_adv = uint64_t(2 * kk);
            const uint64_t b_adv = K::B_KMAJOR ? uint64_t(2 * kk) : uint64_t(8 * K::UMMA_K * kk);
#pragma unroll
            for (int ps = 0; ps < K::PASSES; ++ps) {
              // passes: hi*hi, hi*lo, lo*hi (3xTF32); a single pass for bf16
              const int ao = ps == 2 ? 1 : 0, bo = ps == 1 ? 1 : 0;
              if (!(args.ablate & 2)) umma<K>(d_tmem, ad[ao] + a_adv, bd[bo] + b_adv, (kb | kk | ps) != 0);
            }
          }
          umma_commit(&empty[s]);  // stage is free once these MMAs complete
        }
        if (i < 15) tc_stamp(args, i, 3);
        umma_commit(&tfull[a]);    // accumulator ready for the epilogue
        new_b = false;
      }
    }
  } else if (warp >= 2 + K::EPI_WARPS) {
   if constexpr (K::FUSED) {
    // ---------------- converter warps (fused kinds) ----------------
    // x = (+/-)t0 (+/-)t1, hi = tf32_rn(x), lo = tf32_rn(x - hi), in place over
    // the stage's hi (t0) / lo (t1) slots, 16-byte chunk by chunk.
    const int ct = (warp - 2 - K::EPI_WARPS) * 32 + lane;  // 0 .. 32 * CONV_WARPS - 1
    constexpr int NTH = 32 * K::CONV_WARPS;
    constexpr int A_CH = L::A_BYTES / 16, B_CH = L::B_BYTES / 16;
    constexpr int PER = (A_CH + B_CH) / NTH;  // chunks per thread per stage
    static_assert((A_CH + B_CH) % NTH == 0 && A_CH % NTH == 0, "whole chunks per converter thread");
    uint32_t it = 0;
    for (int64_t i = 0;; ++i) {
      const int qs = int(i % QD);
      mbar_wait(&qfull[qs], uint32_t(i / QD) & 1);
      const int32_t id = qid[qs];
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[qs]);
      if (id < 0) break;
      const int tpp = args.tiles_rb * args.tiles_nb;
      const TcProb& P = maps.p[id / tpp];
      const int nta = P.nta, ntb = P.ntb;
      const uint32_t sga = P.sga, sgb = P.sgb;
      for (int kb = 0; kb < args.kblocks; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(&rfull[s], (it / STAGES) & 1);
        const uint32_t sbase = smem_u32(smem);
        uint4 x0[PER], x1[PER];
        // every load of the stage first (PER x 2 LDS.128 in flight), then the math and stores
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int c = ct + u * NTH;
          constexpr int UA = A_CH / NTH;  // the first UA chunk rounds cover A (A_CH % NTH == 0)
          const bool isa = u < UA;
          const uint32_t off = sbase + (isa ? L::a_off(s, 0) + c * 16 : L::b_off(s, 0) + (c - A_CH) * 16);
          const uint32_t off1 = sbase + (isa ? L::a_off(s, 1) + c * 16 : L::b_off(s, 1) + (c - A_CH) * 16);
          x0[u] = lds128(off);
          if ((isa ? nta : ntb) > 1) x1[u] = lds128(off1);
        }
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int c = ct + u * NTH;
          const bool isa = u < A_CH / NTH;
          const int nt = isa ? nta : ntb;
          const uint32_t sg = isa ? sga : sgb;
          float x[4] = {__uint_as_float(x0[u].x), __uint_as_float(x0[u].y), __uint_as_float(x0[u].z),
                        __uint_as_float(x0[u].w)};
          if (sg & 1u)
#pragma unroll
            for (int e = 0; e < 4; ++e) x[e] = -x[e];
          if (nt > 1) {
            const float y[4] = {__uint_as_float(x1[u].x), __uint_as_float(x1[u].y), __uint_as_float(x1[u].z),
                                __uint_as_float(x1[u].w)};
#pragma unroll
            for (int e = 0; e < 4; ++e) x[e] = (sg & 2u) ? x[e] - y[e] : x[e] + y[e];
          }
          uint32_t h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            h[e] = round_tf32_bits(__float_as_uint(x[e]));
            l[e] = round_tf32_bits(__float_as_uint(x[e] - __uint_as_float(h[e])));
          }
          const uint32_t off = sbase + (isa ? L::a_off(s, 0) + c * 16 : L::b_off(s, 0) + (c - A_CH) * 16);
          const uint32_t off1 = sbase + (isa ? L::a_off(s, 1) + c * 16 : L::b_off(s, 1) + (c - A_CH) * 16);
          sts128(off, make_uint4(h[0], h[1], h[2], h[3]));
          sts128(off1, make_uint4(l[0], l[1], l[2], l[3]));
        }
        // generic-proxy smem writes -> visible to the tensor core's async-proxy reads
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
      }
    }
   }
  } else {
    // ---------------- epilogue warps ----------------
    // Each warp drains its TMEM lane quadrant for PER 32-column chunks of the
    // tile, two chunks per tcgen05.ld (32x32b.x64): stage both into
    // 128B-swizzled [32 rows][32 fp32] buffers, one proxy fence, two TMA
    // stores (C = AB) or TMA reduce-adds (C += AB).
    const int q = warp % 4;  // TMEM lane quadrant this warp may access
    const int ew = warp - 2;  // epilogue warp index
    constexpr int CHUNKS = BN / 32, PER = CHUNKS * 4 / K::EPI_WARPS;  // chunks per warp
    static_assert(PER % 2 == 0, "chunk pairs");
    const int c_lo = (ew / 4) * PER;
    unsigned char* stage0 = smem + L::SMEM_EPI + ew * K::EPI_BUFS * L::EPI_BUF;
    int tile = 0;
    uint32_t box = 0;  // boxes staged by this warp (PACO_EPI_RING buffer index)
    (void)box;
    for (int64_t i = 0;; ++i, ++tile) {
      const int qs = int(i % QD);
      mbar_wait(&qfull[qs], uint32_t(i / QD) & 1);
      const int32_t id = qid[qs];
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[qs]);
      if (id < 0) break;
      const int tpp = args.tiles_rb * args.tiles_nb, lid = id % tpp;
      const int nb = lid / args.tiles_rb, rb = lid % args.tiles_rb;
      const TcProb& P = maps.p[id / tpp];
      const int a = tile & 1;
      const uint32_t use = uint32_t(tile >> 1);
      mbar_wait(&tfull[a], use & 1);
      tc_fence_after();
      if (ew == 0 && lane == 0 && i < 15) tc_stamp(args, i, 4);
      const int row0 = rb * BM + 32 * q;
#pragma unroll 1
      for (int c = c_lo; c < c_lo + PER; c += 2) {
        uint32_t v[64];
        const uint32_t taddr = tmem_base + (uint32_t(32 * q) << 16) + uint32_t(a * BN + 32 * c);
#define PACO_R8(i) "=r"(v[i]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), "=r"(v[i + 5]), \
                   "=r"(v[i + 6]), "=r"(v[i + 7])
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, "
            "%34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, "
            "%54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];\n"
            : PACO_R8(0), PACO_R8(8), PACO_R8(16), PACO_R8(24), PACO_R8(32), PACO_R8(40), PACO_R8(48), PACO_R8(56)
            : "r"(taddr));
#undef PACO_R8
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (c + 2 == c_lo + PER) {
          // all of this warp's TMEM reads for the tile are done: release the buffer
          tc_fence_before();
          if (lane == 0) mbar_arrive(&tempty[a]);
        }
        const int col0 = nb * BN + 32 * c;
        if (col0 >= args.m) continue;  // warp-uniform: nothing left to store
        // 64 columns in SUBS boxes of EPI_COLS
        constexpr int EC = K::EPI_COLS, SUBS = 64 / EC, EB = K::EPI_BUFS;
#if PACO_EPI_RING
        // ring of EB staging buffers per warp, one bulk group per box: before
        // box b reuses buffer b % EB, wait until at most EB-1 younger groups are
        // still reading shared memory (box b-EB has been read), so EB-1 stores
        // stay in flight while the next box is staged
#pragma unroll
        for (int h = 0; h < SUBS; ++h) {
          if (col0 + EC * h >= args.m) break;
#pragma unroll 1
          for (int d = 0; d < P.ndst; ++d) {  // every destination of the product (Strassen C terms)
            const uint32_t sgn = ((P.neg >> d) & 1u) << 31;  // -AB: flip the fp32 sign bits
            unsigned char* buf = stage0 + (box % EB) * L::EPI_BUF;
            ++box;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(EB - 1) : "memory");
            __syncwarp();
            if (!(args.ablate & 4)) {
#pragma unroll
              for (int j = 0; j < EC / 4; ++j) {
                const uint4 w = make_uint4(v[EC * h + 4 * j] ^ sgn, v[EC * h + 4 * j + 1] ^ sgn,
                                           v[EC * h + 4 * j + 2] ^ sgn, v[EC * h + 4 * j + 3] ^ sgn);
                const int sw = EC == 32 ? (j ^ (lane & 7)) : (j ^ ((lane >> 1) & 3));
                sts128(smem_u32(buf) + lane * (EC * 4) + sw * 16, w);
              }
              asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            }
            __syncwarp();
            if (lane == 0) {
              if (row0 < args.n && !(args.ablate & 1)) {
                const CUtensorMap* cm = d == 0 ? &P.c : &P.cx[d - 1];
                const int cc0 = d == 0 ? P.c_col0 : P.cx_col0[d - 1];
                if (args.overwrite)
                  tma_store_2d(cm, buf, cc0 + col0 + EC * h, row0);
                else
                  tma_reduce_add_2d(cm, buf, cc0 + col0 + EC * h, row0);
              }
              asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            }
          }
        }
#else
        // groups of EB boxes: wait for the buffers, stage EB boxes, ONE proxy
        // fence, EB TMA stores (or reduce-adds), one bulk group
#pragma unroll
        for (int h0 = 0; h0 < SUBS; h0 += EB) {
          if (col0 + EC * h0 >= args.m) break;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
          __syncwarp();
          if (!(args.ablate & 4)) {
#pragma unroll
            for (int hh = 0; hh < EB; ++hh) {
              const int h = h0 + hh;
              unsigned char* buf = stage0 + hh * L::EPI_BUF;
              // swizzled [32 rows][EC fp32]: 16 B chunk j of row r at j ^ (r-bits of the
              // 128B (EC = 32) / 64B (EC = 16) TMA swizzle pattern)
#pragma unroll
              for (int j = 0; j < EC / 4; ++j) {
                const uint4 w = make_uint4(v[EC * h + 4 * j], v[EC * h + 4 * j + 1], v[EC * h + 4 * j + 2],
                                           v[EC * h + 4 * j + 3]);
                const int sw = EC == 32 ? (j ^ (lane & 7)) : (j ^ ((lane >> 1) & 3));
                *reinterpret_cast<uint4*>(buf + lane * (EC * 4) + sw * 16) = w;
              }
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          }
          __syncwarp();
          if (lane == 0) {
#pragma unroll
            for (int hh = 0; hh < EB; ++hh) {
              const int h = h0 + hh;
              if (row0 < args.n && !(args.ablate & 1) && col0 + EC * h < args.m) {
                unsigned char* buf = stage0 + hh * L::EPI_BUF;
                if (args.overwrite)
                  tma_store_2d(&P.c, buf, P.c_col0 + col0 + EC * h, row0);
                else
                  tma_reduce_add_2d(&P.c, buf, P.c_col0 + col0 + EC * h, row0);
              }
            }
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
          }
        }
#endif
      }
      if (ew == 0 && lane == 0 && i < 15) tc_stamp(args, i, 5);
    }
#if PACO_EXIT_WAIT_READ
    // exit once the last boxes have been READ out of shared memory: the global
    // writes still complete before the grid does (a dependent launch's
    // griddepcontrol.wait sees them), and the next CTA can take this SM meanwhile
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
#else
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
#endif
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(L::TMEM_COLS));
  if (threadIdx.x == 0) tc_stamp(args, 15, 2);
}

// ---------------------------------------------------------------------------
// 3xTF32 on a CTA PAIR (tcgen05 cta_group::2) -- the Strassen leaf GEMM.
//
// The single-CTA kernel moves, per 16-deep k block of a 128 x 256 tile, 48 KB
// of TMA writes and 72 KB of MMA operand reads (three passes) through one
// SM's shared memory -- ~940 clocks at 128 B/clk against ~1000 clocks of
// tf32 MMA work, so the tensor pipe stalls on shared memory.  A CTA pair
// issues M = 256 x N = 256 MMAs: each CTA holds its 128 rows of A and HALF of
// B^T (128 rows), so per CTA the stage is 32 KB of TMA writes and 48 KB of
// operand reads for the same 128 x 256 of output.  The leader CTA (rank 0)
// issues every MMA; both CTAs' TMA loads complete on the leader's stage
// barrier; the leader's commits arrive on both CTAs' barriers (multicast);
// each CTA drains its own TMEM half (its 128 rows) and the peer's epilogue
// releases the accumulator with a remote arrive on the leader's barrier.
// Tiles (256 x 256 of C) are dealt to pairs statically in row-band order.
// ---------------------------------------------------------------------------
#ifndef PACO_PAIR_CG
#define PACO_PAIR_CG 2
#endif
template <int ST, bool FA = false, bool B2 = false, bool CV = false>
struct PairLayout {
  static constexpr int BK = 16, BN = 256, BNH = 128, EC = 16, EW = 4, EB = 2;
  // FA: A is formed in the kernel (Strassen's S_r from <= 2 signed raw views,
  // TMA'd into the stage's hi / lo slots and split there in place by CW
  // converter warps); B^T arrives pre-split.
  // CV (with B2): bf16(hi) of both operands is formed in the kernel from the
  // tf32 hi tiles (fp32 SW64 -> bf16 SW32) by CW converter warps, so each operand
  // element costs 6 bytes of L2 traffic instead of 8
  // CV: CG groups of 4 converter warps take alternate stages, so one group's
  // per-stage latency (loads, fence, named barrier, signal) overlaps the next's
  static constexpr int CG = CV ? PACO_PAIR_CG : 1;
  static constexpr int CW = FA ? 4 : CV ? 4 * CG : 0;
  static constexpr int A_BYTES = BM * BK * 4;          // 8 KB: 128 rows x 16 fp32
  static constexpr int B_BYTES = BNH * BK * 4;         // 8 KB: this CTA's half of B^T
  static constexpr int STAGE_BYTES = 2 * (A_BYTES + B_BYTES);
  static constexpr int SMEM_EPI = ST * STAGE_BYTES;
  static constexpr int EPI_BUF = 32 * EC * 4;
  static constexpr int SMEM_BAR = SMEM_EPI + EW * EB * EPI_BUF;
  static constexpr int THREADS = 64 + 32 * (EW + CW);
  static constexpr int SMEM_ALLOC = SMEM_BAR + 512 + 1024;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static_assert(SMEM_ALLOC <= 232448, "shared memory budget");
  // F32 accumulate, TF32 A/B (both K-major), N = 256, M = 256 (cta_group::2)
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(BN >> 3) << 17) |
                                    (uint32_t(256 >> 4) << 24);
  __device__ static int a_off(int s, int o) { return s * STAGE_BYTES + o * A_BYTES; }
  __device__ static int b_off(int s, int o) { return s * STAGE_BYTES + 2 * A_BYTES + o * B_BYTES; }
  // B2 (tf32 + 2 x bf16): per stage the tf32 hi tiles of A and B^T (8 KB each) and
  // four 4 KB bf16 tiles (32-byte K-major rows, SWIZZLE_32B): bf16(hi) and bf16(x - hi)
  // of each -- the same 32 KB as the 3xTF32 stage, but the two correction products
  // run as kind::f16 MMAs (K = 16 per instruction: half the tensor time of tf32)
  static constexpr int H16_BYTES = BM * BK * 2;
  __device__ static int hi_a(int s) { return s * STAGE_BYTES; }
  __device__ static int hi_b(int s) { return s * STAGE_BYTES + A_BYTES; }
  __device__ static int x16(int s, int which) { return s * STAGE_BYTES + 2 * A_BYTES + which * H16_BYTES; }
  // x16 slots: 0 = bf16(A hi), 1 = bf16(A lo), 2 = bf16(B^T hi), 3 = bf16(B^T lo)
  static constexpr uint32_t IDESC_BF16 = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) |
                                         (uint32_t(256 >> 4) << 24);
};

// K-major, 32B swizzle: 32-byte rows, 8-row groups 256 B apart, layout type 6.
__device__ __forceinline__ uint64_t smem_desc_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(256 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(6) << 61;
  return d;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// arrive on an mbarrier given by its shared::cluster address (own or the peer's)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
// TMA load into this CTA's smem completing on a barrier in either CTA of the pair
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void umma_pair_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit: arrive on the barrier at this offset in BOTH CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}

// tile t (of all problems) -> (problem, 256-row block, 256-column block), row-band walk
__device__ __forceinline__ void pair_tile(const TcArgs& a, int32_t t, int& q, int& rb, int& nb) {
  const int32_t tpp = a.tiles_rb * a.tiles_nb;
  q = t / tpp;
  const int32_t u = t % tpp;
  const int32_t band = u / (kRowBand * a.tiles_nb), r0 = band * kRowBand;
  const int32_t rows = a.tiles_rb - r0 < kRowBand ? a.tiles_rb - r0 : kRowBand;
  const int32_t v = u - r0 * a.tiles_nb;
  nb = v / rows;
  rb = r0 + v % rows;
}

// RAW (with CV): the operands arrive as plain fp32 x; the tf32 MMA reads x itself
// (the tensor core uses its top 19 bits: hi = trunc_tf32(x)) and the converters
// form bf16(hi) and bf16(x - hi) -- 4 bytes of L2 traffic per operand element.
//
// B3 (bf16x3): the operands arrive pre-split as bf16 planes hi = bf16(x), lo =
// bf16(x - hi) (paco_lincomb_split); a stage holds 32 k of A hi / lo and of this
// CTA's half of B^T hi / lo (four 8 KB SW64 tiles, the 3xTF32 stage geometry) and
// the leader issues hi*hi, hi*lo, lo*hi as kind::f16 MMAs: no converter warps, and
// per CTA a stage is 32 KB of TMA writes + 48 KB of operand reads against 768
// clocks of MMA -- the tensor pipe, not shared memory, bounds it.
//
// BMN (with B3): B arrives in its own k x m layout (MN-major) instead of as B^T: a
// stage's B tile per CTA is [32 k rows][128 n] as two SWIZZLE_128B boxes of 64
// columns (128 B), read by the MMA through MN-major descriptors -- Strassen's T_r
// planes are formed from B's quadrants directly, with no transpose pass.
template <int ST, bool FA, bool B2, bool CV = false, bool RAW = false, bool B3 = false, bool BMN = false>
__global__ void __launch_bounds__(PairLayout<ST, FA, B2, CV>::THREADS, 1)
    tc_pair_kernel(const __grid_constant__ TcMaps maps, const TcArgs args) {
  using L = PairLayout<ST, FA, B2, CV>;
  constexpr int BK = L::BK, BN = L::BN;
  constexpr int KSTEP = B3 ? 2 * BK : BK;  // k per stage
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::SMEM_BAR);
  uint64_t* empty = full + 16;
  uint64_t* tfull = empty + 16;
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;  // FA: this CTA's raw A terms landed in stage s
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rfull + 16);
  unsigned char* sig = reinterpret_cast<unsigned char*>(rfull + 18);  // converter signal landing slots: 16 B per (group, rank)

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  int32_t pair, npairs;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(pair));
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(npairs));
  const int32_t total = args.tiles_rb * args.tiles_nb * args.count;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);  // the leader's expect_tx; TMA and (FA) converter signals complete it
      mbar_init(&empty[s], 1);
      mbar_init(&rfull[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * L::EW);  // both CTAs' epilogue warps release the (pair) accumulator
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int q = 0; q < args.count; ++q) {
      for (int o = 0; o < 2; ++o) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&maps.p[q].a[o])) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&maps.p[q].b[o])) : "memory");
      }
    }
  }
  if (warp == 1) {
    // one warp in EACH CTA of the pair (tools/microbench/pair_probe.cu)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's barriers are initialised before any remote complete_tx / arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs: own A rows, own half of B^T) ----------------
      const uint32_t full_leader0 = mapa_rank(smem_u32(&full[0]), 0);
      uint32_t it = 0;
      for (int32_t t = pair; t < total; t += npairs) {
        int q, rb, nb;
        pair_tile(args, t, q, rb, nb);
        const TcProb& P = maps.p[q];
        const int arow = rb * 256 + int(rank) * BM, brow = nb * BN + int(rank) * L::BNH;
        for (int kb = 0; kb < args.kblocks; ++kb, ++it) {
          const int s = it % ST;
          mbar_wait(&empty[s], ((it / ST) & 1) ^ 1);
          const uint32_t fb = full_leader0 + uint32_t(s) * 8u;
          if constexpr (FA) {
            // raw A terms -> own stage (own barrier, the converters split them);
            // pre-split B^T halves -> the leader's stage barrier
            // B^T halves of both CTAs + both CTAs' 16-byte "A converted" signals
            if (leader) mbar_expect_tx_relaxed(&full[s], 2 * 2 * L::B_BYTES + 2 * 16);
            mbar_expect_tx_relaxed(&rfull[s], uint32_t(P.nta * L::A_BYTES));
#pragma unroll
            for (int o = 0; o < 2; ++o) {
              if (o < P.nta) tma_load_2d(smem + L::a_off(s, o), &P.a[o], &rfull[s], P.a_col0[o] + kb * BK, arow);
              tma_load_2d_pair(smem + L::b_off(s, o), &P.b[o], fb, P.b_col0[o] + kb * BK, brow);
            }
          } else if constexpr (CV) {
            // hi (fp32) and bf16(x - hi) tiles into this CTA's stage on its own barrier;
            // the converters add bf16(hi) and signal the leader (2 x 16 bytes)
            if (leader) mbar_expect_tx_relaxed(&full[s], 2 * 16);
            mbar_expect_tx_relaxed(&rfull[s], uint32_t(L::A_BYTES + L::B_BYTES + (RAW ? 0 : 2 * L::H16_BYTES)));
            const int kc = kb * BK;
            tma_load_2d(smem + L::hi_a(s), &P.a[0], &rfull[s], P.a_col0[0] + kc, arow);
            tma_load_2d(smem + L::hi_b(s), &P.b[0], &rfull[s], P.b_col0[0] + kc, brow);
            if constexpr (!RAW) {
              tma_load_2d(smem + L::x16(s, 1), &P.a2, &rfull[s], P.a2_col0 + kc, arow);
              tma_load_2d(smem + L::x16(s, 3), &P.b2, &rfull[s], P.b2_col0 + kc, brow);
            }
          } else if constexpr (B2) {
            if (leader) mbar_expect_tx_relaxed(&full[s], 2 * L::STAGE_BYTES);
            const int kc = kb * BK;
            tma_load_2d_pair(smem + L::hi_a(s), &P.a[0], fb, P.a_col0[0] + kc, arow);
            tma_load_2d_pair(smem + L::hi_b(s), &P.b[0], fb, P.b_col0[0] + kc, brow);
            tma_load_2d_pair(smem + L::x16(s, 0), &P.a[1], fb, P.a_col0[1] + kc, arow);
            tma_load_2d_pair(smem + L::x16(s, 1), &P.a2, fb, P.a2_col0 + kc, arow);
            tma_load_2d_pair(smem + L::x16(s, 2), &P.b[1], fb, P.b_col0[1] + kc, brow);
            tma_load_2d_pair(smem + L::x16(s, 3), &P.b2, fb, P.b2_col0 + kc, brow);
          } else {
            if (leader) mbar_expect_tx_relaxed(&full[s], 2 * L::STAGE_BYTES);
#pragma unroll
            for (int o = 0; o < 2; ++o) {
              tma_load_2d_pair(smem + L::a_off(s, o), &P.a[o], fb, P.a_col0[o] + kb * KSTEP, arow);
              if constexpr (BMN) {
#pragma unroll
                for (int j = 0; j < 2; ++j)  // [32 k][64 n] boxes: this CTA's 128 columns of B
                  tma_load_2d_pair(smem + L::b_off(s, o) + j * (KSTEP * 128), &P.b[o], fb,
                                   P.b_col0[o] + brow + 64 * j, kb * KSTEP);
              } else {
                tma_load_2d_pair(smem + L::b_off(s, o), &P.b[o], fb, P.b_col0[o] + kb * KSTEP, brow);
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ---------------- MMA issuer (leader CTA only) ----------------
      uint32_t it = 0;
      int tile = 0;
      for (int32_t t = pair; t < total; t += npairs, ++tile) {
        const int a = tile & 1;
        const uint32_t use = uint32_t(tile >> 1);
        mbar_wait(&tempty[a], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + uint32_t(a * BN);
        for (int kb = 0; kb < args.kblocks; ++kb, ++it) {
          const int s = it % ST;
          mbar_wait(&full[s], (it / ST) & 1);
          tc_fence_after();
          if constexpr (B2 || CV) {
            // hi*hi on the tf32 path (two K = 8 steps), hi*lo and lo*hi as bf16 (one K = 16 each)
            const uint64_t ah = smem_desc_sw64(smem_u32(smem + L::hi_a(s)));
            const uint64_t bh = smem_desc_sw64(smem_u32(smem + L::hi_b(s)));
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk)
              umma_pair(d_tmem, ah + uint64_t(2 * kk), bh + uint64_t(2 * kk), L::IDESC, (kb | kk) != 0);
            umma_pair_f16(d_tmem, smem_desc_sw32(smem_u32(smem + L::x16(s, 0))),
                          smem_desc_sw32(smem_u32(smem + L::x16(s, 3))), L::IDESC_BF16, 1);
            umma_pair_f16(d_tmem, smem_desc_sw32(smem_u32(smem + L::x16(s, 1))),
                          smem_desc_sw32(smem_u32(smem + L::x16(s, 2))), L::IDESC_BF16, 1);
          } else {
            const uint64_t ad[2] = {smem_desc_sw64(smem_u32(smem + L::a_off(s, 0))),
                                    smem_desc_sw64(smem_u32(smem + L::a_off(s, 1)))};
            const uint64_t bd[2] = {BMN ? smem_desc_mn_sw128(smem_u32(smem + L::b_off(s, 0)), KSTEP)
                                        : smem_desc_sw64(smem_u32(smem + L::b_off(s, 0))),
                                    BMN ? smem_desc_mn_sw128(smem_u32(smem + L::b_off(s, 1)), KSTEP)
                                        : smem_desc_sw64(smem_u32(smem + L::b_off(s, 1)))};
            // 32 bytes of a 64-byte K-major row per step: 8 fp32 (tf32 K = 8) or 16 bf16 (f16 K = 16);
            // MN-major B: 16 k rows of 128 B per step
            constexpr uint64_t BADV = BMN ? 8 * 16 : 2;
            constexpr uint32_t IDB3 = L::IDESC_BF16 | (BMN ? (1u << 16) : 0u);
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk)
#pragma unroll
              for (int ps = 0; ps < 3; ++ps) {  // hi*hi, hi*lo, lo*hi
                const int ao = ps == 2 ? 1 : 0, bo = ps == 1 ? 1 : 0;
                if constexpr (B3)
                  umma_pair_f16(d_tmem, ad[ao] + uint64_t(2 * kk), bd[bo] + BADV * kk, IDB3, (kb | kk | ps) != 0);
                else
                  umma_pair(d_tmem, ad[ao] + uint64_t(2 * kk), bd[bo] + uint64_t(2 * kk), L::IDESC,
                            (kb | kk | ps) != 0);
              }
          }
          umma_commit_pair(&empty[s]);  // both CTAs' stage s is free once these MMAs complete
        }
        umma_commit_pair(&tfull[a]);    // both CTAs' accumulator halves are ready
      }
    }
  } else if (warp >= 2 + L::EW) {
    if constexpr (CV) {
      // ---------------- converter warps (CV, both CTAs): bf16(hi) tiles from the tf32 hi tiles ----------------
      // fp32 tile: row r at r*64, 16-byte chunk c (4 elements) at (c ^ ((r >> 1) & 3)) * 16 (SWIZZLE_64B);
      // bf16 tile: row r at r*32, 16-byte chunk c8 (8 elements) at (c8 ^ ((r >> 2) & 1)) * 16 (SWIZZLE_32B)
      const int grp = (warp - 2 - L::EW) / 4;
      const int ct = ((warp - 2 - L::EW) & 3) * 32 + lane;
      constexpr int NTH = 128;
      constexpr int CH = (BM + L::BNH) * 4;  // fp32 16-byte chunks of the A and B^T hi tiles
      static_assert(CH % NTH == 0, "whole chunks per converter thread");
      const uint32_t full_leader0 = mapa_rank(smem_u32(&full[0]), 0);
      const uint32_t sig_leader = mapa_rank(smem_u32(sig), 0);
      const uint32_t sbase = smem_u32(smem);
      uint32_t it = 0;
      for (int32_t t = pair; t < total; t += npairs) {
        for (int kb = 0; kb < args.kblocks; ++kb, ++it) {
          if (int(it % L::CG) != grp) continue;
          const int s = it % ST;
          mbar_wait(&rfull[s], (it / ST) & 1);
          uint4 x[CH / NTH];
#pragma unroll
          for (int u = 0; u < CH / NTH; ++u) {
            const int c = ct + u * NTH, isb = c >= BM * 4, cc = isb ? c - BM * 4 : c;
            const int r = cc >> 2, c4 = cc & 3;
            x[u] = lds128(sbase + (isb ? L::hi_b(s) : L::hi_a(s)) + r * 64 + ((c4 ^ ((r >> 1) & 3)) << 4));
          }
#pragma unroll
          for (int u = 0; u < CH / NTH; ++u) {
            const int c = ct + u * NTH, isb = c >= BM * 4, cc = isb ? c - BM * 4 : c;
            const int r = cc >> 2, c4 = cc & 3, c8 = c4 >> 1;
            const uint32_t pos = r * 32 + ((c8 ^ ((r >> 2) & 1)) << 4) + (c4 & 1) * 8;
            if constexpr (RAW) {
              // hi = what the tf32 MMA reads of x (its top 19 bits), lo = x - hi exactly
              const uint32_t xb[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
              float h[4], l[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                h[e] = __uint_as_float(xb[e] & 0xFFFFE000u);
                l[e] = __uint_as_float(xb[e]) - h[e];
              }
              asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(sbase + L::x16(s, isb ? 2 : 0) + pos),
                           "r"(pack_bf16x2(h[0], h[1])), "r"(pack_bf16x2(h[2], h[3]))
                           : "memory");
              asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(sbase + L::x16(s, isb ? 3 : 1) + pos),
                           "r"(pack_bf16x2(l[0], l[1])), "r"(pack_bf16x2(l[2], l[3]))
                           : "memory");
            } else {
              const uint32_t dst = sbase + L::x16(s, isb ? 2 : 0) + pos;
              const uint32_t lo = pack_bf16x2(__uint_as_float(x[u].x), __uint_as_float(x[u].y));
              const uint32_t hi = pack_bf16x2(__uint_as_float(x[u].z), __uint_as_float(x[u].w));
              asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(dst), "r"(lo), "r"(hi) : "memory");
            }
          }
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "n"(NTH) : "memory");
          if (ct == 0)
            asm volatile(
                "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];\n" ::"r"(
                    sig_leader + uint32_t(grp * 2 + int(rank)) * 16u),
                "r"(smem_u32(sig)), "r"(full_leader0 + uint32_t(s) * 8u)
                : "memory");
        }
      }
    } else if constexpr (FA) {
      // ---------------- converter warps (FA, both CTAs): S_r tile formed and split in place ----------------
      const int ct = (warp - 2 - L::EW) * 32 + lane;
      constexpr int NTH = 32 * (L::CW > 0 ? L::CW : 1), A_CH = L::A_BYTES / 16, PER = A_CH / NTH;
      static_assert(A_CH % NTH == 0, "whole A chunks per converter thread");
      const uint32_t full_leader0 = mapa_rank(smem_u32(&full[0]), 0);
      const uint32_t sig_leader = mapa_rank(smem_u32(sig), 0);
      const uint32_t sbase = smem_u32(smem);
      uint32_t it = 0;
      for (int32_t t = pair; t < total; t += npairs) {
        int q, rb, nb;
        pair_tile(args, t, q, rb, nb);
        const int nta = maps.p[q].nta;
        const uint32_t sga = maps.p[q].sga;
        for (int kb = 0; kb < args.kblocks; ++kb, ++it) {
          const int s = it % ST;
          mbar_wait(&rfull[s], (it / ST) & 1);
          uint4 x0[PER], x1[PER];
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const uint32_t off = sbase + L::a_off(s, 0) + (ct + u * NTH) * 16;
            x0[u] = lds128(off);
            if (nta > 1) x1[u] = lds128(off + L::A_BYTES);
          }
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            float x[4] = {__uint_as_float(x0[u].x), __uint_as_float(x0[u].y), __uint_as_float(x0[u].z),
                          __uint_as_float(x0[u].w)};
            if (sga & 1u)
#pragma unroll
              for (int e = 0; e < 4; ++e) x[e] = -x[e];
            if (nta > 1) {
              const float y[4] = {__uint_as_float(x1[u].x), __uint_as_float(x1[u].y), __uint_as_float(x1[u].z),
                                  __uint_as_float(x1[u].w)};
#pragma unroll
              for (int e = 0; e < 4; ++e) x[e] = (sga & 2u) ? x[e] - y[e] : x[e] + y[e];
            }
            uint32_t h[4], l[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              h[e] = round_tf32_bits(__float_as_uint(x[e]));
              l[e] = round_tf32_bits(__float_as_uint(x[e] - __uint_as_float(h[e])));
            }
            const uint32_t off = sbase + L::a_off(s, 0) + (ct + u * NTH) * 16;
            sts128(off, make_uint4(h[0], h[1], h[2], h[3]));
            sts128(off + L::A_BYTES, make_uint4(l[0], l[1], l[2], l[3]));
          }
          // generic-proxy writes -> the tensor core's async-proxy reads (of both CTAs' A halves).
          // The handoff to the leader is itself an async-proxy op -- a 16-byte bulk copy into
          // the leader's signal slot completing on its stage barrier -- so it needs no
          // cluster-scope release fence (a release.cluster arrive per stage stalled the
          // converters on ERRBAR for ~1 us each)
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          asm volatile("bar.sync 1, %0;\n" ::"n"(32 * (L::CW > 0 ? L::CW : 1)) : "memory");
          if (ct == 0)
            asm volatile(
                "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];\n" ::"r"(
                    sig_leader + rank * 16u),
                "r"(smem_u32(sig)), "r"(full_leader0 + uint32_t(s) * 8u)
                : "memory");
        }
      }
    }
  } else {
    // ---------------- epilogue warps (both CTAs: own 128 rows of the pair tile) ----------------
    const int q4 = warp % 4;  // TMEM lane quadrant
    const int ew = warp - 2;
    unsigned char* stage0 = smem + L::SMEM_EPI + ew * L::EB * L::EPI_BUF;
    const uint32_t tempty_leader0 = mapa_rank(smem_u32(&tempty[0]), 0);
    int tile = 0;
    uint32_t box = 0;
    for (int32_t t = pair; t < total; t += npairs, ++tile) {
      int pq, rb, nb;
      pair_tile(args, t, pq, rb, nb);
      const TcProb& P = maps.p[pq];
      const int a = tile & 1;
      const uint32_t use = uint32_t(tile >> 1);
      mbar_wait(&tfull[a], use & 1);
      tc_fence_after();
      const int row0 = rb * 256 + int(rank) * BM + 32 * q4;
#pragma unroll 1
      for (int c = 0; c < BN / 32; c += 2) {
        uint32_t v[64];
        const uint32_t taddr = tmem_base + (uint32_t(32 * q4) << 16) + uint32_t(a * BN + 32 * c);
#define PACO_R8(i) "=r"(v[i]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), "=r"(v[i + 5]), \
                   "=r"(v[i + 6]), "=r"(v[i + 7])
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, "
            "%34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, "
            "%54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];\n"
            : PACO_R8(0), PACO_R8(8), PACO_R8(16), PACO_R8(24), PACO_R8(32), PACO_R8(40), PACO_R8(48), PACO_R8(56)
            : "r"(taddr));
#undef PACO_R8
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (c + 2 == BN / 32) {
          tc_fence_before();
          if (lane == 0) mbar_arrive_cluster(tempty_leader0 + uint32_t(a) * 8u);
        }
        const int col0 = nb * BN + 32 * c;
        if (col0 >= args.m) continue;
        constexpr int EC = L::EC, SUBS = 64 / EC, EB = L::EB;
#pragma unroll
        for (int h = 0; h < SUBS; ++h) {
          if (col0 + EC * h >= args.m) break;
#pragma unroll 1
          for (int d = 0; d < P.ndst; ++d) {
            const uint32_t sgn = ((P.neg >> d) & 1u) << 31;
            unsigned char* buf = stage0 + (box % EB) * L::EPI_BUF;
            ++box;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(EB - 1) : "memory");
            __syncwarp();
#pragma unroll
            for (int j = 0; j < EC / 4; ++j) {
              const uint4 w = make_uint4(v[EC * h + 4 * j] ^ sgn, v[EC * h + 4 * j + 1] ^ sgn,
                                         v[EC * h + 4 * j + 2] ^ sgn, v[EC * h + 4 * j + 3] ^ sgn);
              const int sw = j ^ ((lane >> 1) & 3);  // 64B swizzle of the [32][16 fp32] box
              sts128(smem_u32(buf) + lane * (EC * 4) + sw * 16, w);
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              if (row0 < args.n) {
                const CUtensorMap* cm = d == 0 ? &P.c : &P.cx[d - 1];
                const int cc0 = d == 0 ? P.c_col0 : P.cx_col0[d - 1];
                if (args.overwrite)
                  tma_store_2d(cm, buf, cc0 + col0 + EC * h, row0);
                else
                  tma_reduce_add_2d(cm, buf, cc0 + col0 + EC * h, row0);
              }
              asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            }
          }
        }
      }
    }
#if PACO_EXIT_WAIT_READ
    // exit once the last boxes have been READ out of shared memory: the global
    // writes still complete before the grid does (a dependent launch's
    // griddepcontrol.wait sees them), and the next CTA can take this SM meanwhile
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
#else
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
#endif
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no MMA of the pair writes TMEM and no remote arrive is pending any more
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(L::TMEM_COLS));
  }
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
             int64_t cols, int64_t ld, uint32_t box_cols, uint32_t box_rows, int32_t* col_off,
             CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
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
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) for %lldx%lld ld=%lld", int(r), (long long)rows,
              (long long)cols, (long long)ld);
    return PACO_ERR_CUDA;
  }
  return PACO_OK;
}

}  // namespace

int encode_map_2d(CUtensorMap* map, int elsize, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                  uint32_t box_cols, uint32_t box_rows) {
  if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0) {
    set_error("internal: tensor map base must be 16-byte aligned");
    return PACO_ERR_UNSUPPORTED;
  }
  int32_t off = 0;
  return make_map(map, elsize == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, elsize, ptr,
                  rows, cols, ld, box_cols, box_rows, &off, CU_TENSOR_MAP_SWIZZLE_NONE);
}

namespace {
// ---------------------------------------------------------------------------
// Early operand loads under programmatic dependent launch.  The tcgen05 kernels
// signal launch_dependents at entry, so the next launch on the stream may start
// while they (and, transitively, their own predecessors) still run; its
// griddepcontrol.wait then orders everything after it.  A resident-B launch may
// TMA-load its first tile before that wait only if no operand byte can be
// written by a launch still in flight: kernels without the early signal (every
// other kernel of this library, and the caller's) finish before a dependent
// starts, so only this library's tcgen05 launches matter, and their outputs
// are recorded per stream here (the last kPdlKeep ranges: a superset of any
// chain that can still be resident).  Assumes no third-party kernel that
// itself signals launch_dependents early writes the operands right before.
// ---------------------------------------------------------------------------
struct MemRange {
  uintptr_t lo, hi;
};
MemRange view_range(const void* p, int64_t ld, int64_t rows, int64_t cols, int es) {
  const uintptr_t lo = reinterpret_cast<uintptr_t>(p);
  if (rows <= 0 || cols <= 0) return {lo, lo};
  return {lo, lo + uintptr_t(((rows - 1) * ld + cols) * int64_t(es))};
}
std::mutex g_pdl_mu;  // held from the check to the launch: record order = stream order
std::map<std::pair<int, cudaStream_t>, std::vector<MemRange>> g_pdl_out;
constexpr size_t kPdlKeep = 1024;
// true: none of `reads` overlaps a recorded output; then `writes` are recorded
bool pdl_track(int device, cudaStream_t st, const MemRange* reads, int nr, const MemRange* writes, int nw) {
  std::vector<MemRange>& q = g_pdl_out[{device, st}];
  bool ok = nr > 0;
  for (int i = 0; i < nr && ok; ++i)
    for (const MemRange& w : q)
      if (reads[i].lo < w.hi && w.lo < reads[i].hi) {
        ok = false;
        break;
      }
  for (int i = 0; i < nw; ++i) q.push_back(writes[i]);
  if (q.size() > kPdlKeep) q.erase(q.begin(), q.begin() + (q.size() - kPdlKeep));
  return ok;
}
// record a batch's destinations: dst[4 q + d] for d < ndst[q], or single[q]
void pdl_record(int device, cudaStream_t st, int count, const int32_t* ndst, void* const* dst,
                const void* const* single, int64_t ldc, int64_t n, int64_t m) {
  std::vector<MemRange> w;
  for (int q = 0; q < count; ++q) {
    if (ndst)
      for (int d = 0; d < ndst[q]; ++d) w.push_back(view_range(dst[4 * q + d], ldc, n, m, 4));
    else if (single)
      w.push_back(view_range(single[q], ldc, n, m, 4));
  }
  pdl_track(device, st, nullptr, 0, w.data(), int(w.size()));
}

// Scratch for split / repacked operands: stream-ordered allocations from the
// device's default memory pool (kept cached: release threshold = max), freed
// on the launch stream after the kernel.  Concurrent launches on different
// streams (mm_execute workers, Strassen leaves) each get their own buffers.
struct Scratch {
  cudaStream_t st = nullptr;
  std::vector<void*> bufs;
  ~Scratch() {
    for (void* p : bufs) cudaFreeAsync(p, st);
  }
};

// Tile-scheduler counters of the tcgen05 launches on one (device, stream):
// allocated zeroed once; each kernel leaves them zeroed when it finishes, so
// consecutive launches on a stream need no memset, and launches on different
// streams (the parallel executors) never share counters.
// PDL on the tcgen05 launches (PACO_TC_PDL=0 turns it off)
static const bool kPdl = !dev_knob("PACO_TC_PDL") || atoi(dev_knob("PACO_TC_PDL")) != 0;

int stream_counters(int device, cudaStream_t st, int32_t** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, int32_t*> slots;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(device, st);
  auto it = slots.find(key);
  if (it == slots.end()) {
    cudaStreamCaptureStatus cap;
    PACO_CUDA_TRY(cudaStreamIsCapturing(st, &cap));
    if (cap != cudaStreamCaptureStatusNone) {  // no synchronous allocation inside a capture
      *out = nullptr;
      return PACO_OK;
    }
    void* p = nullptr;
    PACO_CUDA_TRY(cudaMalloc(&p, sizeof(int32_t) * (kNumSMs + 1)));
    PACO_CUDA_TRY(cudaMemset(p, 0, sizeof(int32_t) * (kNumSMs + 1)));
    it = slots.emplace(key, static_cast<int32_t*>(p)).first;
  }
  *out = it->second;
  return PACO_OK;
}

int scratch(int device, Scratch& sc, size_t bytes, cudaStream_t st, void** out) {
  static std::mutex mu;
  static bool pool_ready[64] = {};
  {
    std::lock_guard<std::mutex> lock(mu);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    PACO_CUDA_TRY(cudaStreamIsCapturing(st, &cs));
    // pool attributes may not change while a stream captures (a CUDA graph's
    // first launch through the library): set them at the next uncaptured call
    if (!pool_ready[device & 63] && cs == cudaStreamCaptureStatusNone) {
      cudaMemPool_t pool;
      PACO_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, device));
      uint64_t keep = UINT64_MAX;
      PACO_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
      pool_ready[device & 63] = true;
    }
  }
  sc.st = st;
  PACO_CUDA_TRY(cudaMallocAsync(out, bytes, st));
  sc.bufs.push_back(*out);
  return PACO_OK;
}

// TMA takes a view in place only when its first element and row pitch are
// 16-byte aligned: a tensor map over an aligned-down base with a column
// offset is accepted by cuTensorMapEncodeTiled, but boxes whose rows start
// off a 16-byte boundary never complete (the kernel's bounded mbarrier wait
// then traps) -- such views are repacked into scratch instead.
bool pitch_ok(const void* p, int64_t ld, int elsize) {
  return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && (ld * elsize) % 16 == 0;
}

// C is written by TMA stores / reduce-adds, which clip at the tensor edge in
// 16-byte units: a row end inside a 16-byte chunk would clobber (or add into)
// the neighbouring columns, which may belong to another task's block of C.
bool c_ok(const void* p, int64_t ld, int64_t m) { return pitch_ok(p, ld, 4) && (m * 4) % 16 == 0; }
}  // namespace

namespace tc {
// x -> (hi, lo) = (tf32_rn(x), tf32_rn(x - hi)).  Packed outputs with a 16-byte row pitch `ldo`; kT writes them transposed
// (cols x rows) through a 32x32 smem tile so both sides stay coalesced.

// Up to four signed input views summed (Strassen S/T formation, PAPER.md:
// 1839-1852) and split; nin = 1, coef = +1 is the plain split.
struct SplitIn {
  const float* p[4];
  int64_t ld[4];
  int32_t coef[4];
  int32_t nin;
};

__device__ __forceinline__ float lc_value(const SplitIn& in, int64_t i, int64_t j) {
  float v = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (q < in.nin) {
      const float x = in.p[q][i * in.ld[q] + j];
      v = in.coef[q] > 0 ? v + x : v - x;
    }
  return v;
}

// Transposed output (cols x rows) through a 64x64 smem tile: 16-byte loads
// along the input rows, 16-byte stores along the output rows (the K-major
// B^T the 3xTF32 MMAs read).  kVec: every view 16 B aligned, cols % 4 == 0.
// kB2 (the tf32 + 2 x bf16 format): hi = tf32_rn(x) as fp32, h16 = bf16_rn(hi),
// l16 = bf16_rn(x - hi) -- `lo` unused.

template <bool kVec, bool kB2>
__global__ void __launch_bounds__(256) split_tf32_t_kernel(const SplitIn in, float* __restrict__ hi,
                                                           float* __restrict__ lo, int64_t ldo, int64_t rows,
                                                           int64_t cols, __nv_bfloat16* __restrict__ h16,
                                                           __nv_bfloat16* __restrict__ l16) {
  __shared__ float th[64][65], tl[64][65];
  const int64_t r0 = int64_t(blockIdx.y) * 64, c0 = int64_t(blockIdx.x) * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  // interior tile: all 4 rows x nin 16-byte loads in flight before any arithmetic
  float4 xin[4][4];
  const bool interior = kVec && r0 + 64 <= rows && c0 + 64 <= cols;
  if (interior) {
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < in.nin)
          xin[p][q] = __ldcs(reinterpret_cast<const float4*>(in.p[q] + (r0 + ty + 16 * p) * in.ld[q] + c0 + 4 * tx));
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int r = ty + 16 * p;
    const int64_t i = r0 + r, j = c0 + 4 * tx;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (interior) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < in.nin) {
          const float sg = in.coef[q] > 0 ? 1.f : -1.f;
          v[0] += sg * xin[p][q].x;
          v[1] += sg * xin[p][q].y;
          v[2] += sg * xin[p][q].z;
          v[3] += sg * xin[p][q].w;
        }
    } else if (i < rows) {
      if (kVec && j + 3 < cols) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q < in.nin) {
            const float4 x = *reinterpret_cast<const float4*>(in.p[q] + i * in.ld[q] + j);
            const float sg = in.coef[q] > 0 ? 1.f : -1.f;
            v[0] += sg * x.x;
            v[1] += sg * x.y;
            v[2] += sg * x.z;
            v[3] += sg * x.w;
          }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = j + e < cols ? lc_value(in, i, j + e) : 0.f;
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float h = round_tf32(v[e]);
      th[r][4 * tx + e] = h;
      // 3xTF32: the MMA would truncate an unrounded lo; kB2: the exact x - hi (bf16-rounded at the store)
      tl[r][4 * tx + e] = kB2 ? v[e] - h : round_tf32(v[e] - h);
    }
  }
  __syncthreads();
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int c = ty + 16 * p;                 // output row j = c0 + c (a column of x)
    const int64_t j = c0 + c, i = r0 + 4 * tx;  // 4 consecutive output columns (rows of x)
    if (j >= cols) continue;
    const float4 h = make_float4(th[4 * tx][c], th[4 * tx + 1][c], th[4 * tx + 2][c], th[4 * tx + 3][c]);
    const float4 l = make_float4(tl[4 * tx][c], tl[4 * tx + 1][c], tl[4 * tx + 2][c], tl[4 * tx + 3][c]);
    if (kVec && i + 3 < rows) {
      *reinterpret_cast<float4*>(hi + j * ldo + i) = h;
      if constexpr (kB2) {
        if (h16)
          *reinterpret_cast<uint2*>(h16 + j * ldo + i) = make_uint2(pack_bf16x2(h.x, h.y), pack_bf16x2(h.z, h.w));
        *reinterpret_cast<uint2*>(l16 + j * ldo + i) = make_uint2(pack_bf16x2(l.x, l.y), pack_bf16x2(l.z, l.w));
      } else {
        *reinterpret_cast<float4*>(lo + j * ldo + i) = l;
      }
    } else {
      const float hv[4] = {h.x, h.y, h.z, h.w}, lv[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (i + e < rows) {
          hi[j * ldo + i + e] = hv[e];
          if constexpr (kB2) {
            if (h16) h16[j * ldo + i + e] = __float2bfloat16_rn(hv[e]);
            l16[j * ldo + i + e] = __float2bfloat16_rn(lv[e]);
          } else {
            lo[j * ldo + i + e] = lv[e];
          }
        }
    }
  }
}

// Row-major output, 4 consecutive elements per thread (16 B accesses when
// every view is 16 B aligned: vec), rows strided over the grid's y.
template <bool kVec, bool kB2>
__global__ void split_tf32_n_kernel(const SplitIn in, float* __restrict__ hi, float* __restrict__ lo,
                                    int64_t ldo, int64_t rows, int64_t cols, __nv_bfloat16* __restrict__ h16,
                                    __nv_bfloat16* __restrict__ l16) {
  const int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (j >= cols) return;
  int64_t i0 = blockIdx.y;
  if (kVec) {
    // U rows per pass, every row's loads issued before any arithmetic or store:
    // U x nin 16-byte loads in flight per thread (one row at a time left the
    // kernel at ~4.6 TB/s)
    constexpr int U = 4;
    const int64_t gy = gridDim.y;
    for (; i0 + (U - 1) * gy < rows; i0 += U * gy) {
      float4 x[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q < in.nin) x[u][q] = __ldcs(reinterpret_cast<const float4*>(in.p[q] + (i0 + u * gy) * in.ld[q] + j));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q < in.nin) {
            const float sg = in.coef[q] > 0 ? 1.f : -1.f;
            v[0] += sg * x[u][q].x;
            v[1] += sg * x[u][q].y;
            v[2] += sg * x[u][q].z;
            v[3] += sg * x[u][q].w;
          }
        float h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          h[e] = round_tf32(v[e]);
          l[e] = kB2 ? v[e] - h[e] : round_tf32(v[e] - h[e]);
        }
        const int64_t i = i0 + u * gy;
        __stcs(reinterpret_cast<float4*>(hi + i * ldo + j), make_float4(h[0], h[1], h[2], h[3]));
        if constexpr (kB2) {
          if (h16)
            __stcs(reinterpret_cast<uint2*>(h16 + i * ldo + j),
                   make_uint2(pack_bf16x2(h[0], h[1]), pack_bf16x2(h[2], h[3])));
          __stcs(reinterpret_cast<uint2*>(l16 + i * ldo + j),
                 make_uint2(pack_bf16x2(l[0], l[1]), pack_bf16x2(l[2], l[3])));
        } else {
          __stcs(reinterpret_cast<float4*>(lo + i * ldo + j), make_float4(l[0], l[1], l[2], l[3]));
        }
      }
    }
  }
  for (int64_t i = i0; i < rows; i += gridDim.y) {
    float v[4];
    if (kVec) {
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < in.nin) {
          const float4 x = *reinterpret_cast<const float4*>(in.p[q] + i * in.ld[q] + j);
          const float s = in.coef[q] > 0 ? 1.f : -1.f;
          v[0] += s * x.x;
          v[1] += s * x.y;
          v[2] += s * x.z;
          v[3] += s * x.w;
        }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = j + e < cols ? lc_value(in, i, j + e) : 0.f;
    }
    float h[4], l[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      h[e] = round_tf32(v[e]);
      l[e] = kB2 ? v[e] - h[e] : round_tf32(v[e] - h[e]);
    }
    if (kVec) {
      *reinterpret_cast<float4*>(hi + i * ldo + j) = make_float4(h[0], h[1], h[2], h[3]);
      if constexpr (kB2) {
        if (h16)
          *reinterpret_cast<uint2*>(h16 + i * ldo + j) = make_uint2(pack_bf16x2(h[0], h[1]), pack_bf16x2(h[2], h[3]));
        *reinterpret_cast<uint2*>(l16 + i * ldo + j) = make_uint2(pack_bf16x2(l[0], l[1]), pack_bf16x2(l[2], l[3]));
      } else {
        *reinterpret_cast<float4*>(lo + i * ldo + j) = make_float4(l[0], l[1], l[2], l[3]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (j + e < cols) {
          hi[i * ldo + j + e] = h[e];
          if constexpr (kB2) {
            if (h16) h16[i * ldo + j + e] = __float2bfloat16_rn(h[e]);
            l16[i * ldo + j + e] = __float2bfloat16_rn(l[e]);
          } else {
            lo[i * ldo + j + e] = l[e];
          }
        }
    }
  }
}
}  // namespace tc

namespace {
// Repack an operand whose row pitch TMA cannot take into padded scratch.
int repack(int device, Scratch& sc, const void** p, int64_t* ld, int64_t rows, int64_t cols, int elsize,
           cudaStream_t st) {
  if (pitch_ok(*p, *ld, elsize)) return PACO_OK;
  const int64_t q = 16 / elsize, ld2 = (cols + q - 1) / q * q;
  void* dst;
  int rc = scratch(device, sc, size_t(rows) * ld2 * elsize, st, &dst);
  if (rc) return rc;
  PACO_CUDA_TRY(cudaMemcpy2DAsync(dst, ld2 * elsize, *p, *ld * elsize, cols * elsize, rows,
                                  cudaMemcpyDeviceToDevice, st));
  *p = dst;
  *ld = ld2;
  return PACO_OK;
}

// x = sum coef_q in_q (rows x cols) -> hi/lo tf32 pair with row pitch ldo
// (elements), transposed (cols x rows) if `transpose`.
int launch_split(const tc::SplitIn& in, int64_t rows, int64_t cols, bool transpose, float* h, float* l,
                 int64_t ldo, cudaStream_t st, __nv_bfloat16* h16 = nullptr, __nv_bfloat16* l16 = nullptr) {
  if (rows <= 0 || cols <= 0) return PACO_OK;
  KernelSpan ks(PACO_KT_TF32_SPLIT, st);
  const bool b2 = l16 != nullptr;  // h16 may be null: the kernel forms bf16(hi) itself
  bool vec = (ldo % 4 == 0) && (reinterpret_cast<uintptr_t>(h) % 16 == 0) &&
             (b2 ? (reinterpret_cast<uintptr_t>(h16) % 8 == 0 && reinterpret_cast<uintptr_t>(l16) % 8 == 0)
                 : (reinterpret_cast<uintptr_t>(l) % 16 == 0));
  for (int q = 0; q < in.nin; ++q)
    vec = vec && (in.ld[q] % 4 == 0) && (reinterpret_cast<uintptr_t>(in.p[q]) % 16 == 0);
  if (transpose) {
    dim3 grid(unsigned((cols + 63) / 64), unsigned((rows + 63) / 64));
    if (b2 && vec)
      tc::split_tf32_t_kernel<true, true><<<grid, 256, 0, st>>>(in, h, l, ldo, rows, cols, h16, l16);
    else if (b2)
      tc::split_tf32_t_kernel<false, true><<<grid, 256, 0, st>>>(in, h, l, ldo, rows, cols, h16, l16);
    else if (vec)
      tc::split_tf32_t_kernel<true, false><<<grid, 256, 0, st>>>(in, h, l, ldo, rows, cols, h16, l16);
    else
      tc::split_tf32_t_kernel<false, false><<<grid, 256, 0, st>>>(in, h, l, ldo, rows, cols, h16, l16);
  } else {
    vec = vec && (cols % 4 == 0);
    const int64_t xblocks = (cols / 4 + 1 + 127) / 128;
    const int64_t yblocks = rows < 65535 ? rows : 65535;
    dim3 grid(unsigned(xblocks), unsigned(yblocks > 2368 / xblocks + 1 ? 2368 / xblocks + 1 : yblocks));
    if (b2 && vec)
      tc::split_tf32_n_kernel<true, true><<<grid, 128, 0, st>>>(in, h, l, ldo, rows, cols, h16, l16);
    else if (b2)
      tc::split_tf32_n_kernel<false, true><<<grid, 128, 0, st>>>(in, h, l, ldo, rows, cols, h16, l16);
    else if (vec)
      tc::split_tf32_n_kernel<true, false><<<grid, 128, 0, st>>>(in, h, l, ldo, rows, cols, h16, l16);
    else
      tc::split_tf32_n_kernel<false, false><<<grid, 128, 0, st>>>(in, h, l, ldo, rows, cols, h16, l16);
  }
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
}

// fp32 operand -> packed hi/lo tf32 pair in scratch; `transpose` stores them
// as (cols x rows), i.e. K-major for a B operand.
int split_operand(int device, Scratch& sc, const void* x, int64_t ldx, int64_t rows, int64_t cols,
                  bool transpose, cudaStream_t st, const void** hi, const void** lo, int64_t* ld) {
  const int64_t orows = transpose ? cols : rows, ocols = transpose ? rows : cols;
  const int64_t ld2 = (ocols + 3) / 4 * 4;
  void *h, *l;
  int rc = scratch(device, sc, size_t(orows) * ld2 * 4, st, &h);
  if (rc) return rc;
  if ((rc = scratch(device, sc, size_t(orows) * ld2 * 4, st, &l))) return rc;
  tc::SplitIn in{};
  in.p[0] = static_cast<const float*>(x);
  in.ld[0] = ldx;
  in.coef[0] = 1;
  in.nin = 1;
  if ((rc = launch_split(in, rows, cols, transpose, static_cast<float*>(h), static_cast<float*>(l), ld2, st)))
    return rc;
  *hi = h;
  *lo = l;
  *ld = ld2;
  return PACO_OK;
}
}  // namespace

// 3xTF32 operands already split (paco_tf32_split): A hi/lo n x k, B^T hi/lo m x k,
// one entry per problem of a batch.
struct Presplit {
  const void *ah, *al, *bh, *bl;
  void* c;
};

// Operand maps of one problem.  Plain calls split (3xTF32) or repack (bf16
// with a pitch TMA cannot take) into stream-ordered scratch first.
template <class K>
int build_operands(int device, Scratch& sc, cudaStream_t stream, const void* A, int64_t lda, const void* B,
                   int64_t ldb, int64_t n, int64_t m, int64_t k, const Presplit* pre, int64_t pre_lda,
                   int64_t pre_ldb, tc::TcProb& P) {
  using L = tc::Layout<K>;
  int rc;
  if constexpr (K::NOPS == 1) {
    if ((rc = repack(device, sc, &A, &lda, n, k, K::ELEM, stream))) return rc;
    if ((rc = repack(device, sc, &B, &ldb, k, m, K::ELEM, stream))) return rc;
    if ((rc = make_map(&P.a[0], K::DT, K::ELEM, A, n, k, lda, K::BK, tc::BM, &P.a_col0[0]))) return rc;
    if ((rc = make_map(&P.b[0], K::DT, K::ELEM, B, k, m, ldb, L::BOX_N, K::BK, &P.b_col0[0]))) return rc;
  } else {
    const void *ah, *al, *bh, *bl;
    int64_t lda2, ldb2;
    if (pre) {
      if (!K::B_KMAJOR) {
        set_error("internal: pre-split B operands are K-major");
        return PACO_ERR_UNSUPPORTED;
      }
      ah = pre->ah, al = pre->al, bh = pre->bh, bl = pre->bl, lda2 = pre_lda, ldb2 = pre_ldb;
      if (!pitch_ok(ah, lda2, 4) || !pitch_ok(al, lda2, 4) || !pitch_ok(bh, ldb2, 4) || !pitch_ok(bl, ldb2, 4)) {
        set_error("paco_mm_tf32x3: operand row pitches must be multiples of 16 bytes");
        return PACO_ERR_UNSUPPORTED;
      }
    } else {
      if ((rc = split_operand(device, sc, A, lda, n, k, false, stream, &ah, &al, &lda2))) return rc;
      if ((rc = split_operand(device, sc, B, ldb, k, m, K::B_KMAJOR, stream, &bh, &bl, &ldb2))) return rc;
    }
    constexpr CUtensorMapSwizzle SW = K::SWZ == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
    if ((rc = make_map(&P.a[0], K::DT, K::ELEM, ah, n, k, lda2, K::BK, tc::BM, &P.a_col0[0], SW))) return rc;
    if ((rc = make_map(&P.a[1], K::DT, K::ELEM, al, n, k, lda2, K::BK, tc::BM, &P.a_col0[1], SW))) return rc;
    if constexpr (K::B_KMAJOR) {
      if ((rc = make_map(&P.b[0], K::DT, K::ELEM, bh, m, k, ldb2, K::BK, K::BN, &P.b_col0[0], SW))) return rc;
      if ((rc = make_map(&P.b[1], K::DT, K::ELEM, bl, m, k, ldb2, K::BK, K::BN, &P.b_col0[1], SW))) return rc;
    } else {
      if ((rc = make_map(&P.b[0], K::DT, K::ELEM, bh, k, m, ldb2, L::BOX_N, K::BK, &P.b_col0[0]))) return rc;
      if ((rc = make_map(&P.b[1], K::DT, K::ELEM, bl, k, m, ldb2, L::BOX_N, K::BK, &P.b_col0[1]))) return rc;
    }
  }
  return PACO_OK;
}

template <class K>
int build_output(tc::TcProb& P, void* C, int64_t ldc, int64_t n, int64_t m, CUtensorMap* map = nullptr,
                 int32_t* col0 = nullptr) {
  if (!map) {
    P.ndst = 1;
    P.neg = 0;
  }
  return make_map(map ? map : &P.c, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, C, n, m, ldc, K::EPI_COLS, 32,
                  col0 ? col0 : &P.c_col0, K::EPI_COLS == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
}

template <class K>
int check_tc_call(void* C, int64_t ldc, int64_t n, int64_t m, int64_t k, const int32_t* pieces, int n_pieces,
                  int flags) {
  if (pieces && n_pieces > 0) {
    set_error("the tcgen05 kernels take their own CTA plan (pass pieces=NULL)");
    return PACO_ERR_UNSUPPORTED;
  }
  if (n > INT32_MAX || m > INT32_MAX || k > INT32_MAX) {
    set_error("tcgen05 path: extents must fit int32");
    return PACO_ERR_ARG;
  }
  if ((flags & (PACO_MM_REMOTE | PACO_MM_SYS)) || ((flags & PACO_MM_ATOMIC) && !c_ok(C, ldc, m))) {
    // the TMA reduce-add epilogue is atomic, but only on local C with a TMA-able pitch
    set_error("tcgen05 path: atomic folding needs a local C with a 16-byte aligned start, pitch and row length");
    return PACO_ERR_UNSUPPORTED;
  }
  if ((flags & PACO_MM_ATOMIC) && (flags & PACO_MM_OVERWRITE)) {
    set_error("PACO_MM_OVERWRITE cannot be combined with atomic folding");
    return PACO_ERR_ARG;
  }
  return PACO_OK;
}

template <class K>
int run_tc(int device, Scratch& sc, cudaStream_t stream, const tc::TcMaps& maps, int count, int64_t n, int64_t m,
           int64_t k, int flags, bool early = false) {
  using L = tc::Layout<K>;
  int rc;
  tc::TcArgs args;
  args.n = n;
  args.m = m;
  args.k = k;
  args.count = count;
  args.overwrite = (flags & PACO_MM_OVERWRITE) ? 1 : 0;
  args.tiles_rb = int32_t((n + tc::BM - 1) / tc::BM);
  args.tiles_nb = int32_t((m + K::BN - 1) / K::BN);
  args.kblocks = int32_t((k + K::BK - 1) / K::BK);
  {
    static const int ablate = dev_knob("PACO_TC_ABLATE") ? atoi(dev_knob("PACO_TC_ABLATE")) : 0;
    args.ablate = ablate;
    args.trace = g_trace_buffer;
  }
  const int64_t tiles = int64_t(args.tiles_rb) * args.tiles_nb * count;
  if (tiles > INT32_MAX) {
    set_error("tcgen05 path: too many tiles");
    return PACO_ERR_ARG;
  }
  const int grid = int(tiles < kNumSMs ? tiles : kNumSMs);
  // resident B: one group per column block, but only as many groups as divide
  // the grid evenly (148 = 4 x 37), else the groups' CTA counts differ and the
  // smaller groups finish last; a group then walks several column blocks.
  args.groups = 1;
  if (K::B_RES && count == 1) {
    int g = args.tiles_nb < grid ? args.tiles_nb : grid;
    while (g > 1 && grid % g) --g;
    args.groups = g;
  }
  static const bool early_on = !dev_knob("PACO_TC_EARLY") || atoi(dev_knob("PACO_TC_EARLY")) != 0;
  args.early = (early && early_on) || PACO_TC_EARLY_ABLATE ? 1 : 0;
  if ((rc = stream_counters(device, stream, &args.sched))) return rc;
  if (!args.sched) {  // first launch on a capturing stream: stream-ordered counters
    void* counters;
    if ((rc = scratch(device, sc, sizeof(int32_t) * (kNumSMs + 1), stream, &counters))) return rc;
    PACO_CUDA_TRY(cudaMemsetAsync(counters, 0, sizeof(int32_t) * (kNumSMs + 1), stream));
    args.sched = static_cast<int32_t*>(counters);
  }
  auto kern = tc::tc_gemm_kernel<K>;
  {
    static std::atomic<uint64_t> attr_set{0};  // devices whose attribute is set
    const uint64_t bit = uint64_t(1) << (device & 63);
    if (!(attr_set.load() & bit)) {
      PACO_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM_ALLOC));
      attr_set.fetch_or(bit);
    }
  }
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(L::THREADS);
    cfg.dynamicSmemBytes = L::SMEM_ALLOC;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = kPdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    KernelSpan ks(PACO_KT_TC_GEMM, stream);
    PACO_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, maps, args));
  }
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
}

template <class K>
int launch_tc(int device, cudaStream_t stream, const void* A, int64_t lda, const void* B, int64_t ldb,
              void* C, int64_t ldc, int64_t n, int64_t m, int64_t k, const int32_t* pieces, int n_pieces,
              int flags) {
  int rc;
  if ((rc = check_tc_call<K>(C, ldc, n, m, k, pieces, n_pieces, flags))) return rc;
  Scratch sc;  // freed (stream-ordered) when this call returns
  static tc::TcMaps maps;  // ~5.6 KB, copied into the launch's parameter buffer
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if ((rc = build_operands<K>(device, sc, stream, A, lda, B, ldb, n, m, k, nullptr, 0, 0, maps.p[0]))) return rc;
  void* c_user = nullptr;
  int64_t ldc_user = ldc;
  if (!c_ok(C, ldc, m)) {  // stage C through padded scratch, copy back exactly n x m
    const int64_t ld2 = (m + 3) / 4 * 4;
    void* p;
    if ((rc = scratch(device, sc, size_t(n) * ld2 * 4, stream, &p))) return rc;
    if (!(flags & PACO_MM_OVERWRITE))
      PACO_CUDA_TRY(cudaMemcpy2DAsync(p, ld2 * 4, C, ldc * 4, m * 4, n, cudaMemcpyDeviceToDevice, stream));
    c_user = C;
    C = p;
    ldc = ld2;
  }
  if ((rc = build_output<K>(maps.p[0], C, ldc, n, m))) return rc;
  bool early;
  {
    std::lock_guard<std::mutex> pl(g_pdl_mu);
    const MemRange rd[2] = {view_range(A, lda, n, k, K::ELEM),
                            K::B_KMAJOR ? view_range(B, ldb, m, k, K::ELEM) : view_range(B, ldb, k, m, K::ELEM)};
    const MemRange wr[2] = {view_range(C, ldc, n, m, 4), view_range(c_user ? c_user : C, ldc_user, n, m, 4)};
    early = pdl_track(device, stream, rd, 2, wr, 2);
    if ((rc = run_tc<K>(device, sc, stream, maps, 1, n, m, k, flags, early))) return rc;
  }
  if (c_user)
    PACO_CUDA_TRY(cudaMemcpy2DAsync(c_user, ldc_user * 4, C, ldc * 4, m * 4, n, cudaMemcpyDeviceToDevice, stream));
  return PACO_OK;
}

// A batch of same-shape 3xTF32 problems from pre-split operands, one launch
// (one tile queue): Strassen's seven leaf products of a node.
// Optional destination lists (ndst/dst/sign, problem q's at [4q, 4q + ndst[q])):
// each product is folded (+)= or (-)= into every one of its destinations by the
// epilogue's TMA reduce-adds -- Strassen's C-block combination without the
// M buffers or the combination pass.
template <class K>
int launch_tc_batch(int device, cudaStream_t stream, int count, const Presplit* pre, int64_t lda, int64_t ldb,
                    int64_t ldc, int64_t n, int64_t m, int64_t k, int flags, const int32_t* ndst = nullptr,
                    void* const* dst = nullptr, const int32_t* sign = nullptr) {
  int rc;
  if (count < 1 || count > tc::kMaxBatch) {
    set_error("paco_mm_tf32x3: count=%d (1..%d)", count, tc::kMaxBatch);
    return PACO_ERR_ARG;
  }
#if !PACO_EPI_RING
  if (ndst) {  // only the staging-ring epilogue walks the destination list and applies the signs
    set_error("paco_mm_tf32x3_multi: this build's epilogue (PACO_EPI_RING=0) has no multi-destination fold");
    return PACO_ERR_UNSUPPORTED;
  }
#endif
  for (int q = 0; q < count; ++q) {
    const int nd = ndst ? ndst[q] : 1;
    if (nd < 1 || nd > 4) {
      set_error("paco_mm_tf32x3_multi: problem %d has %d destinations (1..4)", q, nd);
      return PACO_ERR_ARG;
    }
    for (int d = 0; d < nd; ++d) {
      void* c = ndst ? dst[4 * q + d] : pre[q].c;
      if ((rc = check_tc_call<K>(c, ldc, n, m, k, nullptr, 0, flags))) return rc;
      if (!c_ok(c, ldc, m)) {
        set_error("paco_mm_tf32x3: C needs a 16-byte aligned start, row pitch and row length");
        return PACO_ERR_UNSUPPORTED;
      }
    }
  }
  Scratch sc;
  static tc::TcMaps maps;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  for (int q = 0; q < count; ++q) {
    if ((rc = build_operands<K>(device, sc, stream, nullptr, 0, nullptr, 0, n, m, k, &pre[q], lda, ldb, maps.p[q])))
      return rc;
    tc::TcProb& P = maps.p[q];
    if ((rc = build_output<K>(P, ndst ? dst[4 * q] : pre[q].c, ldc, n, m))) return rc;
    if (ndst) {
      P.ndst = ndst[q];
      for (int d = 0; d < ndst[q]; ++d) {
        if (sign[4 * q + d] < 0) P.neg |= 1u << d;
        if (d > 0 && (rc = build_output<K>(P, dst[4 * q + d], ldc, n, m, &P.cx[d - 1], &P.cx_col0[d - 1])))
          return rc;
      }
    }
  }
  std::lock_guard<std::mutex> pl(g_pdl_mu);
  {
    const void* cs[tc::kMaxBatch];
    for (int q = 0; q < count; ++q) cs[q] = pre[q].c;
    pdl_record(device, stream, count, ndst, dst, cs, ldc, n, m);
  }
  return run_tc<K>(device, sc, stream, maps, count, n, m, k, flags);
}

#ifndef PACO_PAIR_ST
#define PACO_PAIR_ST 6
#endif
// Launch a tc_pair_kernel variant (mode 0: 3xTF32, 1: FA (S_r formed in the kernel),
// 2: tf32 + 2 x bf16, 3/4: ... with bf16 parts formed in the kernel, 5: bf16x3 on
// pre-split bf16 planes) over 256 x 256 tiles dealt to the 74 CTA pairs.
int run_pair(int device, cudaStream_t stream, const tc::TcMaps& maps, int count, int64_t n, int64_t m, int64_t k,
             int flags, int mode) {
  using L = tc::PairLayout<PACO_PAIR_ST>;
  tc::TcArgs args{};
  args.n = n;
  args.m = m;
  args.k = k;
  args.count = count;
  args.overwrite = (flags & PACO_MM_OVERWRITE) ? 1 : 0;
  args.tiles_rb = int32_t((n + 255) / 256);
  args.tiles_nb = int32_t((m + L::BN - 1) / L::BN);
  const int kstep = mode >= 5 ? 2 * L::BK : L::BK;
  args.kblocks = int32_t((k + kstep - 1) / kstep);
  args.groups = 1;
  const int64_t tiles = int64_t(args.tiles_rb) * args.tiles_nb * count;
  const int pairs = int(tiles < kNumSMs / 2 ? tiles : kNumSMs / 2);
  auto kern = mode == 6   ? tc::tc_pair_kernel<PACO_PAIR_ST, false, false, false, false, true, true>
              : mode == 5 ? tc::tc_pair_kernel<PACO_PAIR_ST, false, false, false, false, true>
              : mode == 1 ? tc::tc_pair_kernel<PACO_PAIR_ST, true, false>
              : mode == 2 ? tc::tc_pair_kernel<PACO_PAIR_ST, false, true>
              : mode == 3 ? tc::tc_pair_kernel<PACO_PAIR_ST, false, true, true>
              : mode == 4 ? tc::tc_pair_kernel<PACO_PAIR_ST, false, true, true, true>
                          : tc::tc_pair_kernel<PACO_PAIR_ST, false, false>;
  const int threads = mode == 1   ? tc::PairLayout<PACO_PAIR_ST, true>::THREADS
                      : mode == 3 || mode == 4 ? tc::PairLayout<PACO_PAIR_ST, false, true, true>::THREADS
                                  : L::THREADS;
  {
    static std::atomic<uint64_t> attr_set{0};
    const uint64_t bit = uint64_t(1) << ((device & 7) * 8 + mode);
    if (!(attr_set.load() & bit)) {
      PACO_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM_ALLOC));
      attr_set.fetch_or(bit);
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(2 * pairs));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = L::SMEM_ALLOC;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = kPdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  KernelSpan ks(PACO_KT_TC_GEMM, stream);
  PACO_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, maps, args));
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
}

// 3xTF32 batch on CTA pairs (tc_pair_kernel): same contract as launch_tc_batch
// for pre-split operands, optional destination lists.
// fa_terms (FA): problem q's A is the signed sum of fa_nt[q] raw views fa_terms[2q + t]
// (pre[q].ah/al unused); B^T always pre-split.
int launch_tc_pair(int device, cudaStream_t stream, int count, const Presplit* pre, int64_t lda, int64_t ldb,
                   int64_t ldc, int64_t n, int64_t m, int64_t k, int flags, const int32_t* ndst, void* const* dst,
                   const int32_t* sign, const int32_t* fa_nt = nullptr, const void* const* fa_terms = nullptr,
                   const int32_t* fa_sign = nullptr) {
  using L = tc::PairLayout<PACO_PAIR_ST>;
  const bool fa = fa_nt != nullptr;
  int rc;
  constexpr CUtensorMapSwizzle SW = CU_TENSOR_MAP_SWIZZLE_64B;
  static tc::TcMaps maps;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  for (int q = 0; q < count; ++q) {
    const Presplit& p = pre[q];
    const void* a0 = fa ? fa_terms[2 * q] : p.ah;
    const void* a1 = fa ? (fa_nt[q] > 1 ? fa_terms[2 * q + 1] : fa_terms[2 * q]) : p.al;
    if (!pitch_ok(a0, lda, 4) || !pitch_ok(a1, lda, 4) || !pitch_ok(p.bh, ldb, 4) || !pitch_ok(p.bl, ldb, 4)) {
      set_error("paco_mm_tf32x3: operand row pitches must be multiples of 16 bytes");
      return PACO_ERR_UNSUPPORTED;
    }
    tc::TcProb& P = maps.p[q];
    P.nta = fa ? fa_nt[q] : 2;
    P.sga = fa ? ((fa_sign[2 * q] < 0 ? 1u : 0u) | (fa_nt[q] > 1 && fa_sign[2 * q + 1] < 0 ? 2u : 0u)) : 0u;
    if ((rc = make_map(&P.a[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a0, n, k, lda, L::BK, tc::BM, &P.a_col0[0], SW)) ||
        (rc = make_map(&P.a[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a1, n, k, lda, L::BK, tc::BM, &P.a_col0[1], SW)) ||
        (rc = make_map(&P.b[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, p.bh, m, k, ldb, L::BK, L::BNH, &P.b_col0[0], SW)) ||
        (rc = make_map(&P.b[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, p.bl, m, k, ldb, L::BK, L::BNH, &P.b_col0[1], SW)))
      return rc;
    const int nd = ndst ? ndst[q] : 1;
    P.ndst = nd;
    P.neg = 0;
    for (int d = 0; d < nd; ++d) {
      void* c = ndst ? dst[4 * q + d] : p.c;
      if (ndst && sign[4 * q + d] < 0) P.neg |= 1u << d;
      if ((rc = make_map(d == 0 ? &P.c : &P.cx[d - 1], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, c, n, m, ldc, L::EC, 32,
                         d == 0 ? &P.c_col0 : &P.cx_col0[d - 1], SW)))
        return rc;
    }
  }
  std::lock_guard<std::mutex> pl(g_pdl_mu);
  {
    const void* cs[tc::kMaxBatch];
    for (int q = 0; q < count; ++q) cs[q] = pre[q].c;
    pdl_record(device, stream, count, ndst, dst, cs, ldc, n, m);
  }
  return run_pair(device, stream, maps, count, n, m, k, flags, fa ? 1 : 0);
}

// CTA pairs for the 3xTF32 batches with enough 256 x 256 tiles to keep the 74
// pairs busy (Strassen's leaf levels); PACO_TF32_PAIR=0 forces single CTAs.
bool tf32_pair(int64_t n, int64_t m, int count) {
  static const int v = dev_knob("PACO_TF32_PAIR") ? atoi(dev_knob("PACO_TF32_PAIR")) : -1;
  if (v >= 0) return v != 0;
  return ((n + 255) / 256) * ((m + 255) / 256) * count >= 3 * (kNumSMs / 2);
}

// 3xTF32 tile width: N = 256 halves the B-operand traffic per output (the
// kernel is L2-bandwidth bound at N = 128: 48 flop per loaded byte) but only
// pays when the batch has enough tiles for the 148 SMs (4096^3 alone: 512
// tiles = 3.5 per SM).  PACO_TF32_V=0/1 forces 128/256.
bool tf32_wide(int64_t n, int64_t m, int count) {
  static const int v = dev_knob("PACO_TF32_V") ? atoi(dev_knob("PACO_TF32_V")) : -1;
  if (v >= 0) return v != 0;
  return ((n + 127) / 128) * ((m + 255) / 256) * count >= 6 * kNumSMs;
}

int launch_mm_bf16_tc(int device, cudaStream_t stream, const void* A, int64_t lda, const void* B, int64_t ldb,
                      void* C, int64_t ldc, int64_t n, int64_t m, int64_t k, const int32_t* pieces,
                      int n_pieces, int flags) {
  // k <= 256 (cfg3): resident-B kind, 5-stage A ring, 8 epilogue warps staging
  // 16-column boxes -- measured best of 10 layouts (ring depth 2-8, staging
  // buffers 1-4 per warp, 16/32-column boxes, N = 128 tiles: 58 vs 59.5-84 us;
  // DESIGN.md section 6); PACO_TC_RESV=-1 forces the streaming kind.
  static const int resv = dev_knob("PACO_TC_RESV") ? atoi(dev_knob("PACO_TC_RESV")) : 7;
#define PACO_TC_GO(KIND) return launch_tc<KIND>(device, stream, A, lda, B, ldb, C, ldc, n, m, k, pieces, n_pieces, flags)
  if (k <= 256 && resv >= 0) PACO_TC_GO(PACO_TC_ARGS(tc::KindBF16Res<PACO_RES_AST, PACO_RES_EB, 8, PACO_RES_EC>));
#undef PACO_TC_GO
  return launch_tc<tc::KindBF16>(device, stream, A, lda, B, ldb, C, ldc, n, m, k, pieces, n_pieces, flags);
}

int launch_mm_f32_tc(int device, cudaStream_t stream, const void* A, int64_t lda, const void* B, int64_t ldb,
                     void* C, int64_t ldc, int64_t n, int64_t m, int64_t k, const int32_t* pieces,
                     int n_pieces, int flags) {
  if (tf32_wide(n, m, 1))
    return launch_tc<tc::KindTF32x3W>(device, stream, A, lda, B, ldb, C, ldc, n, m, k, pieces, n_pieces, flags);
  return launch_tc<tc::KindTF32x3>(device, stream, A, lda, B, ldb, C, ldc, n, m, k, pieces, n_pieces, flags);
}

int launch_mm_tf32x3_presplit(int device, cudaStream_t stream, int count, const void* const* ah,
                              const void* const* al, int64_t lda, const void* const* bth, const void* const* btl,
                              int64_t ldb, void* const* C, int64_t ldc, int64_t n, int64_t m, int64_t k,
                              int flags) {
  Presplit pre[tc::kMaxBatch];
  if (count < 1 || count > tc::kMaxBatch) {
    set_error("paco_mm_tf32x3: count=%d (1..%d)", count, tc::kMaxBatch);
    return PACO_ERR_ARG;
  }
  for (int q = 0; q < count; ++q) pre[q] = Presplit{ah[q], al[q], bth[q], btl[q], C[q]};
  if (tf32_pair(n, m, count)) {
    for (int q = 0; q < count; ++q) {
      int rc = check_tc_call<tc::KindTF32x3W>(C[q], ldc, n, m, k, nullptr, 0, flags);
      if (rc) return rc;
      if (!c_ok(C[q], ldc, m)) {
        set_error("paco_mm_tf32x3: C needs a 16-byte aligned start, row pitch and row length");
        return PACO_ERR_UNSUPPORTED;
      }
    }
    return launch_tc_pair(device, stream, count, pre, lda, ldb, ldc, n, m, k, flags, nullptr, nullptr, nullptr);
  }
  if (tf32_wide(n, m, count))
    return launch_tc_batch<tc::KindTF32x3W>(device, stream, count, pre, lda, ldb, ldc, n, m, k, flags);
  return launch_tc_batch<tc::KindTF32x3>(device, stream, count, pre, lda, ldb, ldc, n, m, k, flags);
}

int launch_mm_tf32x3_multi(int device, cudaStream_t stream, int count, const void* const* ah,
                           const void* const* al, int64_t lda, const void* const* bth, const void* const* btl,
                           int64_t ldb, const int32_t* ndst, void* const* dst, const int32_t* sign, int64_t ldc,
                           int64_t n, int64_t m, int64_t k, int flags) {
  Presplit pre[tc::kMaxBatch];
  if (count < 1 || count > tc::kMaxBatch || !ndst || !dst || !sign) {
    set_error("paco_mm_tf32x3_multi: count=%d (1..%d) and destination arrays required", count, tc::kMaxBatch);
    return PACO_ERR_ARG;
  }
  for (int q = 0; q < count; ++q) pre[q] = Presplit{ah[q], al[q], bth[q], btl[q], dst[4 * q]};
  if (tf32_pair(n, m, count)) {
    for (int q = 0; q < count; ++q) {
      if (ndst[q] < 1 || ndst[q] > 4) {
        set_error("paco_mm_tf32x3_multi: problem %d has %d destinations (1..4)", q, ndst[q]);
        return PACO_ERR_ARG;
      }
      for (int d = 0; d < ndst[q]; ++d)
        if (!c_ok(dst[4 * q + d], ldc, m)) {
          set_error("paco_mm_tf32x3: C needs a 16-byte aligned start, row pitch and row length");
          return PACO_ERR_UNSUPPORTED;
        }
    }
    return launch_tc_pair(device, stream, count, pre, lda, ldb, ldc, n, m, k, flags, ndst, dst, sign);
  }
  if (tf32_wide(n, m, count))
    return launch_tc_batch<tc::KindTF32x3W>(device, stream, count, pre, lda, ldb, ldc, n, m, k, flags, ndst, dst,
                                            sign);
  return launch_tc_batch<tc::KindTF32x3>(device, stream, count, pre, lda, ldb, ldc, n, m, k, flags, ndst, dst, sign);
}

// Strassen leaf products with the S_r / T_r formation fused into the kernel
// (KindTF32x3F): problem q multiplies A_q = sum_t a_sign * a_terms[2q + t]
// (n x k, K contiguous, pitch lda; t < nta[q] <= 2) by B_q, given as
// B_q^T = sum_t b_sign * bt_terms[2q + t] (m x k, pitch ldb; t < ntb[q] <= 2),
// and folds the product (+/-) into its ndst[q] destinations (as _multi).
int launch_mm_tf32x3_fused(int device, cudaStream_t stream, int count, const int32_t* nta, const void* const* a_terms,
                           const int32_t* a_sign, int64_t lda, const int32_t* ntb, const void* const* bt_terms,
                           const int32_t* b_sign, int64_t ldb, const int32_t* ndst, void* const* dst,
                           const int32_t* sign, int64_t ldc, int64_t n, int64_t m, int64_t k) {
  using K = tc::KindTF32x3F;
  int rc;
  if (count < 1 || count > tc::kMaxBatch || !nta || !a_terms || !a_sign || !ntb || !bt_terms || !b_sign || !ndst ||
      !dst || !sign) {
    set_error("paco_mm_tf32x3_fused: count=%d (1..%d) and every term / destination array required", count,
              tc::kMaxBatch);
    return PACO_ERR_ARG;
  }
  if (n <= 0 || m <= 0 || k <= 0) return PACO_OK;
  if (n > INT32_MAX || m > INT32_MAX || k > INT32_MAX) {
    set_error("tcgen05 path: extents must fit int32");
    return PACO_ERR_ARG;
  }
  for (int q = 0; q < count; ++q) {
    if (nta[q] < 1 || nta[q] > K::NT || ntb[q] < 1 || ntb[q] > K::NT) {
      set_error("paco_mm_tf32x3_fused: problem %d has %d / %d operand terms (1..%d)", q, nta[q], ntb[q], K::NT);
      return PACO_ERR_ARG;
    }
    for (int t = 0; t < nta[q]; ++t)
      if (!a_terms[2 * q + t] || !pitch_ok(a_terms[2 * q + t], lda, 4)) {
        set_error("paco_mm_tf32x3_fused: A term %d of problem %d needs a 16-byte aligned start and pitch", t, q);
        return PACO_ERR_UNSUPPORTED;
      }
    for (int t = 0; t < ntb[q]; ++t)
      if (!bt_terms[2 * q + t] || !pitch_ok(bt_terms[2 * q + t], ldb, 4)) {
        set_error("paco_mm_tf32x3_fused: B^T term %d of problem %d needs a 16-byte aligned start and pitch", t, q);
        return PACO_ERR_UNSUPPORTED;
      }
    if (ndst[q] < 1 || ndst[q] > 4) {
      set_error("paco_mm_tf32x3_fused: problem %d has %d destinations (1..4)", q, ndst[q]);
      return PACO_ERR_ARG;
    }
    for (int d = 0; d < ndst[q]; ++d)
      if (!c_ok(dst[4 * q + d], ldc, m)) {
        set_error("paco_mm_tf32x3_fused: C needs a 16-byte aligned start, row pitch and row length");
        return PACO_ERR_UNSUPPORTED;
      }
  }
  Scratch sc;
  static tc::TcMaps maps;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  constexpr CUtensorMapSwizzle SW = CU_TENSOR_MAP_SWIZZLE_64B;
  for (int q = 0; q < count; ++q) {
    tc::TcProb& P = maps.p[q];
    for (int t = 0; t < K::NT; ++t) {  // unused term slots repeat term 0 (never loaded)
      const int ta = t < nta[q] ? t : 0, tb = t < ntb[q] ? t : 0;
      if ((rc = make_map(&P.a[t], K::DT, 4, a_terms[2 * q + ta], n, k, lda, K::BK, tc::BM, &P.a_col0[t], SW)))
        return rc;
      if ((rc = make_map(&P.b[t], K::DT, 4, bt_terms[2 * q + tb], m, k, ldb, K::BK, K::BN, &P.b_col0[t], SW)))
        return rc;
    }
    P.nta = nta[q];
    P.ntb = ntb[q];
    P.sga = (a_sign[2 * q] < 0 ? 1u : 0u) | (nta[q] > 1 && a_sign[2 * q + 1] < 0 ? 2u : 0u);
    P.sgb = (b_sign[2 * q] < 0 ? 1u : 0u) | (ntb[q] > 1 && b_sign[2 * q + 1] < 0 ? 2u : 0u);
    if ((rc = build_output<K>(P, dst[4 * q], ldc, n, m))) return rc;
    P.ndst = ndst[q];
    for (int d = 0; d < ndst[q]; ++d) {
      if (sign[4 * q + d] < 0) P.neg |= 1u << d;
      if (d > 0 && (rc = build_output<K>(P, dst[4 * q + d], ldc, n, m, &P.cx[d - 1], &P.cx_col0[d - 1]))) return rc;
    }
  }
  std::lock_guard<std::mutex> pl(g_pdl_mu);
  pdl_record(device, stream, count, ndst, dst, nullptr, ldc, n, m);
  return run_tc<K>(device, sc, stream, maps, count, n, m, k, 0);
}

// Strassen leaf batch on CTA pairs with S_r formed in the kernel (tc_pair_kernel<.., true>):
// A_q = sum_t a_sign * a_terms[2q + t] (t < nta[q] <= 2, pitch lda), B_q^T pre-split (bt_hi / bt_lo).
int launch_mm_tf32x3_fused_a(int device, cudaStream_t stream, int count, const int32_t* nta,
                             const void* const* a_terms, const int32_t* a_sign, int64_t lda, const void* const* bt_hi,
                             const void* const* bt_lo, int64_t ldb, const int32_t* ndst, void* const* dst,
                             const int32_t* sign, int64_t ldc, int64_t n, int64_t m, int64_t k) {
  if (count < 1 || count > tc::kMaxBatch || !nta || !a_terms || !a_sign || !bt_hi || !bt_lo || !ndst || !dst ||
      !sign) {
    set_error("paco_mm_tf32x3_fused_a: count=%d (1..%d) and every term / destination array required", count,
              tc::kMaxBatch);
    return PACO_ERR_ARG;
  }
  if (n <= 0 || m <= 0 || k <= 0) return PACO_OK;
  if (n > INT32_MAX || m > INT32_MAX || k > INT32_MAX) {
    set_error("tcgen05 path: extents must fit int32");
    return PACO_ERR_ARG;
  }
  Presplit pre[tc::kMaxBatch];
  for (int q = 0; q < count; ++q) {
    if (nta[q] < 1 || nta[q] > 2) {
      set_error("paco_mm_tf32x3_fused_a: problem %d has %d A terms (1..2)", q, nta[q]);
      return PACO_ERR_ARG;
    }
    if (ndst[q] < 1 || ndst[q] > 4) {
      set_error("paco_mm_tf32x3_fused_a: problem %d has %d destinations (1..4)", q, ndst[q]);
      return PACO_ERR_ARG;
    }
    for (int d = 0; d < ndst[q]; ++d)
      if (!c_ok(dst[4 * q + d], ldc, m)) {
        set_error("paco_mm_tf32x3_fused_a: C needs a 16-byte aligned start, row pitch and row length");
        return PACO_ERR_UNSUPPORTED;
      }
    pre[q] = Presplit{nullptr, nullptr, bt_hi[q], bt_lo[q], dst[4 * q]};
  }
  return launch_tc_pair(device, stream, count, pre, lda, ldb, ldc, n, m, k, 0, ndst, dst, sign, nta, a_terms, a_sign);
}


// tf32 + 2 x bf16 batch on CTA pairs: C[q] (+/-)= A[q] B[q] with A[q] given as
// (hi fp32, bf16(hi), bf16(x - hi)) n x k (pitch lda, elements) and B[q]^T likewise m x k
// (pitch ldb) -- paco_tf32b2_split outputs -- destinations as _multi.
int launch_mm_tf32b2_multi(int device, cudaStream_t stream, int count, const void* const* a_hi,
                           const void* const* a_h16, const void* const* a_l16, int64_t lda, const void* const* b_hi,
                           const void* const* b_h16, const void* const* b_l16, int64_t ldb, const int32_t* ndst,
                           void* const* dst, const int32_t* sign, int64_t ldc, int64_t n, int64_t m, int64_t k) {
  using L = tc::PairLayout<PACO_PAIR_ST>;
  const bool cv = a_h16 == nullptr;       // bf16(hi) formed in the kernel (mode 3)
  const bool raw = cv && a_l16 == nullptr;  // plain fp32 operands, both bf16 parts formed in the kernel (mode 4)
  if (count < 1 || count > tc::kMaxBatch || !a_hi || !b_hi || !ndst || !dst || !sign ||
      (!cv && (!a_h16 || !b_h16)) || (!raw && (!a_l16 || !b_l16))) {
    set_error("paco_mm_tf32b2_multi: count=%d (1..%d) and every operand / destination array required", count,
              tc::kMaxBatch);
    return PACO_ERR_ARG;
  }
  if (n <= 0 || m <= 0 || k <= 0) return PACO_OK;
  if (n > INT32_MAX || m > INT32_MAX || k > INT32_MAX) {
    set_error("tcgen05 path: extents must fit int32");
    return PACO_ERR_ARG;
  }
  int rc;
  constexpr CUtensorMapSwizzle S64 = CU_TENSOR_MAP_SWIZZLE_64B, S32 = CU_TENSOR_MAP_SWIZZLE_32B;
  constexpr CUtensorMapDataType F32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32, B16 = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  static tc::TcMaps maps;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  for (int q = 0; q < count; ++q) {
    if (!pitch_ok(a_hi[q], lda, 4) || !pitch_ok(b_hi[q], ldb, 4) || (!cv && !pitch_ok(a_h16[q], lda, 2)) ||
        (!raw && !pitch_ok(a_l16[q], lda, 2)) || (!cv && !pitch_ok(b_h16[q], ldb, 2)) ||
        (!raw && !pitch_ok(b_l16[q], ldb, 2))) {
      set_error("paco_mm_tf32b2_multi: operands need 16-byte aligned starts and row pitches");
      return PACO_ERR_UNSUPPORTED;
    }
    if (ndst[q] < 1 || ndst[q] > 4) {
      set_error("paco_mm_tf32b2_multi: problem %d has %d destinations (1..4)", q, ndst[q]);
      return PACO_ERR_ARG;
    }
    tc::TcProb& P = maps.p[q];
    if ((rc = make_map(&P.a[0], F32, 4, a_hi[q], n, k, lda, L::BK, tc::BM, &P.a_col0[0], S64)) ||
        (!raw && (rc = make_map(&P.a[1], B16, 2, cv ? a_l16[q] : a_h16[q], n, k, lda, L::BK, tc::BM,
                                &P.a_col0[1], S32))) ||
        (!raw && (rc = make_map(&P.a2, B16, 2, a_l16[q], n, k, lda, L::BK, tc::BM, &P.a2_col0, S32))) ||
        (rc = make_map(&P.b[0], F32, 4, b_hi[q], m, k, ldb, L::BK, L::BNH, &P.b_col0[0], S64)) ||
        (!raw && (rc = make_map(&P.b[1], B16, 2, cv ? b_l16[q] : b_h16[q], m, k, ldb, L::BK, L::BNH,
                                &P.b_col0[1], S32))) ||
        (!raw && (rc = make_map(&P.b2, B16, 2, b_l16[q], m, k, ldb, L::BK, L::BNH, &P.b2_col0, S32))))
      return rc;
    P.ndst = ndst[q];
    P.neg = 0;
    for (int d = 0; d < ndst[q]; ++d) {
      if (!c_ok(dst[4 * q + d], ldc, m)) {
        set_error("paco_mm_tf32b2_multi: C needs a 16-byte aligned start, row pitch and row length");
        return PACO_ERR_UNSUPPORTED;
      }
      if (sign[4 * q + d] < 0) P.neg |= 1u << d;
      if ((rc = make_map(d == 0 ? &P.c : &P.cx[d - 1], F32, 4, dst[4 * q + d], n, m, ldc, L::EC, 32,
                         d == 0 ? &P.c_col0 : &P.cx_col0[d - 1], S64)))
        return rc;
    }
  }
  if (raw)  // the unused maps are never loaded; give prefetch.tensormap valid ones
    for (int q = 0; q < count; ++q) {
      maps.p[q].a[1] = maps.p[q].a2 = maps.p[q].a[0];
      maps.p[q].b[1] = maps.p[q].b2 = maps.p[q].b[0];
    }
  std::lock_guard<std::mutex> pl(g_pdl_mu);
  pdl_record(device, stream, count, ndst, dst, nullptr, ldc, n, m);
  return run_pair(device, stream, maps, count, n, m, k, 0, raw ? 4 : (cv ? 3 : 2));
}

// bf16x3 batch on CTA pairs: C[q] (+/-)= A[q] B[q] with A[q] = a_hi + a_lo (bf16
// planes, n x k, pitch lda elements) and B[q]^T = b_hi + b_lo (m x k, pitch ldb);
// hi*hi + hi*lo + lo*hi accumulate in fp32 TMEM; destinations as _multi.
// b_natural: B[q] given as k x m planes (pitch ldb) instead of B^T (MN-major tiles).
int launch_mm_bf16x3_multi(int device, cudaStream_t stream, int count, const void* const* a_hi,
                           const void* const* a_lo, int64_t lda, const void* const* b_hi, const void* const* b_lo,
                           int64_t ldb, const int32_t* ndst, void* const* dst, const int32_t* sign, int64_t ldc,
                           int64_t n, int64_t m, int64_t k, int b_natural) {
  using L = tc::PairLayout<PACO_PAIR_ST>;
  constexpr int KSTEP = 2 * L::BK;  // 32 bf16 = one 64-byte swizzled row
  if (count < 1 || count > tc::kMaxBatch || !a_hi || !a_lo || !b_hi || !b_lo || !ndst || !dst || !sign) {
    set_error("paco_mm_bf16x3_multi: count=%d (1..%d) and every operand / destination array required", count,
              tc::kMaxBatch);
    return PACO_ERR_ARG;
  }
  if (n <= 0 || m <= 0 || k <= 0) return PACO_OK;
  if (n > INT32_MAX || m > INT32_MAX || k > INT32_MAX) {
    set_error("tcgen05 path: extents must fit int32");
    return PACO_ERR_ARG;
  }
  int rc;
  constexpr CUtensorMapSwizzle S64 = CU_TENSOR_MAP_SWIZZLE_64B;
  constexpr CUtensorMapDataType F32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32, B16 = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  static tc::TcMaps maps;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  for (int q = 0; q < count; ++q) {
    if (!pitch_ok(a_hi[q], lda, 2) || !pitch_ok(a_lo[q], lda, 2) || !pitch_ok(b_hi[q], ldb, 2) ||
        !pitch_ok(b_lo[q], ldb, 2)) {
      set_error("paco_mm_bf16x3_multi: operands need 16-byte aligned starts and row pitches");
      return PACO_ERR_UNSUPPORTED;
    }
    if (ndst[q] < 1 || ndst[q] > 4) {
      set_error("paco_mm_bf16x3_multi: problem %d has %d destinations (1..4)", q, ndst[q]);
      return PACO_ERR_ARG;
    }
    tc::TcProb& P = maps.p[q];
    if ((rc = make_map(&P.a[0], B16, 2, a_hi[q], n, k, lda, KSTEP, tc::BM, &P.a_col0[0], S64)) ||
        (rc = make_map(&P.a[1], B16, 2, a_lo[q], n, k, lda, KSTEP, tc::BM, &P.a_col0[1], S64)))
      return rc;
    if (b_natural) {
      if ((rc = make_map(&P.b[0], B16, 2, b_hi[q], k, m, ldb, 64, KSTEP, &P.b_col0[0], CU_TENSOR_MAP_SWIZZLE_128B)) ||
          (rc = make_map(&P.b[1], B16, 2, b_lo[q], k, m, ldb, 64, KSTEP, &P.b_col0[1], CU_TENSOR_MAP_SWIZZLE_128B)))
        return rc;
    } else if ((rc = make_map(&P.b[0], B16, 2, b_hi[q], m, k, ldb, KSTEP, L::BNH, &P.b_col0[0], S64)) ||
               (rc = make_map(&P.b[1], B16, 2, b_lo[q], m, k, ldb, KSTEP, L::BNH, &P.b_col0[1], S64))) {
      return rc;
    }
    P.a2 = P.a[0];  // never loaded; valid maps for prefetch.tensormap
    P.b2 = P.b[0];
    P.ndst = ndst[q];
    P.neg = 0;
    for (int d = 0; d < ndst[q]; ++d) {
      if (!c_ok(dst[4 * q + d], ldc, m)) {
        set_error("paco_mm_bf16x3_multi: C needs a 16-byte aligned start, row pitch and row length");
        return PACO_ERR_UNSUPPORTED;
      }
      if (sign[4 * q + d] < 0) P.neg |= 1u << d;
      if ((rc = make_map(d == 0 ? &P.c : &P.cx[d - 1], F32, 4, dst[4 * q + d], n, m, ldc, L::EC, 32,
                         d == 0 ? &P.c_col0 : &P.cx_col0[d - 1], S64)))
        return rc;
    }
  }
  std::lock_guard<std::mutex> pl(g_pdl_mu);
  pdl_record(device, stream, count, ndst, dst, nullptr, ldc, n, m);
  return run_pair(device, stream, maps, count, n, m, k, 0, b_natural ? 6 : 5);
}

int launch_tf32b2_split(cudaStream_t stream, int nin, const void* const* ins, const int64_t* lds,
                        const int32_t* coefs, int64_t rows, int64_t cols, int transpose, void* hi, void* h16,
                        void* l16, int64_t ldo) {
  if (nin < 1 || nin > 4) {
    set_error("paco_tf32b2_split: nin=%d (1..4 supported)", nin);
    return PACO_ERR_ARG;
  }
  if (!hi || !l16 || ldo < (transpose ? rows : cols)) {
    set_error("paco_tf32b2_split: bad outputs or pitch");
    return PACO_ERR_ARG;
  }
  tc::SplitIn in{};
  for (int q = 0; q < nin; ++q) {
    in.p[q] = static_cast<const float*>(ins[q]);
    in.ld[q] = lds[q];
    in.coef[q] = coefs[q] >= 0 ? 1 : -1;
  }
  in.nin = nin;
  return launch_split(in, rows, cols, transpose != 0, static_cast<float*>(hi), nullptr, ldo, stream,
                      static_cast<__nv_bfloat16*>(h16), static_cast<__nv_bfloat16*>(l16));
}

int launch_tf32_split(cudaStream_t stream, int nin, const void* const* ins, const int64_t* lds,
                      const int32_t* coefs, int64_t rows, int64_t cols, int transpose, void* hi, void* lo,
                      int64_t ldo) {
  if (nin < 1 || nin > 4) {
    set_error("paco_tf32_split: nin=%d (1..4 supported)", nin);
    return PACO_ERR_ARG;
  }
  if (!hi || !lo || ldo < (transpose ? rows : cols)) {
    set_error("paco_tf32_split: bad outputs or pitch");
    return PACO_ERR_ARG;
  }
  tc::SplitIn in{};
  for (int q = 0; q < nin; ++q) {
    in.p[q] = static_cast<const float*>(ins[q]);
    in.ld[q] = lds[q];
    in.coef[q] = coefs[q] >= 0 ? 1 : -1;
  }
  in.nin = nin;
  return launch_split(in, rows, cols, transpose != 0, static_cast<float*>(hi), static_cast<float*>(lo), ldo,
                      stream);
}

int tc_tile_shape(int semiring, int* bm, int* bn, int* bk, int* cps) {
  *bm = tc::BM;
  *bn = semiring == PACO_SR_BF16_F32 ? tc::KindBF16::BN : tc::KindTF32x3::BN;
  *bk = semiring == PACO_SR_BF16_F32 ? tc::KindBF16::BK : tc::KindTF32x3::BK;
  *cps = 1;
  return PACO_OK;
}

}  // namespace paco
