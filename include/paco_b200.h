/*
 * paco_b200.h -- C ABI of the B200 (sm_100a) PACO semiring-MM library.
 *
 * This is the drop-in boundary for the reference's semiring-MM hot path
 * (/root/reference/pkg/src/paco/matmul.py).  Every entry point replaces one
 * NumPy operation the reference executes per task:
 *
 *   paco_mm        <- mm_seq(A, B, C, semiring, base)            matmul.py:342-397
 *                     i.e. the COMPUTE-task body of mm_execute   matmul.py:441-454
 *                     and Semiring.block_mm(C, A, B)             matmul.py:41,45-50
 *   paco_mm_batch  <- every COMPUTE task of one device's share of a plan at once
 *                     (the runner loop of mm_execute, matmul.py:440-454)
 *   paco_fold      <- REDUCE-task body: copyto(t, vadd(t, temp)); temp.fill(zero)
 *                                                                matmul.py:455-460
 *   paco_fill      <- np.full(shape, semiring.zero)              matmul.py:430-433
 *   paco_mm_naive  <- mm_oracle(A, B, semiring) (defining sums)  matmul.py:400-414
 *   paco_plan_one_piece <- mm_one_piece_partition(n, m, k, p)    matmul.py:250-300
 *                     (cuboid geometry only)
 *   paco_plan_cta / paco_cta_grid   the CTA-level plans paco_mm runs (this
 *                     build's second PACO level: MM-1-Piece over tile units,
 *                     or the default tile grid with a k split)
 *   paco_lincomb   <- Strassen S_r/T_r formation and C-block combination
 *                     (reference has no code: SPEC.md:474-552)
 *   paco_tf32_split / paco_mm_tf32x3   the fp32 Strassen leaf level: S_r/T_r
 *                     sums as tf32 hi/lo pairs + batched 3xTF32 products
 *                     (SPEC.md:490-498 strassen_seq leaves)
 *   paco_copy2d    <- the reference's implicit NumPy host residency: staging of
 *                     host operands for mm_seq (matmul.py:342-366)
 *   paco_device_alloc / paco_ipc_* / paco_enable_peer   multi-GPU plumbing for
 *                     the parallel executor (core.py:301-326, one worker per GPU)
 *
 * Conventions: plain pointers, row-major matrices with a leading dimension in
 * ELEMENTS, int64 extents, an explicit device ordinal and cudaStream_t passed
 * as void*.  All calls are asynchronous on `stream`, re-entrant, and never
 * allocate user-visible memory.  Status: 0 = OK, negative = error; the text of
 * the last error on the calling thread is returned by paco_last_error().
 */
#ifndef PACO_B200_H_
#define PACO_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PACO_ABI_VERSION 1
#define PACO_MAX_PIECES 640

/* status codes */
#define PACO_OK 0
#define PACO_ERR_ARG (-1)         /* bad argument (maps to ValueError / PlanError) */
#define PACO_ERR_CUDA (-2)        /* CUDA runtime failure */
#define PACO_ERR_UNSUPPORTED (-3) /* layout/alignment the kernel cannot take */

/* semiring ids (element types: A, B -> C) */
#define PACO_SR_INT_I64 0         /* (+,x)  int64,int64 -> int64 (wrapping)   = SEMIRING_INT   matmul.py:53 */
#define PACO_SR_INT_I32_I64 1     /* (+,x)  int32,int32 -> int64                                        */
#define PACO_SR_F64 2             /* (+,x)  f64 -> f64                         = SEMIRING_F64   matmul.py:54 */
#define PACO_SR_MINPLUS_I64 3     /* (min,+) int64 wrapping add, zero 2^62     = SEMIRING_MINPLUS matmul.py:55 */
#define PACO_SR_MINPLUS_SAT32 4   /* (min,+) int32 storage, domain [0,2^30], INF=2^30, saturating      */
#define PACO_SR_MAXPLUS_SAT32 5   /* (max,+) int32 storage, domain [-2^30,2^30), -INF=-2^30, saturating */
#define PACO_SR_F32 6             /* (+,x)  f32 -> f32 (FFMA)                                          */
#define PACO_SR_BF16_F32 7        /* (+,x)  bf16,bf16 -> f32 (tcgen05 tensor cores)                    */
#define PACO_SR_F32_TC 8          /* (+,x)  f32 -> f32 as 3xTF32 on tcgen05 (hi/lo split, ~fp32 accuracy) */
#define PACO_SR_MINPLUS_U32 9     /* (min,+) u32 lanes, no clamp, zero 2^32-1: SEMIRING_MINPLUS on operands
                                     in [0, 2^31) (range-checked narrowing, paco_narrow_i64)            */
#define PACO_SR_COUNT 10

#define PACO_TROPICAL_INF (1 << 30)

/* paco_mm flags */
#define PACO_MM_OVERWRITE 1 /* C = A (x) B: C is not read (caller guarantees C == zero) */
#define PACO_MM_ATOMIC 2    /* fold every C element atomically (semiring (+) in L2): other
                               launches may fold into the same C concurrently (fused k-cut
                               folds of a PACO plan) */
#define PACO_MM_REMOTE 4    /* C is peer memory (NVLink): fold with element atomics, not TMA */
#define PACO_MM_PACO_PLAN 8 /* pieces == NULL: CTAs take the balanced PACO plan (paco_plan_cta over
                               148 x ctas_per_sm x 4 workers) instead of the tile grid (paco_cta_grid) */
#define PACO_MM_SYS 16      /* with PACO_MM_ATOMIC: element folds at system scope (another GPU folds into
                               the same C over NVLink); TMA bulk folds stay allowed (SIMT kernels only) */

/* dtype ids for paco_lincomb */
#define PACO_DT_F32 0
#define PACO_DT_F64 1
#define PACO_DT_I64 2

/*
 * C (+)= A (x) B on `device`/`stream`.  A is n x k (lda), B is k x m (ldb),
 * C is n x m (ldc).  `pieces` is an optional HOST array of n_pieces x 6 int32
 * (ti0, tj0, tl0, tn, tm, tk) in the units of paco_mm_tile_shape (C tiles
 * along n and m, k quanta along k): an explicit CTA-level plan, one CTA per
 * piece.  Pass NULL/0 for the default: the tile grid of paco_cta_grid (or,
 * with PACO_MM_PACO_PLAN, paco_plan_cta's balanced PACO plan).  Pieces that
 * split k fold into C with the semiring (+) in L2 (TMA bulk reduce).
 */
int paco_mm(int device, void* stream, int semiring, const void* A, int64_t lda, const void* B,
            int64_t ldb, void* C, int64_t ldc, int64_t n, int64_t m, int64_t k,
            const int32_t* pieces, int n_pieces, int flags);

/* One problem of a paco_mm_batch: C (+)= A (x) B on views (leading dimensions
 * in elements); flags as paco_mm (PACO_MM_REMOTE not allowed). */
typedef struct {
  const void* A;
  int64_t lda;
  const void* B;
  int64_t ldb;
  void* C;
  int64_t ldc;
  int64_t n, m, k;
  int32_t flags;
} paco_mm_problem;

#define PACO_MAX_BATCH 64

/* Up to PACO_MAX_BATCH independent problems of one SIMT semiring as ONE launch
 * (each gets its tile-grid CTA plan; CTA ranges are concatenated): e.g. all
 * COMPUTE cuboids of a GPU-level PACO plan on one device, their k-cut folds
 * fused (PACO_MM_ATOMIC), replacing one launch per task (matmul.py:441-454). */
int paco_mm_batch(int device, void* stream, int semiring, int count, const paco_mm_problem* problems);

/* Piece units of paco_mm's CTA plan: C tile (bm x bn), k quantum bk (piece k
 * bounds are multiples of bk elements), and resident CTAs per SM. */
int paco_mm_tile_shape(int semiring, int* bm, int* bn, int* bk, int* ctas_per_sm);

/* Cuboid geometry of mm_one_piece_partition(n, m, k, p): writes p rows of
 * (i0, j0, l0, n, m, k) into out[p*6], worker order.  Host only. */
int paco_plan_one_piece(int64_t n, int64_t m, int64_t k, int p, int64_t* out);

/* The default CTA-level plan of paco_mm for the SIMT semirings: one CTA per C
 * tile and k quantum range, the k extent split `*ksplit` ways (CTA idx ->
 * tile idx / ksplit in row-major tile order, k part idx % ksplit), `*ctas`
 * CTAs in all.  ksplit minimises ceil(tiles * s / 148) * (k / s + 64): whole
 * SM-waves of pieces, each charged a fixed per-visit cost.  Host only. */
int paco_cta_grid(int semiring, int64_t n, int64_t m, int64_t k, int* ksplit, int64_t* ctas);

/* Tail split of that tile grid (used when ksplit == 1): the tiles of the partial
 * last SM-wave -- from tile `*head` on -- are each split into `*tail` k parts
 * (CTA idx >= head: tile head + (idx - head) / tail, k part (idx - head) % tail),
 * minimising ceil(rem * t / 148) * (k / t + 64) against one wave of whole tiles.
 * *tail = 0: no tail split.  PACO_CTA_TAIL=0 disables it, > 1 forces it.  Host only. */
int paco_cta_grid_tail(int semiring, int64_t n, int64_t m, int64_t k, int* tail, int64_t* head);

/* The CTA-level plan paco_mm builds with PACO_MM_PACO_PLAN: MM-1-Piece over the
 * (bm, bn, bk) unit grid of `semiring` for p workers, with nearest-unit cuts
 * and a fall-back to the finest axis when a cut would miss the p-ratio by
 * > 1%.  Writes p rows of (ti0, tj0, tl0, tn, tm, tk) into out[p*6]. Host only. */
int paco_plan_cta(int semiring, int64_t n, int64_t m, int64_t k, int p, int32_t* out);

/* dst (+)= src elementwise (n x m views).  flags: PACO_FOLD_RESET -- src = semiring
 * zero afterwards (the REDUCE body); PACO_FOLD_ATOMIC -- one global atomic (+) per
 * element, so other kernels may fold into dst concurrently (fused k-cut folds). */
#define PACO_FOLD_RESET 1
#define PACO_FOLD_ATOMIC 2
int paco_fold(int device, void* stream, int semiring, void* dst, int64_t ld_dst, void* src,
              int64_t ld_src, int64_t n, int64_t m, int flags);

/* dst = semiring zero (the value the reference fills temporaries with). */
int paco_fill(int device, void* stream, int semiring, void* dst, int64_t ld, int64_t n, int64_t m);

/* Device ground truth: C = C (+) (defining sum over l), one thread per element. */
int paco_mm_naive(int device, void* stream, int semiring, const void* A, int64_t lda,
                  const void* B, int64_t ldb, void* C, int64_t ldc, int64_t n, int64_t m,
                  int64_t k);

/* out (= or +=) sum_i coef[i] * in[i] over n x m views (coef in {-1, +1}). */
int paco_lincomb(int device, void* stream, int dtype, void* out, int64_t ld_out, int64_t n,
                 int64_t m, int nin, const void* const* ins, const int64_t* lds,
                 const int32_t* coefs, int accumulate);

/* nout (<= 8) fp32 sums of the same nin (<= 4) n x m inputs in one pass:
 * outs[o] = sum_i coefs[o * nin + i] * ins[i] (coefs in {-1, 0, +1}) -- Strassen's
 * formation of a node (S1, S2, S5, S6, S7 from A's four quadrants) reads every
 * input once.  16-byte aligned views, m % 4 == 0. */
int paco_lincomb_multi(int device, void* stream, int64_t n, int64_t m, int nin, const void* const* ins,
                       const int64_t* lds, int nout, void* const* outs, const int64_t* ldo, const int32_t* coefs);

/* Strassen leaf operands for the 3xTF32 tensor-core MM, with the S/T sum
 * fused in (replaces a lincomb + split pair): x = sum_i
 * coef[i] * in[i] over rows x cols fp32 views (nin 1..4, coef +1/-1) is
 * written as hi = tf32_rn(x), lo = tf32_rn(x - hi), row pitch ldo elements,
 * transposed (cols x rows) when `transpose` (the K-major B^T operand). */
int paco_tf32_split(int device, void* stream, int nin, const void* const* ins, const int64_t* lds,
                    const int32_t* coefs, int64_t rows, int64_t cols, int transpose, void* hi, void* lo,
                    int64_t ldo);

/* C[q] (+)= A[q] x B[q], q < count (1..8), as 3xTF32 on tcgen05 from pre-split
 * operands -- one launch whose tiles of all `count` same-shape products share
 * one dynamic queue (Strassen's seven leaf products of a node).  A_hi/A_lo
 * n x k (lda), B^T_hi/B^T_lo m x k (ldb) -- paco_tf32_split outputs; C n x m
 * (ldc); row pitches must be multiples of 16 bytes.  flags as paco_mm. */
int paco_mm_tf32x3(int device, void* stream, int count, const void* const* a_hi, const void* const* a_lo,
                   int64_t lda, const void* const* bt_hi, const void* const* bt_lo, int64_t ldb, void* const* C,
                   int64_t ldc, int64_t n, int64_t m, int64_t k, int flags);

/* As paco_mm_tf32x3, but product q is folded into each of its ndst[q] (1..4)
 * destinations dst[4q + d] with sign sign[4q + d] (+1: C += AB, -1: C -= AB) by
 * the epilogue's TMA reduce-adds -- the Strassen C-block combination
 * (C00 = M1 + M4 - M5 + M7, ...) composed over the levels
 * above the leaves, with no M buffers and no combination pass.  Destinations
 * share ldc; they must hold their initial values (e.g. zero). */
int paco_mm_tf32x3_multi(int device, void* stream, int count, const void* const* a_hi, const void* const* a_lo,
                         int64_t lda, const void* const* bt_hi, const void* const* bt_lo, int64_t ldb,
                         const int32_t* ndst, void* const* dst, const int32_t* sign, int64_t ldc, int64_t n,
                         int64_t m, int64_t k);

/* Range-checked narrowing of an int64 view to 32-bit words -- the fast path
 * for the reference's own int64 semirings (SEMIRING_MINPLUS, SEMIRING_INT,
 * matmul.py:45-55) when their operands fit 32 bits: dst = (uint32)src for
 * lo <= src <= hi.  A value below lo, or above hi without `saturate`, sets
 * *flag (device int32, caller-zeroed) to 1 and the caller must take the int64
 * kernel instead; with `saturate` values above hi are stored as hi. */
int paco_narrow_i64(int device, void* stream, const int64_t* src, int64_t ld_src, void* dst32, int64_t ld_dst,
                    int64_t rows, int64_t cols, int64_t lo, int64_t hi, int saturate, int32_t* flag);

/* Widen a PACO_SR_MINPLUS_U32 result into the int64 C it was narrowed from:
 * c = (r == 2^32 - 1) ? c : r  (r == 2^32 - 1 only where no term reached C's
 * saturated image, i.e. C's original int64 value stands). */
int paco_widen_u32_i64(int device, void* stream, const void* r32, int64_t ld_r, int64_t* c, int64_t ld_c,
                       int64_t rows, int64_t cols);

/* Narrowing of a SEMIRING_MINPLUS operand (int64, zero INF = 2^62,
 * matmul.py:29,55) for the u32 kernel with the INF sentinel kept exact:
 * x in [0, 2^30 - 2] -> x + 1, x == 2^62 -> 2^31; any other value sets *flag.
 * On the kernel's wrapping u32 adds a term is then a + b + 2 < 2^31 (both
 * finite), 2^31 + f + 1 (one INF: the reference's 2^62 + f) or 0 (both INF:
 * the reference's int64 wrap of 2^63 to -2^63), an order-preserving code that
 * paco_widen_minplus_i64 decodes.  Replaces the reference's int64 inner loop
 * (matmul.py:49-50) when the operands hold INF. */
int paco_narrow_minplus_inf(int device, void* stream, const int64_t* src, int64_t ld_src, void* dst32,
                            int64_t ld_dst, int64_t rows, int64_t cols, int32_t* flag);

/* c = min(c, decode(r)) in int64 for a PACO_SR_MINPLUS_U32 product r computed
 * from the semiring zero (r == 2^32 - 1: no term): with inf_encoded the
 * paco_narrow_minplus_inf code (0 -> -2^63, r < 2^31 -> r - 2, else
 * 2^62 + r - 2^31 - 1), else r itself. */
int paco_widen_minplus_i64(int device, void* stream, const void* r32, int64_t ld_r, int64_t* c, int64_t ld_c,
                           int64_t rows, int64_t cols, int inf_encoded);

/* Strassen's leaf level with the operand formation fused into the 3xTF32
 * kernel: problem q (< count <= 8) multiplies
 * A_q = sum_{t < nta[q]} a_sign[2q+t] * a_terms[2q+t]   (n x k, pitch lda)
 * by B_q, passed transposed as
 * B_q^T = sum_{t < ntb[q]} b_sign[2q+t] * bt_terms[2q+t] (m x k, pitch ldb),
 * with nta, ntb in 1..2 and signs +1/-1 -- i.e. the leaf's S_r of A and T_r^T
 * of B^T as quadrant views -- and folds the product into its ndst[q] (1..4)
 * destinations with sign[4q+d] (as paco_mm_tf32x3_multi).  The sums and the
 * tf32 hi/lo split happen in shared memory inside the GEMM: no split launches,
 * no hi/lo round trip through HBM.  Views: 16-byte aligned starts and pitches. */
int paco_mm_tf32x3_fused(int device, void* stream, int count, const int32_t* nta, const void* const* a_terms,
                         const int32_t* a_sign, int64_t lda, const int32_t* ntb, const void* const* bt_terms,
                         const int32_t* b_sign, int64_t ldb, const int32_t* ndst, void* const* dst,
                         const int32_t* sign, int64_t ldc, int64_t n, int64_t m, int64_t k);

/* The leaf level on CTA pairs with only the A side formed in the kernel: A_q =
 * sum_{t < nta[q] <= 2} a_sign * a_terms[2q+t] (n x k, pitch lda) is TMA'd raw and
 * split into tf32 hi/lo in shared memory; B_q^T comes pre-split (bt_hi / bt_lo,
 * m x k, pitch ldb, from paco_tf32_split); destinations as _multi.  The A-side
 * split launches disappear while each SM's shared-memory traffic stays under
 * its bandwidth (the pair halves the B bytes per SM). */
int paco_mm_tf32x3_fused_a(int device, void* stream, int count, const int32_t* nta, const void* const* a_terms,
                           const int32_t* a_sign, int64_t lda, const void* const* bt_hi, const void* const* bt_lo,
                           int64_t ldb, const int32_t* ndst, void* const* dst, const int32_t* sign, int64_t ldc,
                           int64_t n, int64_t m, int64_t k);

/* The tf32 + 2 x bf16 format of an fp32 operand (the Strassen leaves' default on
 * CTA pairs): x = sum_i coef[i] * in[i] (as paco_tf32_split) is written as
 * hi = tf32_rn(x) (fp32), h16 = bf16_rn(hi), l16 = bf16_rn(x - hi) (bf16 arrays),
 * all with row pitch ldo elements, transposed when `transpose` (h16 may be NULL). */
int paco_tf32b2_split(int device, void* stream, int nin, const void* const* ins, const int64_t* lds,
                      const int32_t* coefs, int64_t rows, int64_t cols, int transpose, void* hi, void* h16, void* l16,
                      int64_t ldo);

/* C (+/-)= A x B for fp32 operands given in that format: the main product
 * hi * hi on the tf32 tensor path and the corrections hi * lo + lo * hi as bf16
 * products (kind::f16: half the tensor time of tf32), fp32 accumulation in TMEM,
 * on CTA pairs (cta_group::2).  The corrections are 2^-11 of the product, so their
 * bf16 rounding adds ~2^-19 relative per term -- below the fp32 accumulation and
 * Strassen formation errors of cfg5 (tests/test_gpu_tf32_fused.py).  A n x k (lda),
 * B^T m x k (ldb), destinations as paco_mm_tf32x3_multi.  a_h16 = b_h16 = NULL:
 * the kernel forms bf16(hi) from the hi tiles itself (6 instead of 8 bytes of
 * operand traffic per element; paco_tf32b2_split then takes h16 = NULL too).  All
 * four bf16 arrays NULL: a_hi / b_hi are plain fp32 operands (no split pass at
 * all); the tf32 MMA reads x (hi = its top 19 bits) and the kernel forms bf16(hi)
 * and bf16(x - hi) -- 4 bytes per element. */
int paco_mm_tf32b2_multi(int device, void* stream, int count, const void* const* a_hi, const void* const* a_h16,
                         const void* const* a_l16, int64_t lda, const void* const* b_hi, const void* const* b_h16,
                         const void* const* b_l16, int64_t ldb, const int32_t* ndst, void* const* dst,
                         const int32_t* sign, int64_t ldc, int64_t n, int64_t m, int64_t k);

/* Strassen leaf operands in the bf16x3 format: like paco_lincomb_multi (but up
 * to 8 inputs: a leaf node's operands straight from the level-0 blocks), and
 * output o is written as two bf16 planes his[o] = bf16_rn(x), los[o] =
 * bf16_rn(x - his[o]) (pitch ldo[o] elements, shared by both planes); a
 * one-term row is a split copy.  16-byte aligned views, m % 8 == 0. */
int paco_lincomb_split(int device, void* stream, int64_t n, int64_t m, int nin, const void* const* ins,
                       const int64_t* lds, int nout, void* const* his, void* const* los, const int64_t* ldo,
                       const int32_t* coefs);

/* All 49 leaf operands of one side of a 2-level Strassen in one pass: x is the
 * 4h x 4h operand (A: side 0, S formulas; B in its own layout: side 1, T
 * formulas), leaf (r, r') (r, r' = 1..7, output index 7 (r - 1) + r' - 1) is the
 * signed sum of x's 4 x 4 blocks of size h given by formula r over the
 * quadrants and r' over their sub-quadrants, written as
 * bf16 hi / lo planes (pitch ldo).  Every element of x is read once. */
int paco_strassen_split49(int device, void* stream, int side, const void* x, int64_t ldx, int64_t h,
                          void* const* his, void* const* los, int64_t ldo);

/* bf16x3 batch on tcgen05 CTA pairs -- cfg5's Strassen leaf products: C[q] (+/-)=
 * A[q] B[q] with A[q] = a_hi[q] + a_lo[q] (bf16 planes, n x k, pitch lda) and
 * B[q]^T = b_hi[q] + b_lo[q] (m x k, pitch ldb), computed as hi*hi + hi*lo +
 * lo*hi on kind::f16 with fp32 accumulation; destinations and signs as
 * paco_mm_tf32x3_multi (up to 4 per problem, count <= 8). */
int paco_mm_bf16x3_multi(int device, void* stream, int count, const void* const* a_hi, const void* const* a_lo,
                         int64_t lda, const void* const* b_hi, const void* const* b_lo, int64_t ldb,
                         const int32_t* ndst, void* const* dst, const int32_t* sign, int64_t ldc, int64_t n,
                         int64_t m, int64_t k);

/* The same batch with B[q] given in its own k x m layout (b_hi[q] + b_lo[q], pitch
 * ldb; MN-major operand tiles): Strassen's T_r planes formed from B's quadrants
 * with no transpose pass.  16-byte aligned planes and row pitches. */
int paco_mm_bf16x3_multi_bn(int device, void* stream, int count, const void* const* a_hi, const void* const* a_lo,
                            int64_t lda, const void* const* b_hi, const void* const* b_lo, int64_t ldb,
                            const int32_t* ndst, void* const* dst, const int32_t* sign, int64_t ldc, int64_t n,
                            int64_t m, int64_t k);

/* dst (cols x rows, pitch ld_dst) = src^T (rows x cols, pitch ld_src); 4- or
 * 8-byte elements.  Strassen transposes B once so every T_r^T operand of the
 * fused leaves is a K-major view. */
int paco_transpose(int device, void* stream, int elsize, void* dst, int64_t ld_dst, const void* src, int64_t ld_src,
                   int64_t rows, int64_t cols);

/* Asynchronous 2-D copy (host<->device or device<->device; pitches and width in
 * BYTES): the staging primitive of the overlapped host pipeline. */
int paco_copy2d(int device, void* stream, void* dst, int64_t dpitch, const void* src, int64_t spitch,
                int64_t width, int64_t rows);

/* Parallel host memcpy (pitches and width in BYTES) between pageable and pinned
 * host memory, `threads` participants (a persistent pool + the caller): the
 * staging step that feeds paco_copy2d from the reference's pageable NumPy
 * operands (matmul.py:342-366).  Synchronous; call without holding locks the
 * pool could need.  */
int paco_host_copy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width, int64_t rows,
                     int threads);

/* Page-lock (and later release) a caller's host buffer so paco_copy2d can DMA
 * straight from it: the NumPy operands of repeated mm_seq / mm_execute calls are
 * registered once (first call) instead of staged every call. */
int paco_host_register(void* ptr, size_t bytes);
int paco_host_unregister(void* ptr);

/* Device memory for buffers shared across processes (CUDA IPC) -- the only
 * allocation the library makes on a caller's behalf. */
int paco_device_alloc(int device, size_t bytes, void** ptr);
int paco_device_free(int device, void* ptr);
/* CUDA IPC: export a paco_device_alloc'd pointer (64-byte handle), map a peer's. */
int paco_ipc_handle(int device, void* ptr, void* handle64);
int paco_ipc_open(int device, const void* handle64, void** ptr);
int paco_ipc_close(int device, void* ptr);

/* Enable peer access from `device` to `peer` (idempotent). */
int paco_enable_peer(int device, int peer);

/* ALU issue-rate probe: runs `which` (0 = VIADDMNMX.U32 min-plus, 1 = VIADDMNMX.S32
 * max-plus, 2 = FFMA, 3 = DFMA) on every SM and returns the
 * measured terms per clock per SM and the SM clock (MHz) seen during the run. */
int paco_alu_probe(int device, void* stream, int which, int iters, double* terms_per_clk_sm,
                   double* sm_mhz);

/* Live kernel timing.  paco_kernel_timing(1) clears the record and starts
 * bracketing every launch of the library with a CUDA event pair on its
 * stream (0 stops); paco_kernel_timing_read synchronises the recorded events
 * of one kernel family and returns their summed duration and launch count.
 * Families: */
#define PACO_KT_SIMT_MM 0     /* simt_mm_kernel / simt_mm_batch_kernel (tropical, integer, fp32, fp64) */
#define PACO_KT_TC_GEMM 1     /* tc_gemm_kernel (tcgen05: bf16, 3xTF32) */
#define PACO_KT_TF32_SPLIT 2  /* split_tf32_{n,t}_kernel (Strassen leaf operands) */
#define PACO_KT_LINCOMB 3     /* lincomb_kernel (Strassen S/T/C sums) */
#define PACO_KT_ELEMENTWISE 4 /* fold / fill / narrow / widen */
#define PACO_KT_COUNT 5
int paco_kernel_timing(int enable);
int paco_kernel_timing_read(int family, double* ms_total, int64_t* launches);

/* Diagnostics: while `device_buffer` (>= 10 x grid int64) is set, each
 * SIMT paco_mm CTA writes (smid, start ns, end ns, stage count, its piece
 * ti0,tj0,tl0,tn,tm,tk) -- 10 int64 per CTA.  NULL disables. */
int paco_debug_trace(void* device_buffer);

const char* paco_last_error(void);
int paco_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PACO_B200_H_ */
