/*
 * CPU ORACLE -- test infrastructure only.  Nothing in the product path
 * (paper_2011_01441_b200/) links, loads or calls this file; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg do, as a checker.
 *
 * Plain-C restatement of the reference's defining sums for semiring MM,
 * /root/reference/pkg/src/paco/matmul.py:
 *   mm_oracle (400-414): acc = semiring zero; for l: acc = acc (+) a[i,l] (x) b[l,j];
 *                        C[i,j] = C[i,j] (+) acc   ((+) = vadd for min-plus, 413)
 *   _int_block (45-46) / _minplus_block (49-50): the same sums, blocked.
 * Semiring ids match include/paco_b200.h.  The (min,+) saturating and (max,+)
 * variants are the reference min-plus on the documented 32-bit domains:
 * minplus_sat(C, A, B) == min(C, 2^30) of SEMIRING_MINPLUS on int64 copies,
 * maxplus(A, B) == -minplus(-A, -B); tests/test_oracle.py
 * pins both against golden vectors produced by the reference itself.
 *
 * Loop order is (row block, column block) -> l -> row -> j over an accumulator
 * block, so gcc vectorises the j loop; blocks are split across OpenMP threads (rows are independent, so the
 * result is bit-identical to the serial sum for the integer semirings).
 *
 * The two 32-bit tropical semirings (the full-size cfg2 / cfg4 whole-C checks,
 * 5.5e11 and 4.4e12 terms) take a cache-blocked path instead: packed A / B
 * blocks and a 6 x 16 register tile per l step (the textbook GEMM loop nest).
 * (min, max) are associative and commutative, so any term order gives the
 * same bits; oracle_mm_rows_simple keeps the plain loop above for every id and
 * tests/test_oracle.py checks the two against each other and the goldens.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum {
  SR_INT_I64 = 0, SR_INT_I32_I64 = 1, SR_F64 = 2, SR_MINPLUS_I64 = 3,
  SR_MINPLUS_SAT32 = 4, SR_MAXPLUS_SAT32 = 5, SR_F32 = 6
};

#define INF32 (1 << 30)

#define RB 16   /* rows per block: B is streamed once per row block */
#define JB 512   /* columns per block: the accumulator block stays in L1/L2 */

#define ROW_LOOP(ACC_T, INIT, A_T, B_T, C_T, TERM, FOLD)                                  \
  {                                                                                       \
    const int64_t nrb = (r1 - r0 + RB - 1) / RB, njb = (m + JB - 1) / JB;                 \
    _Pragma("omp parallel for schedule(dynamic, 1)")                                     \
    for (int64_t t = 0; t < nrb * njb; ++t) {                                             \
      const int64_t i0 = r0 + (t / njb) * RB, j0 = (t % njb) * JB;                        \
      const int64_t rn = (r1 - i0) < RB ? (r1 - i0) : RB;                                 \
      const int64_t jn = (m - j0) < JB ? (m - j0) : JB;                                   \
      ACC_T accb[RB][JB];                                                                 \
      for (int64_t r = 0; r < rn; ++r)                                                    \
        for (int64_t j = 0; j < jn; ++j) accb[r][j] = (INIT);                             \
      for (int64_t l = 0; l < k; ++l) {                                                   \
        const B_T* brow = (const B_T*)B + l * ldb + j0;                                   \
        for (int64_t r = 0; r < rn; ++r) {                                                \
          const A_T a = ((const A_T*)A)[(i0 + r) * lda + l];                              \
          ACC_T* acc = accb[r];                                                           \
          for (int64_t j = 0; j < jn; ++j) { const B_T b = brow[j]; TERM; }               \
        }                                                                                 \
      }                                                                                   \
      for (int64_t r = 0; r < rn; ++r) {                                                  \
        C_T* crow = (C_T*)C + (i0 + r) * ldc + j0;                                        \
        const ACC_T* acc = accb[r];                                                       \
        for (int64_t j = 0; j < jn; ++j) { FOLD; }                                        \
      }                                                                                   \
    }                                                                                     \
  }

/* C (+)= A (x) B over rows [r0, r1) with the plain loop.  0, or -1 for an unknown id. */
int oracle_mm_rows_simple(int sr, const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                   int64_t ldc, int64_t n, int64_t m, int64_t k, int64_t r0, int64_t r1) {
  if (r0 < 0) r0 = 0;
  if (r1 > n) r1 = n;
  switch (sr) {
    case SR_INT_I64:  /* int64 ring, two's-complement wrap like NumPy */
      ROW_LOOP(uint64_t, 0, int64_t, int64_t, int64_t,
               acc[j] += (uint64_t)a * (uint64_t)b,
               crow[j] = (int64_t)((uint64_t)crow[j] + acc[j]))
      return 0;
    case SR_INT_I32_I64:
      ROW_LOOP(int64_t, 0, int32_t, int32_t, int64_t,
               acc[j] += (int64_t)a * (int64_t)b,
               crow[j] = (int64_t)((uint64_t)crow[j] + (uint64_t)acc[j]))
      return 0;
    case SR_F64:
      ROW_LOOP(double, 0.0, double, double, double, acc[j] += a * b, crow[j] += acc[j])
      return 0;
    case SR_F32:
      ROW_LOOP(double, 0.0, float, float, float, acc[j] += (double)a * (double)b,
               crow[j] = (float)((double)crow[j] + acc[j]))
      return 0;
    case SR_MINPLUS_I64:  /* matmul.py:49-50 with its wrapping int64 add */
      ROW_LOOP(int64_t, INT64_MAX, int64_t, int64_t, int64_t,
               { const int64_t s = (int64_t)((uint64_t)a + (uint64_t)b); acc[j] = s < acc[j] ? s : acc[j]; },
               crow[j] = acc[j] < crow[j] ? acc[j] : crow[j])
      return 0;
    case SR_MINPLUS_SAT32:  /* inputs in [0, 2^30]: sums <= 2^31 fit u32; clamp at INF */
      ROW_LOOP(uint32_t, 0xFFFFFFFFu, int32_t, int32_t, int32_t,
               { const uint32_t s = (uint32_t)a + (uint32_t)b; acc[j] = s < acc[j] ? s : acc[j]; },
               { uint32_t v = acc[j] < (uint32_t)INF32 ? acc[j] : (uint32_t)INF32;
                 crow[j] = (int32_t)v < crow[j] ? (int32_t)v : crow[j]; })
      return 0;
    case SR_MAXPLUS_SAT32:  /* inputs in [-2^30, 2^30): sums fit s32; clamp at -INF */
      ROW_LOOP(int32_t, INT32_MIN, int32_t, int32_t, int32_t,
               { const int32_t s = a + b; acc[j] = s > acc[j] ? s : acc[j]; },
               { int32_t v = acc[j] > -INF32 ? acc[j] : -INF32;
                 crow[j] = v > crow[j] ? v : crow[j]; })
      return 0;
    default:
      return -1;
  }
}


/* ---- cache-blocked 32-bit tropical path -------------------------------- */
#define MR 6
#define NR 16
#define KC 256
#define NCB 512
#define MCB 96

/* kind 0: (min,+) saturating on u32 lanes; kind 1: (max,+) on s32 lanes */
#define TROP_MICRO(NAME, T, OPEXPR)                                                      \
  static void NAME(const T* ap, const T* bp, T* acc, int64_t ldacc, int64_t kc) {          \
    T c[MR][NR];                                                                         \
    for (int r = 0; r < MR; ++r)                                                         \
      for (int j = 0; j < NR; ++j) c[r][j] = acc[r * ldacc + j];                         \
    for (int64_t l = 0; l < kc; ++l) {                                                   \
      const T* b = bp + l * NCB;                                                         \
      for (int r = 0; r < MR; ++r) {                                                     \
        const T a = ap[r * KC + l];                                                      \
        for (int j = 0; j < NR; ++j) { const T s = (T)(a + b[j]); c[r][j] = OPEXPR; }    \
      }                                                                                  \
    }                                                                                    \
    for (int r = 0; r < MR; ++r)                                                         \
      for (int j = 0; j < NR; ++j) acc[r * ldacc + j] = c[r][j];                         \
  }
TROP_MICRO(micro_minplus, uint32_t, (s < c[r][j] ? s : c[r][j]))
TROP_MICRO(micro_maxplus, int32_t, (s > c[r][j] ? s : c[r][j]))

static void trop32_blocked(int kind, const int32_t* A, int64_t lda, const int32_t* B, int64_t ldb, int32_t* C,
                           int64_t ldc, int64_t m, int64_t k, int64_t r0, int64_t r1) {
  const int64_t nmb = (r1 - r0 + MCB - 1) / MCB, njb = (m + NCB - 1) / NCB;
  _Pragma("omp parallel")
  {
    int32_t* ap = (int32_t*)aligned_alloc(64, sizeof(int32_t) * MCB * KC);
    int32_t* bp = (int32_t*)aligned_alloc(64, sizeof(int32_t) * KC * NCB);
    int32_t* acc = (int32_t*)aligned_alloc(64, sizeof(int32_t) * MCB * NCB);
    _Pragma("omp for schedule(dynamic, 1)")
    for (int64_t t = 0; t < nmb * njb; ++t) {
      const int64_t i0 = r0 + (t / njb) * MCB, j0 = (t % njb) * NCB;
      const int64_t rn = (r1 - i0) < MCB ? (r1 - i0) : MCB;
      const int64_t jn = (m - j0) < NCB ? (m - j0) : NCB;
      const int32_t init = kind == 0 ? (int32_t)0xFFFFFFFFu : INT32_MIN;
      for (int64_t e = 0; e < MCB * NCB; ++e) acc[e] = init;
      for (int64_t l0 = 0; l0 < k; l0 += KC) {
        const int64_t kc = (k - l0) < KC ? (k - l0) : KC;
        for (int64_t r = 0; r < MCB; ++r)  /* pack A (rows past rn: 0, results discarded) */
          for (int64_t l = 0; l < kc; ++l) ap[r * KC + l] = r < rn ? A[(i0 + r) * lda + l0 + l] : 0;
        for (int64_t l = 0; l < kc; ++l) { /* pack B (columns past jn: 0, discarded) */
          const int32_t* brow = B + (l0 + l) * ldb + j0;
          for (int64_t j = 0; j < NCB; ++j) bp[l * NCB + j] = j < jn ? brow[j] : 0;
        }
        for (int64_t ir = 0; ir < rn; ir += MR)
          for (int64_t jr = 0; jr < jn; jr += NR) {
            if (kind == 0)
              micro_minplus((const uint32_t*)ap + ir * KC, (const uint32_t*)bp + jr, (uint32_t*)acc + ir * NCB + jr,
                            NCB, kc);
            else
              micro_maxplus(ap + ir * KC, bp + jr, acc + ir * NCB + jr, NCB, kc);
          }
      }
      for (int64_t r = 0; r < rn; ++r) {
        int32_t* crow = C + (i0 + r) * ldc + j0;
        const int32_t* arow = acc + r * NCB;
        for (int64_t j = 0; j < jn; ++j) {
          if (kind == 0) {
            const uint32_t a = (uint32_t)arow[j];
            const int32_t v = (int32_t)(a < (uint32_t)INF32 ? a : (uint32_t)INF32);
            crow[j] = v < crow[j] ? v : crow[j];
          } else {
            const int32_t v = arow[j] > -INF32 ? arow[j] : -INF32;
            crow[j] = v > crow[j] ? v : crow[j];
          }
        }
      }
    }
    free(ap);
    free(bp);
    free(acc);
  }
}

/* C (+)= A (x) B over rows [r0, r1).  Returns 0, or -1 for an unknown id. */
int oracle_mm_rows(int sr, const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                   int64_t n, int64_t m, int64_t k, int64_t r0, int64_t r1) {
  if (r0 < 0) r0 = 0;
  if (r1 > n) r1 = n;
  if ((sr == SR_MINPLUS_SAT32 || sr == SR_MAXPLUS_SAT32) && k > 0 && r1 > r0 && m > 0) {
    trop32_blocked(sr == SR_MINPLUS_SAT32 ? 0 : 1, (const int32_t*)A, lda, (const int32_t*)B, ldb, (int32_t*)C, ldc,
                   m, k, r0, r1);
    return 0;
  }
  return oracle_mm_rows_simple(sr, A, lda, B, ldb, C, ldc, n, m, k, r0, r1);
}
