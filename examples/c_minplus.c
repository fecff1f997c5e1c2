/* A plain-C caller of the drop-in boundary (include/paco_b200.h): no CUDA
 * headers, no torch.  Allocates device buffers through the library, copies a
 * seeded (min,+) problem in, runs paco_mm with the default CTA plan and with a
 * 5-way GPU-level MM-1-Piece split folded through paco_fold, copies C back and
 * checks every element against the defining sums.  Exit code 0 = all equal. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "paco_b200.h"

#define INF PACO_TROPICAL_INF
#define CHECK(x)                                                  \
  do {                                                            \
    if ((x) != PACO_OK) {                                         \
      fprintf(stderr, "%s failed: %s\n", #x, paco_last_error());  \
      return 1;                                                   \
    }                                                             \
  } while (0)

static uint64_t rng = 88172645463325252ull;
static uint32_t next_u32(void) {
  rng ^= rng << 13;
  rng ^= rng >> 7;
  rng ^= rng << 17;
  return (uint32_t)rng;
}

int main(void) {
  const int64_t n = 300, m = 260, k = 515;
  int32_t *A = malloc(n * k * 4), *B = malloc(k * m * 4), *C = malloc(n * m * 4);
  for (int64_t i = 0; i < n * k; ++i) A[i] = (next_u32() % 10 == 0) ? INF : (int32_t)(next_u32() % (1u << 20));
  for (int64_t i = 0; i < k * m; ++i) B[i] = (next_u32() % 10 == 0) ? INF : (int32_t)(next_u32() % (1u << 20));
  void *dA, *dB, *dC, *dT;
  CHECK(paco_device_alloc(0, n * k * 4, &dA));
  CHECK(paco_device_alloc(0, k * m * 4, &dB));
  CHECK(paco_device_alloc(0, n * m * 4, &dC));
  CHECK(paco_device_alloc(0, n * m * 4, &dT));
  CHECK(paco_copy2d(0, NULL, dA, k * 4, A, k * 4, k * 4, n));
  CHECK(paco_copy2d(0, NULL, dB, m * 4, B, m * 4, m * 4, k));
  int bad = 0;
  for (int variant = 0; variant < 2; ++variant) {
    CHECK(paco_fill(0, NULL, PACO_SR_MINPLUS_SAT32, dC, m, n, m));
    if (variant == 0) {  /* one launch, default CTA-level plan */
      CHECK(paco_mm(0, NULL, PACO_SR_MINPLUS_SAT32, dA, k, dB, m, dC, m, n, m, k, NULL, 0, 0));
    } else {  /* GPU-level MM-1-Piece over 5 workers; k-cut pieces go to a temp + paco_fold */
      int64_t cub[5 * 6];
      CHECK(paco_plan_one_piece(n, m, k, 5, cub));
      for (int w = 0; w < 5; ++w) {
        const int64_t *c = cub + 6 * w; /* i0, j0, l0, n, m, k */
        const char *a = (const char *)dA + 4 * (c[0] * k + c[2]);
        const char *b = (const char *)dB + 4 * (c[2] * m + c[1]);
        char *out = (char *)(c[2] == 0 ? dC : dT) + 4 * (c[0] * m + c[1]);
        if (c[2] != 0) CHECK(paco_fill(0, NULL, PACO_SR_MINPLUS_SAT32, out, m, c[3], c[4]));
        CHECK(paco_mm(0, NULL, PACO_SR_MINPLUS_SAT32, a, k, b, m, out, m, c[3], c[4], c[5], NULL, 0, 0));
        if (c[2] != 0) /* REDUCE: C block (+)= temp block */
          CHECK(paco_fold(0, NULL, PACO_SR_MINPLUS_SAT32, (char *)dC + 4 * (c[0] * m + c[1]), m, out, m, c[3],
                          c[4], 1));
      }
    }
    CHECK(paco_copy2d(0, NULL, C, m * 4, dC, m * 4, m * 4, n)); /* synchronous on the NULL stream */
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < m; ++j) {
        int64_t best = INF;
        for (int64_t l = 0; l < k; ++l) {
          const int64_t s = (int64_t)A[i * k + l] + B[l * m + j];
          if (s < best) best = s;
        }
        if (C[i * m + j] != (int32_t)(best < INF ? best : INF)) ++bad;
      }
    printf("variant %d: %s\n", variant, bad ? "MISMATCH" : "ok");
  }
  paco_device_free(0, dA);
  paco_device_free(0, dB);
  paco_device_free(0, dC);
  paco_device_free(0, dT);
  free(A);
  free(B);
  free(C);
  return bad != 0;
}
