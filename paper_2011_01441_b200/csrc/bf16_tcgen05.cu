// placeholder until the tcgen05 kernel lands
#include "common.cuh"
namespace paco {
int launch_mm_bf16_tc(int, cudaStream_t, const void*, int64_t, const void*, int64_t, void*, int64_t,
                      int64_t, int64_t, int64_t, const int32_t*, int, int) {
  set_error("bf16 tcgen05 kernel not built yet");
  return PACO_ERR_UNSUPPORTED;
}
int bf16_tile_shape(int* bm, int* bn, int* bk, int* cps) {
  *bm = 128; *bn = 256; *bk = 64; *cps = 1;
  return PACO_OK;
}
}  // namespace paco
