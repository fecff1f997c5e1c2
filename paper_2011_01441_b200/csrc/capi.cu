// extern "C" boundary of libpaco_b200.so (declared in include/paco_b200.h).
// Validates arguments, selects the device, maps semirings to kernels and
// reports errors through return codes + a thread-local message.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include <cuda.h>

#include "common.cuh"

namespace paco {

static thread_local char g_err[512] = "";

std::atomic<int> g_ktime_on{0};

namespace {
struct KRec {
  cudaEvent_t a = nullptr, b = nullptr;
  int fam = 0;
  int dev = 0;
};
std::mutex g_kt_mu;
std::vector<KRec> g_kt_recs;
thread_local std::vector<size_t> t_kt_open;  // records opened by this thread, innermost last
}  // namespace

void ktime_record(int family, cudaStream_t st, bool start) {
  if (start) {
    KRec r;
    r.fam = family;
    cudaGetDevice(&r.dev);
    if (cudaEventCreate(&r.a) != cudaSuccess || cudaEventCreate(&r.b) != cudaSuccess) return;
    cudaEventRecord(r.a, st);
    std::lock_guard<std::mutex> lock(g_kt_mu);
    g_kt_recs.push_back(r);
    t_kt_open.push_back(g_kt_recs.size() - 1);
  } else {
    if (t_kt_open.empty()) return;
    std::lock_guard<std::mutex> lock(g_kt_mu);
    const size_t idx = t_kt_open.back();
    t_kt_open.pop_back();
    if (idx < g_kt_recs.size()) cudaEventRecord(g_kt_recs[idx].b, st);
  }
}

const char* dev_knob(const char* name) {
  static const bool on = [] {
    const char* e = getenv("PACO_DEV_KNOBS");
    return e && e[0] == '1';
  }();
  return on ? getenv(name) : nullptr;
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// defined in the kernel translation units
int launch_mm_simt(int sr, int device, cudaStream_t stream, const void* A, int64_t lda, const void* B,
                   int64_t ldb, void* C, int64_t ldc, int64_t n, int64_t m, int64_t k,
                   const int32_t* pieces, int n_pieces, int flags);
int simt_tile_shape(int sr, int* bm, int* bn, int* bk, int* cps);
int launch_mm_bf16_tc(int device, cudaStream_t stream, const void* A, int64_t lda, const void* B,
                      int64_t ldb, void* C, int64_t ldc, int64_t n, int64_t m, int64_t k,
                      const int32_t* pieces, int n_pieces, int flags);
int launch_mm_f32_tc(int device, cudaStream_t stream, const void* A, int64_t lda, const void* B,
                     int64_t ldb, void* C, int64_t ldc, int64_t n, int64_t m, int64_t k,
                     const int32_t* pieces, int n_pieces, int flags);
int tc_tile_shape(int semiring, int* bm, int* bn, int* bk, int* cps);
int launch_mm_simt_batch(int sr, int device, cudaStream_t stream, int count, const paco_mm_problem* problems);
int launch_mm_tf32x3_presplit(int device, cudaStream_t stream, int count, const void* const* ah,
                              const void* const* al, int64_t lda, const void* const* bth, const void* const* btl,
                              int64_t ldb, void* const* C, int64_t ldc, int64_t n, int64_t m, int64_t k,
                              int flags);
int launch_mm_tf32x3_multi(int device, cudaStream_t stream, int count, const void* const* ah,
                           const void* const* al, int64_t lda, const void* const* bth, const void* const* btl,
                           int64_t ldb, const int32_t* ndst, void* const* dst, const int32_t* sign, int64_t ldc,
                           int64_t n, int64_t m, int64_t k, int flags);
int launch_mm_tf32x3_fused(int device, cudaStream_t stream, int count, const int32_t* nta, const void* const* a_terms,
                           const int32_t* a_sign, int64_t lda, const int32_t* ntb, const void* const* bt_terms,
                           const int32_t* b_sign, int64_t ldb, const int32_t* ndst, void* const* dst,
                           const int32_t* sign, int64_t ldc, int64_t n, int64_t m, int64_t k);
int launch_mm_tf32x3_fused_a(int device, cudaStream_t stream, int count, const int32_t* nta,
                             const void* const* a_terms, const int32_t* a_sign, int64_t lda, const void* const* bt_hi,
                             const void* const* bt_lo, int64_t ldb, const int32_t* ndst, void* const* dst,
                             const int32_t* sign, int64_t ldc, int64_t n, int64_t m, int64_t k);
int launch_mm_tf32b2_multi(int device, cudaStream_t stream, int count, const void* const* a_hi,
                           const void* const* a_h16, const void* const* a_l16, int64_t lda, const void* const* b_hi,
                           const void* const* b_h16, const void* const* b_l16, int64_t ldb, const int32_t* ndst,
                           void* const* dst, const int32_t* sign, int64_t ldc, int64_t n, int64_t m, int64_t k);
int launch_tf32b2_split(cudaStream_t stream, int nin, const void* const* ins, const int64_t* lds,
                        const int32_t* coefs, int64_t rows, int64_t cols, int transpose, void* hi, void* h16,
                        void* l16, int64_t ldo);
int launch_tf32_split(cudaStream_t stream, int nin, const void* const* ins, const int64_t* lds,
                      const int32_t* coefs, int64_t rows, int64_t cols, int transpose, void* hi, void* lo,
                      int64_t ldo);
int launch_fold(int sr, cudaStream_t st, void* dst, int64_t ldd, void* src, int64_t lds, int64_t n,
                int64_t m, int reset);
int launch_fill(int sr, cudaStream_t st, void* dst, int64_t ld, int64_t n, int64_t m);
int launch_naive(int sr, cudaStream_t st, const void* A, int64_t lda, const void* B, int64_t ldb,
                 void* C, int64_t ldc, int64_t n, int64_t m, int64_t k);
int launch_lincomb(int dtype, cudaStream_t st, void* out, int64_t ldo, int64_t n, int64_t m, int nin,
                   const void* const* ins, const int64_t* lds, const int32_t* coefs, int acc);
int launch_narrow_i64(cudaStream_t st, const int64_t* src, int64_t lds, void* dst, int64_t ldd, int64_t n,
                      int64_t m, int64_t lo, int64_t hi, int saturate, int32_t* flag);
int launch_narrow_minplus_inf(cudaStream_t st, const int64_t* src, int64_t lds, void* dst, int64_t ldd, int64_t n,
                              int64_t m, int32_t* flag);
int launch_widen_minplus(cudaStream_t st, const void* r, int64_t ldr, int64_t* c, int64_t ldc, int64_t n, int64_t m,
                         int inf_encoded);
int launch_widen_u32_i64(cudaStream_t st, const void* r, int64_t ldr, int64_t* c, int64_t ldc, int64_t n,
                         int64_t m);
int launch_transpose(cudaStream_t st, int elsize, void* dst, int64_t ldd, const void* src, int64_t lds, int64_t rows,
                     int64_t cols);
int launch_lincomb_multi(cudaStream_t st, int64_t n, int64_t m, int nin, const void* const* ins, const int64_t* lds,
                         int nout, void* const* outs, const int64_t* ldo, const int32_t* coefs);
int launch_strassen_split49(cudaStream_t st, int side, const void* x, int64_t ldx, int64_t h, void* const* his,
                            void* const* los, int64_t ldo);
int launch_lincomb_split(cudaStream_t st, int64_t n, int64_t m, int nin, const void* const* ins, const int64_t* lds,
                         int nout, void* const* his, void* const* los, const int64_t* ldo, const int32_t* coefs);
int launch_mm_bf16x3_multi(int device, cudaStream_t stream, int count, const void* const* a_hi,
                           const void* const* a_lo, int64_t lda, const void* const* b_hi, const void* const* b_lo,
                           int64_t ldb, const int32_t* ndst, void* const* dst, const int32_t* sign, int64_t ldc,
                           int64_t n, int64_t m, int64_t k, int b_natural);
int run_alu_probe(cudaStream_t st, int which, int iters, double* tpc, double* mhz);
struct Box;
}  // namespace paco

using namespace paco;

namespace {
int check_sr(int sr) {
  if (sr < 0 || sr >= PACO_SR_COUNT) {
    set_error("unknown semiring id %d", sr);
    return PACO_ERR_ARG;
  }
  return PACO_OK;
}

// Every entry point selects `device` with cudaSetDevice -- besides selecting
// the device that makes its primary context current on this thread, which the
// driver-API calls we make (cuTensorMapEncodeTiled) need; a fresh worker thread
// whose device is already 0 otherwise has no current context -- and restores
// the caller's context on return, so a C or Python caller's later CUDA work
// without an explicit device still lands where it did before the call.  A
// thread that had no current context gets the previous runtime device back
// only if that device's primary context already exists (never creates one).
class DeviceGuard {
 public:
  int use(int device) {
    static auto get_cur = reinterpret_cast<CUresult (*)(CUcontext*)>(driver_fn("cuCtxGetCurrent"));
    if (get_cur) get_cur(&prev_ctx_);
    cudaGetDevice(&prev_dev_);
    PACO_CUDA_TRY(cudaSetDevice(device));
    dev_ = device;
    return PACO_OK;
  }
  ~DeviceGuard() {
    if (dev_ < 0) return;
    static auto set_cur = reinterpret_cast<CUresult (*)(CUcontext)>(driver_fn("cuCtxSetCurrent"));
    static auto state = reinterpret_cast<CUresult (*)(CUdevice, unsigned*, int*)>(
        driver_fn("cuDevicePrimaryCtxGetState"));
    if (prev_ctx_ && set_cur) {
      set_cur(prev_ctx_);
    } else if (prev_dev_ >= 0 && prev_dev_ != dev_ && state) {
      unsigned flags = 0;
      int active = 0;
      if (state(CUdevice(prev_dev_), &flags, &active) == CUDA_SUCCESS && active) cudaSetDevice(prev_dev_);
    }
  }

 private:
  static void* driver_fn(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return p;
  }
  CUcontext prev_ctx_ = nullptr;
  int prev_dev_ = -1;
  int dev_ = -1;
};

int check_view(const char* what, const void* p, int64_t ld, int64_t rows, int64_t cols) {
  if (rows < 0 || cols < 0) {
    set_error("%s: negative extent %lld x %lld", what, (long long)rows, (long long)cols);
    return PACO_ERR_ARG;
  }
  if (rows > 0 && cols > 0) {
    if (p == nullptr) {
      set_error("%s: null pointer", what);
      return PACO_ERR_ARG;
    }
    if (ld < cols) {
      set_error("%s: leading dimension %lld < columns %lld", what, (long long)ld, (long long)cols);
      return PACO_ERR_ARG;
    }
  }
  return PACO_OK;
}
}  // namespace

#define PACO_TRY(expr)            \
  do {                            \
    int _rc = (expr);             \
    if (_rc != PACO_OK) return _rc; \
  } while (0)

extern "C" {

const char* paco_last_error(void) { return g_err; }
int paco_abi_version(void) { return PACO_ABI_VERSION; }

int paco_mm(int device, void* stream, int semiring, const void* A, int64_t lda, const void* B,
            int64_t ldb, void* C, int64_t ldc, int64_t n, int64_t m, int64_t k, const int32_t* pieces,
            int n_pieces, int flags) {
  PACO_TRY(check_sr(semiring));
  PACO_TRY(check_view("A", A, lda, n, k));
  PACO_TRY(check_view("B", B, ldb, k, m));
  PACO_TRY(check_view("C", C, ldc, n, m));
  if (n == 0 || m == 0) return PACO_OK;
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (k == 0) {
    // empty reduction: C (+)= zero leaves C as is, or C = zero when overwriting
    return (flags & PACO_MM_OVERWRITE) ? launch_fill(semiring, st, C, ldc, n, m) : PACO_OK;
  }
  if (semiring == PACO_SR_BF16_F32)
    return launch_mm_bf16_tc(device, st, A, lda, B, ldb, C, ldc, n, m, k, pieces, n_pieces, flags);
  if (semiring == PACO_SR_F32_TC)
    return launch_mm_f32_tc(device, st, A, lda, B, ldb, C, ldc, n, m, k, pieces, n_pieces, flags);
  return launch_mm_simt(semiring, device, st, A, lda, B, ldb, C, ldc, n, m, k, pieces, n_pieces, flags);
}

int paco_mm_tile_shape(int semiring, int* bm, int* bn, int* bk, int* cps) {
  PACO_TRY(check_sr(semiring));
  if (!bm || !bn || !bk || !cps) {
    set_error("paco_mm_tile_shape: null output pointer");
    return PACO_ERR_ARG;
  }
  if (semiring == PACO_SR_BF16_F32 || semiring == PACO_SR_F32_TC) return tc_tile_shape(semiring, bm, bn, bk, cps);
  return simt_tile_shape(semiring, bm, bn, bk, cps);
}

int paco_fold(int device, void* stream, int semiring, void* dst, int64_t ld_dst, void* src,
              int64_t ld_src, int64_t n, int64_t m, int flags) {
  PACO_TRY(check_sr(semiring));
  if (flags & ~(PACO_FOLD_RESET | PACO_FOLD_ATOMIC)) {
    set_error("paco_fold: unknown flags 0x%x", flags);
    return PACO_ERR_ARG;
  }
  PACO_TRY(check_view("dst", dst, ld_dst, n, m));
  PACO_TRY(check_view("src", src, ld_src, n, m));
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_fold(semiring, static_cast<cudaStream_t>(stream), dst, ld_dst, src, ld_src, n, m, flags);
}

int paco_fill(int device, void* stream, int semiring, void* dst, int64_t ld, int64_t n, int64_t m) {
  PACO_TRY(check_sr(semiring));
  PACO_TRY(check_view("dst", dst, ld, n, m));
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_fill(semiring, static_cast<cudaStream_t>(stream), dst, ld, n, m);
}

int paco_mm_naive(int device, void* stream, int semiring, const void* A, int64_t lda, const void* B,
                  int64_t ldb, void* C, int64_t ldc, int64_t n, int64_t m, int64_t k) {
  PACO_TRY(check_sr(semiring));
  PACO_TRY(check_view("A", A, lda, n, k));
  PACO_TRY(check_view("B", B, ldb, k, m));
  PACO_TRY(check_view("C", C, ldc, n, m));
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_naive(semiring, static_cast<cudaStream_t>(stream), A, lda, B, ldb, C, ldc, n, m, k);
}

int paco_lincomb(int device, void* stream, int dtype, void* out, int64_t ld_out, int64_t n, int64_t m,
                 int nin, const void* const* ins, const int64_t* lds, const int32_t* coefs,
                 int accumulate) {
  PACO_TRY(check_view("out", out, ld_out, n, m));
  for (int q = 0; q < nin; ++q) PACO_TRY(check_view("in", ins[q], lds[q], n, m));
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_lincomb(dtype, static_cast<cudaStream_t>(stream), out, ld_out, n, m, nin, ins, lds,
                        coefs, accumulate);
}

int paco_lincomb_multi(int device, void* stream, int64_t n, int64_t m, int nin, const void* const* ins,
                       const int64_t* lds, int nout, void* const* outs, const int64_t* ldo, const int32_t* coefs) {
  if (!ins || !lds || (nout > 0 && (!outs || !ldo || !coefs))) {
    set_error("paco_lincomb_multi: null arrays");
    return PACO_ERR_ARG;
  }
  for (int q = 0; q < nin && q < 4; ++q) PACO_TRY(check_view("in", ins[q], lds[q], n, m));
  for (int o = 0; o < nout && o < 8; ++o) PACO_TRY(check_view("out", outs[o], ldo[o], n, m));
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_lincomb_multi(static_cast<cudaStream_t>(stream), n, m, nin, ins, lds, nout, outs, ldo, coefs);
}

int paco_lincomb_split(int device, void* stream, int64_t n, int64_t m, int nin, const void* const* ins,
                       const int64_t* lds, int nout, void* const* his, void* const* los, const int64_t* ldo,
                       const int32_t* coefs) {
  if (!ins || !lds || (nout > 0 && (!his || !los || !ldo || !coefs))) {
    set_error("paco_lincomb_split: null arrays");
    return PACO_ERR_ARG;
  }
  for (int q = 0; q < nin && q < 8; ++q) PACO_TRY(check_view("in", ins[q], lds[q], n, m));
  for (int o = 0; o < nout && o < 8; ++o) {
    PACO_TRY(check_view("hi", his[o], ldo[o], n, m));
    PACO_TRY(check_view("lo", los[o], ldo[o], n, m));
  }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_lincomb_split(static_cast<cudaStream_t>(stream), n, m, nin, ins, lds, nout, his, los, ldo, coefs);
}

int paco_strassen_split49(int device, void* stream, int side, const void* x, int64_t ldx, int64_t h,
                          void* const* his, void* const* los, int64_t ldo) {
  if (!x || !his || !los || (side != 0 && side != 1)) {
    set_error("paco_strassen_split49: null arrays or side not 0 (S) / 1 (T)");
    return PACO_ERR_ARG;
  }
  PACO_TRY(check_view("x", x, ldx, 4 * h, 4 * h));
  for (int o = 0; o < 49; ++o) {
    PACO_TRY(check_view("hi", his[o], ldo, h, h));
    PACO_TRY(check_view("lo", los[o], ldo, h, h));
  }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_strassen_split49(static_cast<cudaStream_t>(stream), side, x, ldx, h, his, los, ldo);
}

int paco_mm_bf16x3_multi(int device, void* stream, int count, const void* const* a_hi, const void* const* a_lo,
                         int64_t lda, const void* const* b_hi, const void* const* b_lo, int64_t ldb,
                         const int32_t* ndst, void* const* dst, const int32_t* sign, int64_t ldc, int64_t n,
                         int64_t m, int64_t k) {
  if (count >= 1 && count <= 8 && a_hi && a_lo && b_hi && b_lo && ndst && dst)
    for (int q = 0; q < count; ++q) {
      PACO_TRY(check_view("A_hi", a_hi[q], lda, n, k));
      PACO_TRY(check_view("A_lo", a_lo[q], lda, n, k));
      PACO_TRY(check_view("Bt_hi", b_hi[q], ldb, m, k));
      PACO_TRY(check_view("Bt_lo", b_lo[q], ldb, m, k));
      for (int d = 0; d < ndst[q] && d < 4; ++d) PACO_TRY(check_view("C", dst[4 * q + d], ldc, n, m));
    }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_mm_bf16x3_multi(device, static_cast<cudaStream_t>(stream), count, a_hi, a_lo, lda, b_hi, b_lo, ldb,
                                ndst, dst, sign, ldc, n, m, k, 0);
}

int paco_mm_bf16x3_multi_bn(int device, void* stream, int count, const void* const* a_hi, const void* const* a_lo,
                            int64_t lda, const void* const* b_hi, const void* const* b_lo, int64_t ldb,
                            const int32_t* ndst, void* const* dst, const int32_t* sign, int64_t ldc, int64_t n,
                            int64_t m, int64_t k) {
  if (count >= 1 && count <= 8 && a_hi && a_lo && b_hi && b_lo && ndst && dst)
    for (int q = 0; q < count; ++q) {
      PACO_TRY(check_view("A_hi", a_hi[q], lda, n, k));
      PACO_TRY(check_view("A_lo", a_lo[q], lda, n, k));
      PACO_TRY(check_view("B_hi", b_hi[q], ldb, k, m));
      PACO_TRY(check_view("B_lo", b_lo[q], ldb, k, m));
      for (int d = 0; d < ndst[q] && d < 4; ++d) PACO_TRY(check_view("C", dst[4 * q + d], ldc, n, m));
    }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_mm_bf16x3_multi(device, static_cast<cudaStream_t>(stream), count, a_hi, a_lo, lda, b_hi, b_lo, ldb,
                                ndst, dst, sign, ldc, n, m, k, 1);
}

int paco_mm_batch(int device, void* stream, int semiring, int count, const paco_mm_problem* problems) {
  if (count < 0 || count > PACO_MAX_BATCH || (count > 0 && !problems)) {
    set_error("paco_mm_batch: count=%d (0..%d) with a problem array", count, PACO_MAX_BATCH);
    return PACO_ERR_ARG;
  }
  if (semiring < 0 || semiring >= PACO_SR_COUNT) {
    set_error("unknown semiring id %d", semiring);
    return PACO_ERR_ARG;
  }
  if (semiring == PACO_SR_BF16_F32 || semiring == PACO_SR_F32_TC) {
    set_error("paco_mm_batch: SIMT semirings only (the tcgen05 kernels have their own batch entry)");
    return PACO_ERR_UNSUPPORTED;
  }
  for (int q = 0; q < count; ++q) {
    const paco_mm_problem& P = problems[q];
    if (P.n <= 0 || P.m <= 0) continue;
    PACO_TRY(check_view("C", P.C, P.ldc, P.n, P.m));
    if (P.k > 0) {
      PACO_TRY(check_view("A", P.A, P.lda, P.n, P.k));
      PACO_TRY(check_view("B", P.B, P.ldb, P.k, P.m));
    }
  }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_mm_simt_batch(semiring, device, static_cast<cudaStream_t>(stream), count, problems);
}

int paco_tf32_split(int device, void* stream, int nin, const void* const* ins, const int64_t* lds,
                    const int32_t* coefs, int64_t rows, int64_t cols, int transpose, void* hi, void* lo,
                    int64_t ldo) {
  if (rows <= 0 || cols <= 0) return PACO_OK;
  if (!ins || !lds || !coefs || nin < 1 || nin > 4) {
    set_error("paco_tf32_split: need 1..4 inputs with pitches and coefficients");
    return PACO_ERR_ARG;
  }
  for (int q = 0; q < nin; ++q) PACO_TRY(check_view("in", ins[q], lds[q], rows, cols));
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_tf32_split(static_cast<cudaStream_t>(stream), nin, ins, lds, coefs, rows, cols, transpose, hi,
                           lo, ldo);
}

int paco_mm_tf32x3(int device, void* stream, int count, const void* const* a_hi, const void* const* a_lo,
                   int64_t lda, const void* const* bt_hi, const void* const* bt_lo, int64_t ldb, void* const* C,
                   int64_t ldc, int64_t n, int64_t m, int64_t k, int flags) {
  if (count < 1 || !a_hi || !a_lo || !bt_hi || !bt_lo || !C) {
    set_error("paco_mm_tf32x3: need count >= 1 and pointer arrays");
    return PACO_ERR_ARG;
  }
  if (n <= 0 || m <= 0) return PACO_OK;
  for (int q = 0; q < count; ++q) {
    PACO_TRY(check_view("C", C[q], ldc, n, m));
    if (k > 0) {
      PACO_TRY(check_view("A_hi", a_hi[q], lda, n, k));
      PACO_TRY(check_view("A_lo", a_lo[q], lda, n, k));
      PACO_TRY(check_view("Bt_hi", bt_hi[q], ldb, m, k));
      PACO_TRY(check_view("Bt_lo", bt_lo[q], ldb, m, k));
    }
  }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (k <= 0) {
    if (flags & PACO_MM_OVERWRITE)
      for (int q = 0; q < count; ++q) PACO_TRY(launch_fill(PACO_SR_F32_TC, st, C[q], ldc, n, m));
    return PACO_OK;
  }
  return launch_mm_tf32x3_presplit(device, st, count, a_hi, a_lo, lda, bt_hi, bt_lo, ldb, C, ldc, n, m, k, flags);
}

int paco_mm_tf32x3_multi(int device, void* stream, int count, const void* const* a_hi, const void* const* a_lo,
                         int64_t lda, const void* const* bt_hi, const void* const* bt_lo, int64_t ldb,
                         const int32_t* ndst, void* const* dst, const int32_t* sign, int64_t ldc, int64_t n,
                         int64_t m, int64_t k) {
  if (count < 1 || count > 8 || !a_hi || !a_lo || !bt_hi || !bt_lo || !ndst || !dst || !sign) {
    set_error("paco_mm_tf32x3_multi: need 1 <= count <= 8, pointer arrays and destination lists");
    return PACO_ERR_ARG;
  }
  if (n <= 0 || m <= 0 || k <= 0) return PACO_OK;  // (+)= of an empty product: nothing to fold
  for (int q = 0; q < count; ++q) {
    if (ndst[q] < 1 || ndst[q] > 4) {
      set_error("paco_mm_tf32x3_multi: problem %d has %d destinations (1..4)", q, ndst[q]);
      return PACO_ERR_ARG;
    }
    for (int d = 0; d < ndst[q]; ++d) PACO_TRY(check_view("C", dst[4 * q + d], ldc, n, m));
    PACO_TRY(check_view("A_hi", a_hi[q], lda, n, k));
    PACO_TRY(check_view("A_lo", a_lo[q], lda, n, k));
    PACO_TRY(check_view("Bt_hi", bt_hi[q], ldb, m, k));
    PACO_TRY(check_view("Bt_lo", bt_lo[q], ldb, m, k));
  }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_mm_tf32x3_multi(device, static_cast<cudaStream_t>(stream), count, a_hi, a_lo, lda, bt_hi, bt_lo,
                                ldb, ndst, dst, sign, ldc, n, m, k, 0);
}

int paco_narrow_i64(int device, void* stream, const int64_t* src, int64_t ld_src, void* dst32, int64_t ld_dst,
                    int64_t rows, int64_t cols, int64_t lo, int64_t hi, int saturate, int32_t* flag) {
  PACO_TRY(check_view("src", src, ld_src, rows, cols));
  PACO_TRY(check_view("dst", dst32, ld_dst, rows, cols));
  if (rows > 0 && cols > 0 && !flag) {
    set_error("paco_narrow_i64: null flag");
    return PACO_ERR_ARG;
  }
  if (lo > hi || lo < INT32_MIN || hi > int64_t(UINT32_MAX)) {
    set_error("paco_narrow_i64: range [%lld, %lld] is not a 32-bit range", (long long)lo, (long long)hi);
    return PACO_ERR_ARG;
  }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_narrow_i64(static_cast<cudaStream_t>(stream), src, ld_src, dst32, ld_dst, rows, cols, lo, hi,
                           saturate, flag);
}

int paco_widen_u32_i64(int device, void* stream, const void* r32, int64_t ld_r, int64_t* c, int64_t ld_c,
                       int64_t rows, int64_t cols) {
  PACO_TRY(check_view("r", r32, ld_r, rows, cols));
  PACO_TRY(check_view("c", c, ld_c, rows, cols));
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_widen_u32_i64(static_cast<cudaStream_t>(stream), r32, ld_r, c, ld_c, rows, cols);
}

int paco_narrow_minplus_inf(int device, void* stream, const int64_t* src, int64_t ld_src, void* dst32,
                            int64_t ld_dst, int64_t rows, int64_t cols, int32_t* flag) {
  PACO_TRY(check_view("src", src, ld_src, rows, cols));
  PACO_TRY(check_view("dst", dst32, ld_dst, rows, cols));
  if (rows > 0 && cols > 0 && !flag) {
    set_error("paco_narrow_minplus_inf: null flag");
    return PACO_ERR_ARG;
  }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_narrow_minplus_inf(static_cast<cudaStream_t>(stream), src, ld_src, dst32, ld_dst, rows, cols, flag);
}

int paco_widen_minplus_i64(int device, void* stream, const void* r32, int64_t ld_r, int64_t* c, int64_t ld_c,
                           int64_t rows, int64_t cols, int inf_encoded) {
  PACO_TRY(check_view("r", r32, ld_r, rows, cols));
  PACO_TRY(check_view("c", c, ld_c, rows, cols));
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_widen_minplus(static_cast<cudaStream_t>(stream), r32, ld_r, c, ld_c, rows, cols, inf_encoded);
}

int paco_kernel_timing(int enable) {
  std::lock_guard<std::mutex> lock(g_kt_mu);
  if (enable) {
    for (KRec& r : g_kt_recs) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    g_kt_recs.clear();
  }
  g_ktime_on.store(enable ? 1 : 0);
  return PACO_OK;
}

int paco_kernel_timing_read(int family, double* ms_total, int64_t* launches) {
  if (!ms_total || !launches || family < 0 || family >= PACO_KT_COUNT) {
    set_error("paco_kernel_timing_read: family %d (0..%d) and output pointers", family, PACO_KT_COUNT - 1);
    return PACO_ERR_ARG;
  }
  std::lock_guard<std::mutex> lock(g_kt_mu);
  double tot = 0;
  int64_t cnt = 0;
  for (KRec& r : g_kt_recs) {
    if (r.fam != family) continue;
    DeviceGuard dg;
    PACO_TRY(dg.use(r.dev));
    PACO_CUDA_TRY(cudaEventSynchronize(r.b));
    float ms = 0;
    PACO_CUDA_TRY(cudaEventElapsedTime(&ms, r.a, r.b));
    tot += ms;
    ++cnt;
  }
  *ms_total = tot;
  *launches = cnt;
  return PACO_OK;
}

int paco_mm_tf32x3_fused(int device, void* stream, int count, const int32_t* nta, const void* const* a_terms,
                         const int32_t* a_sign, int64_t lda, const int32_t* ntb, const void* const* bt_terms,
                         const int32_t* b_sign, int64_t ldb, const int32_t* ndst, void* const* dst,
                         const int32_t* sign, int64_t ldc, int64_t n, int64_t m, int64_t k) {
  if (count >= 1 && nta && ntb && a_terms && bt_terms && ndst && dst)
    for (int q = 0; q < count && q < 8; ++q) {
      for (int t = 0; t < nta[q] && t < 2; ++t) PACO_TRY(check_view("A term", a_terms[2 * q + t], lda, n, k));
      for (int t = 0; t < ntb[q] && t < 2; ++t) PACO_TRY(check_view("B^T term", bt_terms[2 * q + t], ldb, m, k));
      for (int d = 0; d < ndst[q] && d < 4; ++d) PACO_TRY(check_view("C", dst[4 * q + d], ldc, n, m));
    }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_mm_tf32x3_fused(device, static_cast<cudaStream_t>(stream), count, nta, a_terms, a_sign, lda, ntb,
                                bt_terms, b_sign, ldb, ndst, dst, sign, ldc, n, m, k);
}

int paco_mm_tf32x3_fused_a(int device, void* stream, int count, const int32_t* nta, const void* const* a_terms,
                           const int32_t* a_sign, int64_t lda, const void* const* bt_hi, const void* const* bt_lo,
                           int64_t ldb, const int32_t* ndst, void* const* dst, const int32_t* sign, int64_t ldc,
                           int64_t n, int64_t m, int64_t k) {
  if (count >= 1 && nta && a_terms && bt_hi && bt_lo && ndst && dst)
    for (int q = 0; q < count && q < 8; ++q) {
      for (int t = 0; t < nta[q] && t < 2; ++t) PACO_TRY(check_view("A term", a_terms[2 * q + t], lda, n, k));
      PACO_TRY(check_view("Bt_hi", bt_hi[q], ldb, m, k));
      PACO_TRY(check_view("Bt_lo", bt_lo[q], ldb, m, k));
      for (int d = 0; d < ndst[q] && d < 4; ++d) PACO_TRY(check_view("C", dst[4 * q + d], ldc, n, m));
    }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_mm_tf32x3_fused_a(device, static_cast<cudaStream_t>(stream), count, nta, a_terms, a_sign, lda, bt_hi,
                                  bt_lo, ldb, ndst, dst, sign, ldc, n, m, k);
}

int paco_tf32b2_split(int device, void* stream, int nin, const void* const* ins, const int64_t* lds,
                      const int32_t* coefs, int64_t rows, int64_t cols, int transpose, void* hi, void* h16, void* l16,
                      int64_t ldo) {
  if (rows <= 0 || cols <= 0) return PACO_OK;
  if (!ins || !lds || !coefs || nin < 1 || nin > 4) {
    set_error("paco_tf32b2_split: need 1..4 inputs with pitches and coefficients");
    return PACO_ERR_ARG;
  }
  for (int q = 0; q < nin; ++q) PACO_TRY(check_view("in", ins[q], lds[q], rows, cols));
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_tf32b2_split(static_cast<cudaStream_t>(stream), nin, ins, lds, coefs, rows, cols, transpose, hi, h16,
                             l16, ldo);
}

int paco_mm_tf32b2_multi(int device, void* stream, int count, const void* const* a_hi, const void* const* a_h16,
                         const void* const* a_l16, int64_t lda, const void* const* b_hi, const void* const* b_h16,
                         const void* const* b_l16, int64_t ldb, const int32_t* ndst, void* const* dst,
                         const int32_t* sign, int64_t ldc, int64_t n, int64_t m, int64_t k) {
  if (count >= 1 && count <= 8 && a_hi && b_hi && ndst && dst)
    for (int q = 0; q < count; ++q) {
      PACO_TRY(check_view("A_hi", a_hi[q], lda, n, k));
      if (a_h16) PACO_TRY(check_view("A_h16", a_h16[q], lda, n, k));
      if (a_l16) PACO_TRY(check_view("A_l16", a_l16[q], lda, n, k));
      PACO_TRY(check_view("Bt_hi", b_hi[q], ldb, m, k));
      if (b_h16) PACO_TRY(check_view("Bt_h16", b_h16[q], ldb, m, k));
      if (b_l16) PACO_TRY(check_view("Bt_l16", b_l16[q], ldb, m, k));
      for (int d = 0; d < ndst[q] && d < 4; ++d) PACO_TRY(check_view("C", dst[4 * q + d], ldc, n, m));
    }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_mm_tf32b2_multi(device, static_cast<cudaStream_t>(stream), count, a_hi, a_h16, a_l16, lda, b_hi,
                                b_h16, b_l16, ldb, ndst, dst, sign, ldc, n, m, k);
}

int paco_transpose(int device, void* stream, int elsize, void* dst, int64_t ld_dst, const void* src, int64_t ld_src,
                   int64_t rows, int64_t cols) {
  PACO_TRY(check_view("src", src, ld_src, rows, cols));
  PACO_TRY(check_view("dst", dst, ld_dst, cols, rows));
  if (elsize != 4 && elsize != 8) {
    set_error("paco_transpose: element size %d (4 or 8)", elsize);
    return PACO_ERR_ARG;
  }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return launch_transpose(static_cast<cudaStream_t>(stream), elsize, dst, ld_dst, src, ld_src, rows, cols);
}

int paco_copy2d(int device, void* stream, void* dst, int64_t dpitch, const void* src, int64_t spitch,
                int64_t width, int64_t rows) {
  if (rows <= 0 || width <= 0) return PACO_OK;
  if (!dst || !src || dpitch < width || spitch < width) {
    set_error("paco_copy2d: bad pointers or pitches");
    return PACO_ERR_ARG;
  }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  PACO_CUDA_TRY(cudaMemcpy2DAsync(dst, size_t(dpitch), src, size_t(spitch), size_t(width), size_t(rows),
                                  cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  return PACO_OK;
}

int paco_host_register(void* ptr, size_t bytes) {
  if (!ptr || bytes == 0) {
    set_error("paco_host_register: empty range");
    return PACO_ERR_ARG;
  }
  PACO_CUDA_TRY(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable));
  return PACO_OK;
}

int paco_host_unregister(void* ptr) {
  PACO_CUDA_TRY(cudaHostUnregister(ptr));
  return PACO_OK;
}

int paco_device_alloc(int device, size_t bytes, void** ptr) {
  if (!ptr) {
    set_error("paco_device_alloc: null output");
    return PACO_ERR_ARG;
  }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  PACO_CUDA_TRY(cudaMalloc(ptr, bytes));
  return PACO_OK;
}

int paco_device_free(int device, void* ptr) {
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  PACO_CUDA_TRY(cudaFree(ptr));
  return PACO_OK;
}

int paco_ipc_handle(int device, void* ptr, void* handle64) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  cudaIpcMemHandle_t h;
  PACO_CUDA_TRY(cudaIpcGetMemHandle(&h, ptr));
  memcpy(handle64, &h, sizeof(h));
  return PACO_OK;
}

int paco_ipc_open(int device, const void* handle64, void** ptr) {
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  PACO_CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return PACO_OK;
}

int paco_ipc_close(int device, void* ptr) {
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  PACO_CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return PACO_OK;
}

int paco_enable_peer(int device, int peer) {
  if (device == peer) return PACO_OK;
  int can = 0;
  PACO_CUDA_TRY(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) {
    set_error("device %d cannot access peer %d", device, peer);
    return PACO_ERR_UNSUPPORTED;
  }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return PACO_OK;
  }
  PACO_CUDA_TRY(e);
  return PACO_OK;
}

int paco_alu_probe(int device, void* stream, int which, int iters, double* tpc, double* mhz) {
  if (!tpc || !mhz || iters < 1) {
    set_error("paco_alu_probe: bad arguments");
    return PACO_ERR_ARG;
  }
  DeviceGuard dg;
  PACO_TRY(dg.use(device));
  return run_alu_probe(static_cast<cudaStream_t>(stream), which, iters, tpc, mhz);
}

}  // extern "C"
