// Elementwise companions of the PACO hot path on sm_100a:
//   fold     REDUCE body  t (+)= temp ; temp = zero        (matmul.py:455-460)
//   fill     temp = semiring zero                          (matmul.py:430-433)
//   naive    defining-sum ground truth, one thread/element (matmul.py:400-414)
//   lincomb  Strassen S/T formation and C-block combination
// All are HBM-bound grid-stride kernels over 2-D strided views; the grid is a
// multiple of the 148 SMs.
#include <cstdio>

#include <cstring>

#include <cuda_bf16.h>

#include "common.cuh"
#include "semiring_ops.cuh"

namespace paco {

namespace {
int ew_grid(int64_t n_elems, int threads) {
  const int64_t want = (n_elems + threads - 1) / threads;
  const int64_t cap = int64_t(kNumSMs) * 16;
  return int(want < 1 ? 1 : (want > cap ? cap : want));
}
}  // namespace

// flags: PACO_FOLD_RESET (src = zero afterwards), PACO_FOLD_ATOMIC (dst (+)= src
// as one global atomic per element: safe while other kernels fold into dst).
template <class Op>
__global__ void fold_kernel(typename Op::TC* dst, int64_t ldd, typename Op::TC* src, int64_t lds,
                            int64_t n, int64_t m, int flags) {
  const auto z = Op::zero();
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y)
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m; j += int64_t(gridDim.x) * blockDim.x) {
      typename Op::TC* s = src + i * lds + j;
      typename Op::TC* d = dst + i * ldd + j;
      if (flags & PACO_FOLD_ATOMIC)
        Op::atomic_combine(d, *s);
      else
        *d = Op::combine(*d, *s);
      if (flags & PACO_FOLD_RESET) *s = z;
    }
}

template <class Op>
__global__ void fill_kernel(typename Op::TC* dst, int64_t ld, int64_t n, int64_t m) {
  const int64_t total = n * m;
  const auto z = Op::zero();
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / m, j = e - i * m;
    dst[i * ld + j] = z;
  }
}

// mm_oracle (matmul.py:400-414): acc starts at the semiring identity, folds
// every term in l order, then C = C (+) acc.  No tiling, no shared memory: an
// independent device-side ground truth for the tiled kernels.
template <class Op>
__global__ void naive_kernel(const typename Op::TA* A, int64_t lda, const typename Op::TB* B,
                             int64_t ldb, typename Op::TC* C, int64_t ldc, int64_t n, int64_t m,
                             int64_t k) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t i = blockIdx.y;
  if (j >= m || i >= n) return;
  typename Op::Acc acc = Op::identity();
  for (int64_t l = 0; l < k; ++l) acc = Op::mac(acc, A[i * lda + l], B[l * ldb + j]);
  C[i * ldc + j] = Op::combine(C[i * ldc + j], Op::finish(acc));
}

template <class T, int NIN>
struct LinArgs {
  const T* in[NIN];
  int64_t ld[NIN];
  int32_t coef[NIN];
};

// 2-D: blockIdx.x covers 4*blockDim.x columns, rows strided over gridDim.y;
// kVec: 16-byte vectors when every view is aligned (f32: 4, f64/i64: 2 lanes).
template <class T>
struct Vec16 {
  static constexpr int N = 16 / sizeof(T);
  T v[N];
};

template <class T, int NIN, bool kVec>
__global__ void lincomb_kernel(T* out, int64_t ldo, int64_t n, int64_t m, const LinArgs<T, NIN> a,
                               int nin, int accumulate) {
  constexpr int V = kVec ? Vec16<T>::N : 1;
  const int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * V;
  if (j >= m) return;
  int64_t i0 = blockIdx.y;
  if (kVec) {
    // U rows per pass with every 16-byte load issued before any arithmetic or
    // store (U x (nin + accumulate) loads in flight per thread)
    constexpr int U = 4;
    const int64_t gy = gridDim.y;
    for (; i0 + (U - 1) * gy < n; i0 += U * gy) {
      Vec16<T> x[U][NIN], acc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * gy;
        if (accumulate)
          acc[u] = *reinterpret_cast<const Vec16<T>*>(out + i * ldo + j);
        else
#pragma unroll
          for (int e = 0; e < V; ++e) acc[u].v[e] = T(0);
#pragma unroll
        for (int q = 0; q < NIN; ++q)
          if (q < nin) x[u][q] = *reinterpret_cast<const Vec16<T>*>(a.in[q] + i * a.ld[q] + j);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int q = 0; q < NIN; ++q)
          if (q < nin)
#pragma unroll
            for (int e = 0; e < V; ++e)
              acc[u].v[e] = a.coef[q] > 0 ? acc[u].v[e] + x[u][q].v[e] : acc[u].v[e] - x[u][q].v[e];
        *reinterpret_cast<Vec16<T>*>(out + (i0 + u * gy) * ldo + j) = acc[u];
      }
    }
  }
  for (int64_t i = i0; i < n; i += gridDim.y) {
    if (kVec) {
      Vec16<T> acc;
      if (accumulate)
        acc = *reinterpret_cast<const Vec16<T>*>(out + i * ldo + j);
      else
#pragma unroll
        for (int e = 0; e < V; ++e) acc.v[e] = T(0);
#pragma unroll
      for (int q = 0; q < NIN; ++q)
        if (q < nin) {
          const Vec16<T> x = *reinterpret_cast<const Vec16<T>*>(a.in[q] + i * a.ld[q] + j);
#pragma unroll
          for (int e = 0; e < V; ++e) acc.v[e] = a.coef[q] > 0 ? acc.v[e] + x.v[e] : acc.v[e] - x.v[e];
        }
      *reinterpret_cast<Vec16<T>*>(out + i * ldo + j) = acc;
    } else {
      T v = accumulate ? out[i * ldo + j] : T(0);
#pragma unroll
      for (int q = 0; q < NIN; ++q)
        if (q < nin) {
          const T x = a.in[q][i * a.ld[q] + j];
          v = a.coef[q] > 0 ? v + x : v - x;
        }
      out[i * ldo + j] = v;
    }
  }
}

int launch_fold(int sr, cudaStream_t st, void* dst, int64_t ldd, void* src, int64_t lds, int64_t n,
                int64_t m, int flags) {
  if (n <= 0 || m <= 0) return PACO_OK;
  return dispatch_op(sr, [&](auto op) -> int {
    using Op = decltype(op);
    using TC = typename Op::TC;
    const int64_t xb = (m + 255) / 256, yb0 = n < 65535 ? n : 65535, ycap = 2368 / xb + 1;
    const dim3 grid(unsigned(xb), unsigned(yb0 < ycap ? yb0 : ycap));
    KernelSpan ks(PACO_KT_ELEMENTWISE, st);
    fold_kernel<Op><<<grid, 256, 0, st>>>(static_cast<TC*>(dst), ldd, static_cast<TC*>(src), lds, n, m, flags);
    PACO_CUDA_TRY(cudaGetLastError());
    return PACO_OK;
  });
}

int launch_fill(int sr, cudaStream_t st, void* dst, int64_t ld, int64_t n, int64_t m) {
  if (n <= 0 || m <= 0) return PACO_OK;
  return dispatch_op(sr, [&](auto op) -> int {
    using Op = decltype(op);
    using TC = typename Op::TC;
    const TC z = Op::zero();
    unsigned char bytes[sizeof(TC)];
    memcpy(bytes, &z, sizeof(TC));
    bool all_zero = true;
    for (size_t i = 0; i < sizeof(TC); ++i) all_zero = all_zero && bytes[i] == 0;
    if (all_zero) {  // (+,x) zero: a 2-D memset runs at the copy engine's write rate
      PACO_CUDA_TRY(cudaMemset2DAsync(dst, size_t(ld) * sizeof(TC), 0, size_t(m) * sizeof(TC), size_t(n), st));
      return PACO_OK;
    }
    KernelSpan ks(PACO_KT_ELEMENTWISE, st);
    fill_kernel<Op><<<ew_grid(n * m, 256), 256, 0, st>>>(static_cast<TC*>(dst), ld, n, m);
    PACO_CUDA_TRY(cudaGetLastError());
    return PACO_OK;
  });
}

int launch_naive(int sr, cudaStream_t st, const void* A, int64_t lda, const void* B, int64_t ldb,
                 void* C, int64_t ldc, int64_t n, int64_t m, int64_t k) {
  if (n <= 0 || m <= 0) return PACO_OK;
  if (n > 65535) {
    set_error("paco_mm_naive: n=%lld exceeds the 65535-row grid limit", (long long)n);
    return PACO_ERR_ARG;
  }
  return dispatch_op(sr, [&](auto op) -> int {
    using Op = decltype(op);
    dim3 grid(unsigned((m + 127) / 128), unsigned(n));
    naive_kernel<Op><<<grid, 128, 0, st>>>(static_cast<const typename Op::TA*>(A), lda,
                                           static_cast<const typename Op::TB*>(B), ldb,
                                           static_cast<typename Op::TC*>(C), ldc, n, m, k);
    PACO_CUDA_TRY(cudaGetLastError());
    return PACO_OK;
  });
}

template <class T>
int lincomb_t(cudaStream_t st, void* out, int64_t ldo, int64_t n, int64_t m, int nin,
              const void* const* ins, const int64_t* lds, const int32_t* coefs, int acc) {
  LinArgs<T, 4> a{};
  for (int q = 0; q < nin; ++q) {
    a.in[q] = static_cast<const T*>(ins[q]);
    a.ld[q] = lds[q];
    a.coef[q] = coefs[q];
  }
  constexpr int V = Vec16<T>::N;
  bool vec = (m % V == 0) && (ldo % V == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  for (int q = 0; q < nin; ++q)
    vec = vec && (lds[q] % V == 0) && (reinterpret_cast<uintptr_t>(ins[q]) % 16 == 0);
  const int64_t lanes = vec ? m / V : m;
  const int64_t xb = (lanes + 127) / 128;
  const int64_t yb = n < 65535 ? n : 65535;
  const int64_t ycap = 2368 / xb + 1;
  dim3 grid(unsigned(xb), unsigned(yb < ycap ? yb : ycap));
  KernelSpan ks(PACO_KT_LINCOMB, st);
  if (vec)
    lincomb_kernel<T, 4, true><<<grid, 128, 0, st>>>(static_cast<T*>(out), ldo, n, m, a, nin, acc);
  else
    lincomb_kernel<T, 4, false><<<grid, 128, 0, st>>>(static_cast<T*>(out), ldo, n, m, a, nin, acc);
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
}

// Several signed sums of the same inputs in one pass (Strassen's formation of a
// node: S1, S2, S5, S6, S7 from A's four quadrants): every input element is
// read once and every output written once -- 4 reads + 5 writes per element
// instead of 10 + 5 for five separate two-term lincombs.  coef[o * NIN + i] in
// {-1, 0, +1}; fp32, 16-byte vectors (all views 16-byte aligned, m % 4 == 0).
constexpr int kMultiIn = 4, kMultiOut = 8;
struct MultiArgs {
  const float* in[kMultiIn];
  int64_t ldi[kMultiIn];
  float* out[kMultiOut];
  int64_t ldo[kMultiOut];
  int8_t coef[kMultiOut * kMultiIn];
  int32_t nin, nout;
};

__global__ void __launch_bounds__(128) lincomb_multi_kernel(const MultiArgs a, int64_t n, int64_t m) {
  const int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (j >= m) return;
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y) {
    float4 x[kMultiIn];
#pragma unroll
    for (int q = 0; q < kMultiIn; ++q)
      if (q < a.nin) x[q] = __ldcs(reinterpret_cast<const float4*>(a.in[q] + i * a.ldi[q] + j));
#pragma unroll
    for (int o = 0; o < kMultiOut; ++o) {
      if (o >= a.nout) break;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int q = 0; q < kMultiIn; ++q) {
        if (q >= a.nin) break;
        const int c = a.coef[o * kMultiIn + q];
        if (c > 0) {
          v.x += x[q].x; v.y += x[q].y; v.z += x[q].z; v.w += x[q].w;
        } else if (c < 0) {
          v.x -= x[q].x; v.y -= x[q].y; v.z -= x[q].z; v.w -= x[q].w;
        }
      }
      __stcs(reinterpret_cast<float4*>(a.out[o] + i * a.ldo[o] + j), v);
    }
  }
}

int launch_lincomb_multi(cudaStream_t st, int64_t n, int64_t m, int nin, const void* const* ins, const int64_t* lds,
                         int nout, void* const* outs, const int64_t* ldo, const int32_t* coefs) {
  if (n <= 0 || m <= 0 || nout == 0) return PACO_OK;
  if (nin < 1 || nin > kMultiIn || nout < 0 || nout > kMultiOut) {
    set_error("paco_lincomb_multi: %d inputs (1..%d), %d outputs (0..%d)", nin, kMultiIn, nout, kMultiOut);
    return PACO_ERR_ARG;
  }
  MultiArgs a{};
  a.nin = nin;
  a.nout = nout;
  bool ok = m % 4 == 0;
  for (int q = 0; q < nin; ++q) {
    a.in[q] = static_cast<const float*>(ins[q]);
    a.ldi[q] = lds[q];
    ok = ok && lds[q] % 4 == 0 && reinterpret_cast<uintptr_t>(ins[q]) % 16 == 0;
  }
  for (int o = 0; o < nout; ++o) {
    a.out[o] = static_cast<float*>(outs[o]);
    a.ldo[o] = ldo[o];
    ok = ok && ldo[o] % 4 == 0 && reinterpret_cast<uintptr_t>(outs[o]) % 16 == 0;
    for (int q = 0; q < nin; ++q) a.coef[o * kMultiIn + q] = int8_t(coefs[o * nin + q] > 0 ? 1 : (coefs[o * nin + q] < 0 ? -1 : 0));
  }
  if (!ok) {
    set_error("paco_lincomb_multi: views need 16-byte aligned starts, pitches and a column count % 4 == 0");
    return PACO_ERR_UNSUPPORTED;
  }
  KernelSpan ks(PACO_KT_LINCOMB, st);
  const int64_t xb = (m / 4 + 127) / 128, yb = n < 65535 ? n : 65535, ycap = 2368 / xb + 1;
  lincomb_multi_kernel<<<dim3(unsigned(xb), unsigned(yb < ycap ? yb : ycap)), 128, 0, st>>>(a, n, m);
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
}

// Strassen leaf operands in the bf16x3 format (paco_lincomb_split): the same
// signed sums as lincomb_multi, each written as two bf16 planes hi = bf16_rn(x),
// lo = bf16_rn(x - hi) (x = hi + lo to 2^-17 relative); a one-term row is a
// split copy.  Eight columns per thread: 2 x 16-byte loads per input, one
// 16-byte store per plane; 4 bytes written per output element, as an fp32 sum.
// Up to 8 inputs: a leaf-level node's operands straight from the level-0 blocks
// (S_r's quadrant q = sum of its terms' sub-quadrants q), skipping the
// level-1 fp32 sums.
constexpr int kSplitIn = 8;
struct SplitArgs {
  const float* in[kSplitIn];
  int64_t ldi[kSplitIn];
  __nv_bfloat16* hi[kMultiOut];
  __nv_bfloat16* lo[kMultiOut];
  int64_t ldo[kMultiOut];
  int8_t coef[kMultiOut * kSplitIn];
  int32_t nin, nout;
};

__device__ __forceinline__ uint32_t bf16x2_bits(__nv_bfloat16 a, __nv_bfloat16 b) {
  return uint32_t(__bfloat16_as_ushort(a)) | (uint32_t(__bfloat16_as_ushort(b)) << 16);
}

template <int NI>
__global__ void __launch_bounds__(128) lincomb_split_kernel(const SplitArgs a, int64_t n, int64_t m) {
  const int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (j >= m) return;
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y) {
    float x[NI][8];
#pragma unroll
    for (int q = 0; q < NI; ++q)
      if (q < a.nin) {
        const float4* p = reinterpret_cast<const float4*>(a.in[q] + i * a.ldi[q] + j);
        const float4 u = __ldcs(p), w = __ldcs(p + 1);
        x[q][0] = u.x; x[q][1] = u.y; x[q][2] = u.z; x[q][3] = u.w;
        x[q][4] = w.x; x[q][5] = w.y; x[q][6] = w.z; x[q][7] = w.w;
      }
#pragma unroll
    for (int o = 0; o < kMultiOut; ++o) {
      if (o >= a.nout) break;
      float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int q = 0; q < NI; ++q) {
        if (q >= a.nin) break;
        const int c = a.coef[o * kSplitIn + q];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = c > 0 ? v[e] + x[q][e] : (c < 0 ? v[e] - x[q][e] : v[e]);
      }
      uint32_t h[4], l[4];
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        const __nv_bfloat16 h0 = __float2bfloat16_rn(v[e]), h1 = __float2bfloat16_rn(v[e + 1]);
        h[e / 2] = bf16x2_bits(h0, h1);
        l[e / 2] = bf16x2_bits(__float2bfloat16_rn(v[e] - __bfloat162float(h0)),
                               __float2bfloat16_rn(v[e + 1] - __bfloat162float(h1)));
      }
      __stcs(reinterpret_cast<uint4*>(a.hi[o] + i * a.ldo[o] + j), make_uint4(h[0], h[1], h[2], h[3]));
      __stcs(reinterpret_cast<uint4*>(a.lo[o] + i * a.ldo[o] + j), make_uint4(l[0], l[1], l[2], l[3]));
    }
  }
}

int launch_lincomb_split(cudaStream_t st, int64_t n, int64_t m, int nin, const void* const* ins, const int64_t* lds,
                         int nout, void* const* his, void* const* los, const int64_t* ldo, const int32_t* coefs) {
  if (n <= 0 || m <= 0 || nout == 0) return PACO_OK;
  if (nin < 1 || nin > kSplitIn || nout < 0 || nout > kMultiOut) {
    set_error("paco_lincomb_split: %d inputs (1..%d), %d outputs (0..%d)", nin, kSplitIn, nout, kMultiOut);
    return PACO_ERR_ARG;
  }
  SplitArgs a{};
  a.nin = nin;
  a.nout = nout;
  bool ok = m % 8 == 0;
  for (int q = 0; q < nin; ++q) {
    a.in[q] = static_cast<const float*>(ins[q]);
    a.ldi[q] = lds[q];
    ok = ok && lds[q] % 4 == 0 && reinterpret_cast<uintptr_t>(ins[q]) % 16 == 0;
  }
  for (int o = 0; o < nout; ++o) {
    a.hi[o] = static_cast<__nv_bfloat16*>(his[o]);
    a.lo[o] = static_cast<__nv_bfloat16*>(los[o]);
    a.ldo[o] = ldo[o];
    ok = ok && ldo[o] % 8 == 0 && reinterpret_cast<uintptr_t>(his[o]) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(los[o]) % 16 == 0;
    for (int q = 0; q < nin; ++q) a.coef[o * kSplitIn + q] = int8_t(coefs[o * nin + q] > 0 ? 1 : (coefs[o * nin + q] < 0 ? -1 : 0));
  }
  if (!ok) {
    set_error("paco_lincomb_split: views need 16-byte aligned starts and pitches and a column count %% 8 == 0");
    return PACO_ERR_UNSUPPORTED;
  }
  KernelSpan ks(PACO_KT_LINCOMB, st);
  const int64_t xb = (m / 8 + 127) / 128, yb = n < 65535 ? n : 65535;
  // one wave: as many row-striding blocks as fit on the 148 SMs at once (a partial
  // last wave of a fixed 2368-block grid cost ~5 %)
  static int occ[2] = {0, 0};
  const int w = nin <= 4 ? 0 : 1;
  if (!occ[w]) {
    int b = 0;
    if (w == 0)
      PACO_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, lincomb_split_kernel<4>, 128, 0));
    else
      PACO_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, lincomb_split_kernel<8>, 128, 0));
    occ[w] = b > 0 ? b : 1;
  }
  const int64_t ywave = int64_t(occ[w]) * kNumSMs / xb;
  const dim3 grid(unsigned(xb), unsigned(yb < ywave ? yb : (ywave > 0 ? ywave : 1)));
  if (w == 0)
    lincomb_split_kernel<4><<<grid, 128, 0, st>>>(a, n, m);
  else
    lincomb_split_kernel<8><<<grid, 128, 0, st>>>(a, n, m);
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
}

// All 49 leaf operands of a 2-level Strassen side in ONE pass over the 16
// level-0 blocks X[q1][q2] (q = 00, 01, 10, 11; X = A for the S side, B for
// the T side, both in natural orientation): leaf (r, r') = sum over the terms
// (c1, q1) of formula r and (c2, q2) of formula r' of c1 c2 X[q1][q2]
// (PAPER.md:1839-1852), written as bf16 hi / lo planes.  Each block is read
// once (the per-node passes re-read a level-0 block once per term: 3 GB vs
// 1 GB per side at cfg5).  The formulas are compile-time tables, so after
// unrolling every input index is a register.
struct Split49Args {
  const float* x;      // the n x n operand, n = 4 h
  int64_t ldx;
  __nv_bfloat16* hi[49];
  __nv_bfloat16* lo[49];
  int64_t ldo;
};
struct StrassenTab {
  int8_t q[7][2], c[7][2];
};
__host__ __device__ constexpr StrassenTab strassen_tab(bool t) {
  // formula r (0..6) -> up to two terms: quadrant q (00, 01, 10, 11 = 0..3; -1 = none)
  // with sign c -- strassen.py S_TERMS (A's terms) / T_TERMS (B's terms)
  return t ? StrassenTab{{{0, 3}, {0, -1}, {1, 3}, {2, 0}, {3, -1}, {0, 1}, {2, 3}},
                         {{1, 1}, {1, 0}, {1, -1}, {1, -1}, {1, 0}, {1, 1}, {1, 1}}}
           : StrassenTab{{{0, 3}, {2, 3}, {0, -1}, {3, -1}, {0, 1}, {2, 0}, {1, 3}},
                         {{1, 1}, {1, 1}, {1, 0}, {1, 0}, {1, 1}, {1, -1}, {1, -1}}};
}

template <bool T>
__global__ void __launch_bounds__(128) strassen_split49_kernel(const Split49Args a, int64_t h) {
  // four columns per thread: 64 input registers, so four CTAs fit per SM and the
  // next row's loads of one warp overlap another warp's 98 plane stores
  constexpr StrassenTab tab = strassen_tab(T);
  const int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (j >= h) return;
  for (int64_t i = blockIdx.y; i < h; i += gridDim.y) {
    float x[16][4];  // [q1 * 4 + q2][column]
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      const int q1 = b >> 2, q2 = b & 3;
      const int64_t row = (q1 >> 1) * 2 * h + (q2 >> 1) * h + i, col = (q1 & 1) * 2 * h + (q2 & 1) * h + j;
      const float4 u = __ldcs(reinterpret_cast<const float4*>(a.x + row * a.ldx + col));
      x[b][0] = u.x; x[b][1] = u.y; x[b][2] = u.z; x[b][3] = u.w;
    }
#pragma unroll
    for (int r = 0; r < 7; ++r)
#pragma unroll
      for (int r2 = 0; r2 < 7; ++r2) {
        float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int t1 = 0; t1 < 2; ++t1)
#pragma unroll
          for (int t2 = 0; t2 < 2; ++t2) {
            const int q1 = tab.q[r][t1], q2 = tab.q[r2][t2];
            if (q1 < 0 || q2 < 0) continue;
            const int c = tab.c[r][t1] * tab.c[r2][t2];
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = c > 0 ? v[e] + x[q1 * 4 + q2][e] : v[e] - x[q1 * 4 + q2][e];
          }
        uint32_t hh[2], ll[2];
#pragma unroll
        for (int e = 0; e < 4; e += 2) {
          const __nv_bfloat16 h0 = __float2bfloat16_rn(v[e]), h1 = __float2bfloat16_rn(v[e + 1]);
          hh[e / 2] = bf16x2_bits(h0, h1);
          ll[e / 2] = bf16x2_bits(__float2bfloat16_rn(v[e] - __bfloat162float(h0)),
                                  __float2bfloat16_rn(v[e + 1] - __bfloat162float(h1)));
        }
        const int o = r * 7 + r2;
        __stcs(reinterpret_cast<uint2*>(a.hi[o] + i * a.ldo + j), make_uint2(hh[0], hh[1]));
        __stcs(reinterpret_cast<uint2*>(a.lo[o] + i * a.ldo + j), make_uint2(ll[0], ll[1]));
      }
  }
}

int launch_strassen_split49(cudaStream_t st, int side, const void* x, int64_t ldx, int64_t h, void* const* his,
                            void* const* los, int64_t ldo) {
  if (h <= 0) return PACO_OK;
  Split49Args a{};
  a.x = static_cast<const float*>(x);
  a.ldx = ldx;
  a.ldo = ldo;
  bool ok = h % 8 == 0 && ldx % 4 == 0 && ldo % 8 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0;
  for (int o = 0; o < 49; ++o) {
    a.hi[o] = static_cast<__nv_bfloat16*>(his[o]);
    a.lo[o] = static_cast<__nv_bfloat16*>(los[o]);
    ok = ok && reinterpret_cast<uintptr_t>(his[o]) % 16 == 0 && reinterpret_cast<uintptr_t>(los[o]) % 16 == 0;
  }
  if (!ok) {
    set_error("paco_strassen_split49: 16-byte aligned operand and planes, h %% 8 == 0");
    return PACO_ERR_UNSUPPORTED;
  }
  KernelSpan ks(PACO_KT_LINCOMB, st);
  static int occ[2] = {0, 0};
  const int w = side ? 1 : 0;
  if (!occ[w]) {
    int b = 0;
    if (w)
      PACO_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, strassen_split49_kernel<true>, 128, 0));
    else
      PACO_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, strassen_split49_kernel<false>, 128, 0));
    occ[w] = b > 0 ? b : 1;
  }
  const int64_t xb = (h / 4 + 127) / 128, ywave = int64_t(occ[w]) * kNumSMs / xb;
  const dim3 grid(unsigned(xb), unsigned(h < ywave ? h : (ywave > 0 ? ywave : 1)));
  if (w)
    strassen_split49_kernel<true><<<grid, 128, 0, st>>>(a, h);
  else
    strassen_split49_kernel<false><<<grid, 128, 0, st>>>(a, h);
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
}

int launch_lincomb(int dtype, cudaStream_t st, void* out, int64_t ldo, int64_t n, int64_t m, int nin,
                   const void* const* ins, const int64_t* lds, const int32_t* coefs, int acc) {
  if (nin < 0 || nin > 4) {
    set_error("paco_lincomb: nin=%d (1..4 supported)", nin);
    return PACO_ERR_ARG;
  }
  if (n <= 0 || m <= 0) return PACO_OK;
  switch (dtype) {
    case PACO_DT_F32: return lincomb_t<float>(st, out, ldo, n, m, nin, ins, lds, coefs, acc);
    case PACO_DT_F64: return lincomb_t<double>(st, out, ldo, n, m, nin, ins, lds, coefs, acc);
    case PACO_DT_I64: return lincomb_t<long long>(st, out, ldo, n, m, nin, ins, lds, coefs, acc);
    default: set_error("paco_lincomb: unknown dtype %d", dtype); return PACO_ERR_ARG;
  }
}

// Range-checked int64 -> 32-bit narrowing (paco_narrow_i64): two elements per
// thread per row pass, rows over blockIdx.y; out-of-range values raise the
// block's vote and one thread stores the flag.
__global__ void narrow_i64_kernel(const int64_t* __restrict__ src, int64_t lds, uint32_t* __restrict__ dst,
                                  int64_t ldd, int64_t n, int64_t m, int64_t lo, int64_t hi, int saturate,
                                  int32_t* flag) {
  int bad = 0;
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y)
    for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 2; j < m;
         j += int64_t(gridDim.x) * blockDim.x * 2) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (j + e >= m) break;
        int64_t v = __ldcs(src + i * lds + j + e);
        if (v < lo) bad = 1;
        if (v > hi) {
          if (saturate)
            v = hi;
          else
            bad = 1;
        }
        dst[i * ldd + j + e] = static_cast<uint32_t>(v);
      }
    }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

__global__ void widen_u32_i64_kernel(const uint32_t* __restrict__ r, int64_t ldr, int64_t* __restrict__ c,
                                     int64_t ldc, int64_t n, int64_t m) {
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y)
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m; j += int64_t(gridDim.x) * blockDim.x) {
      const uint32_t v = __ldcs(r + i * ldr + j);
      if (v != 0xFFFFFFFFu) c[i * ldc + j] = int64_t(v);
    }
}

// SEMIRING_MINPLUS operand -> u32 code keeping INF = 2^62 exact (paco_narrow_minplus_inf)
__global__ void narrow_minplus_inf_kernel(const int64_t* __restrict__ src, int64_t lds, uint32_t* __restrict__ dst,
                                          int64_t ldd, int64_t n, int64_t m, int32_t* flag) {
  constexpr int64_t kInf = int64_t(1) << 62, kMaxFinite = (int64_t(1) << 30) - 2;
  int bad = 0;
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y)
    for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 2; j < m;
         j += int64_t(gridDim.x) * blockDim.x * 2) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (j + e >= m) break;
        const int64_t v = __ldcs(src + i * lds + j + e);
        uint32_t code = 0;
        if (v == kInf)
          code = 0x80000000u;
        else if (v >= 0 && v <= kMaxFinite)
          code = uint32_t(v) + 1u;
        else
          bad = 1;
        dst[i * ldd + j + e] = code;
      }
    }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

// c = min(c, decode(r)) in int64 (paco_widen_minplus_i64)
__global__ void widen_minplus_kernel(const uint32_t* __restrict__ r, int64_t ldr, int64_t* __restrict__ c,
                                     int64_t ldc, int64_t n, int64_t m, int inf_encoded) {
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y)
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m; j += int64_t(gridDim.x) * blockDim.x) {
      const uint32_t v = __ldcs(r + i * ldr + j);
      if (v == 0xFFFFFFFFu) continue;  // no term reached this element
      int64_t x;
      if (!inf_encoded)
        x = int64_t(v);
      else if (v == 0u)
        x = INT64_MIN;  // INF + INF: the reference's int64 sum 2^63 wraps
      else if (v < 0x80000000u)
        x = int64_t(v) - 2;
      else
        x = (int64_t(1) << 62) + int64_t(v - 0x80000001u);
      int64_t* p = c + i * ldc + j;
      if (x < *p) *p = x;
    }
}

// dst (cols x rows) = src^T through a padded 32 x 32 smem tile: reads and
// writes both coalesced along rows (blockDim 32 x 8, each thread 4 rows).
template <class T>
__global__ void __launch_bounds__(256) transpose_kernel(T* __restrict__ dst, int64_t ldd, const T* __restrict__ src,
                                                        int64_t lds, int64_t rows, int64_t cols) {
  __shared__ T tile[32][33];
  const int64_t c0 = int64_t(blockIdx.x) * 32, r0 = int64_t(blockIdx.y) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int64_t r = r0 + ty + k, c = c0 + tx;
    if (r < rows && c < cols) tile[ty + k][tx] = __ldcs(src + r * lds + c);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int64_t orow = c0 + ty + k, ocol = r0 + tx;  // output row = input column
    if (orow < cols && ocol < rows) __stcs(dst + orow * ldd + ocol, tile[tx][ty + k]);
  }
}

int launch_transpose(cudaStream_t st, int elsize, void* dst, int64_t ldd, const void* src, int64_t lds, int64_t rows,
                     int64_t cols) {
  if (rows <= 0 || cols <= 0) return PACO_OK;
  if ((cols + 31) / 32 > INT32_MAX || (rows + 31) / 32 > 65535 * 32) {
    set_error("paco_transpose: %lld x %lld exceeds the grid", (long long)rows, (long long)cols);
    return PACO_ERR_ARG;
  }
  KernelSpan ks(PACO_KT_ELEMENTWISE, st);
  const dim3 block(32, 8);
  const int64_t gy = (rows + 31) / 32;
  // grid.y is capped at 65535: walk the row tiles in chunks
  for (int64_t y0 = 0; y0 < gy; y0 += 65535) {
    const int64_t ny = gy - y0 < 65535 ? gy - y0 : 65535;
    const dim3 grid(unsigned((cols + 31) / 32), unsigned(ny));
    const int64_t r_off = y0 * 32;
    if (elsize == 4)
      transpose_kernel<uint32_t><<<grid, block, 0, st>>>(static_cast<uint32_t*>(dst) + r_off, ldd,
                                                         static_cast<const uint32_t*>(src) + r_off * lds, lds,
                                                         rows - r_off, cols);
    else
      transpose_kernel<unsigned long long><<<grid, block, 0, st>>>(
          static_cast<unsigned long long*>(dst) + r_off, ldd, static_cast<const unsigned long long*>(src) + r_off * lds,
          lds, rows - r_off, cols);
  }
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
}

namespace {
dim3 rows_grid(int64_t n, int64_t m, int per_block) {
  const int64_t xb = (m + per_block - 1) / per_block, yb = n < 65535 ? n : 65535, ycap = 2368 / xb + 1;
  return dim3(unsigned(xb), unsigned(yb < ycap ? yb : ycap));
}
}  // namespace

int launch_narrow_i64(cudaStream_t st, const int64_t* src, int64_t lds, void* dst, int64_t ldd, int64_t n,
                      int64_t m, int64_t lo, int64_t hi, int saturate, int32_t* flag) {
  if (n <= 0 || m <= 0) return PACO_OK;
  KernelSpan ks(PACO_KT_ELEMENTWISE, st);
  narrow_i64_kernel<<<rows_grid(n, m, 512), 256, 0, st>>>(src, lds, static_cast<uint32_t*>(dst), ldd, n, m, lo,
                                                           hi, saturate, flag);
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
}

int launch_narrow_minplus_inf(cudaStream_t st, const int64_t* src, int64_t lds, void* dst, int64_t ldd, int64_t n,
                              int64_t m, int32_t* flag) {
  if (n <= 0 || m <= 0) return PACO_OK;
  KernelSpan ks(PACO_KT_ELEMENTWISE, st);
  narrow_minplus_inf_kernel<<<rows_grid(n, m, 512), 256, 0, st>>>(src, lds, static_cast<uint32_t*>(dst), ldd, n, m,
                                                                   flag);
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
}

int launch_widen_minplus(cudaStream_t st, const void* r, int64_t ldr, int64_t* c, int64_t ldc, int64_t n, int64_t m,
                         int inf_encoded) {
  if (n <= 0 || m <= 0) return PACO_OK;
  KernelSpan ks(PACO_KT_ELEMENTWISE, st);
  widen_minplus_kernel<<<rows_grid(n, m, 256), 256, 0, st>>>(static_cast<const uint32_t*>(r), ldr, c, ldc, n, m,
                                                              inf_encoded);
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
}

int launch_widen_u32_i64(cudaStream_t st, const void* r, int64_t ldr, int64_t* c, int64_t ldc, int64_t n,
                         int64_t m) {
  if (n <= 0 || m <= 0) return PACO_OK;
  KernelSpan ks(PACO_KT_ELEMENTWISE, st);
  widen_u32_i64_kernel<<<rows_grid(n, m, 256), 256, 0, st>>>(static_cast<const uint32_t*>(r), ldr, c, ldc, n, m);
  PACO_CUDA_TRY(cudaGetLastError());
  return PACO_OK;
}

// ---------------------------------------------------------------------------
// ALU issue-rate probe (the roofline denominator for the non-tensor kernels).
// 32 independent accumulators per thread, 8 warps x 2 CTAs per SM; per-SM
// terms/clock from clock64 and the SM clock from %globaltimer.
// ---------------------------------------------------------------------------
template <int V>
__global__ void __launch_bounds__(256, 2) alu_probe_kernel(uint32_t* sink, long long* cyc, long long* ns,
                                                           int iters, uint32_t seed) {
  constexpr int N = 32;
  uint32_t acc[N], x[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    acc[i] = seed * (i + 3) + threadIdx.x;
    x[i] = seed ^ (i * 977u + threadIdx.x);
  }
  uint32_t y = seed + threadIdx.x;
  __syncthreads();
  long long t0 = clock64(), g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  double dacc[V == 3 ? N : 1];
#pragma unroll
  for (int i = 0; i < (V == 3 ? N : 1); ++i) dacc[i] = double(acc[i]) * 1e-9;
  const double dy = 1.0 + 1e-12 * double(y);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (V == 0) acc[i] = min(acc[i], x[i] + y);
      if (V == 1) acc[i] = uint32_t(max(int(acc[i]), int(x[i] + y)));
      if (V == 2) acc[i] = __float_as_uint(fmaf(__uint_as_float(x[i]), __uint_as_float(y), __uint_as_float(acc[i])));
      if (V == 3) dacc[i] = fma(dacc[i], dy, 1e-7);
    }
    y += 0x9e3779b9u;
  }
  if (V == 3) {
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] ^= uint32_t(__double_as_longlong(dacc[i]));
  }
  long long t1 = clock64(), g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) s ^= acc[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = t1 - t0;
    ns[blockIdx.x] = g1 - g0;
  }
}

int run_alu_probe(cudaStream_t st, int which, int iters, double* tpc, double* mhz) {
  if (which < 0 || which > 3) {
    set_error("paco_alu_probe: which=%d not in 0..3", which);
    return PACO_ERR_ARG;
  }
  const int blocks = kNumSMs * 2, threads = 256;
  uint32_t* sink;
  long long *cyc, *ns;
  PACO_CUDA_TRY(cudaMallocAsync(&sink, size_t(blocks) * threads * 4, st));
  PACO_CUDA_TRY(cudaMallocAsync(&cyc, blocks * 8, st));
  PACO_CUDA_TRY(cudaMallocAsync(&ns, blocks * 8, st));
  if (which == 0) alu_probe_kernel<0><<<blocks, threads, 0, st>>>(sink, cyc, ns, iters, 7);
  if (which == 1) alu_probe_kernel<1><<<blocks, threads, 0, st>>>(sink, cyc, ns, iters, 7);
  if (which == 2) alu_probe_kernel<2><<<blocks, threads, 0, st>>>(sink, cyc, ns, iters, 7);
  if (which == 3) alu_probe_kernel<3><<<blocks, threads, 0, st>>>(sink, cyc, ns, iters, 7);
  PACO_CUDA_TRY(cudaGetLastError());
  long long hc[kNumSMs * 2], hn[kNumSMs * 2];
  PACO_CUDA_TRY(cudaMemcpyAsync(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost, st));
  PACO_CUDA_TRY(cudaMemcpyAsync(hn, ns, sizeof(hn), cudaMemcpyDeviceToHost, st));
  PACO_CUDA_TRY(cudaFreeAsync(sink, st));
  PACO_CUDA_TRY(cudaFreeAsync(cyc, st));
  PACO_CUDA_TRY(cudaFreeAsync(ns, st));
  PACO_CUDA_TRY(cudaStreamSynchronize(st));
  // two co-resident CTAs per SM: each CTA's loop saw the SM shared with its twin
  long long mx = 0;
  double mhz_sum = 0;
  for (int b = 0; b < blocks; ++b) {
    mx = hc[b] > mx ? hc[b] : mx;
    mhz_sum += double(hc[b]) / double(hn[b] > 0 ? hn[b] : 1) * 1e3;
  }
  const double terms_per_sm = double(iters) * 32 * threads * 2;
  *tpc = terms_per_sm / double(mx);
  *mhz = mhz_sum / blocks;
  return PACO_OK;
}

}  // namespace paco
