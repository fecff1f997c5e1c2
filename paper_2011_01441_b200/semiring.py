"""Semirings of the hot path and their sm_100a kernel bindings.

The reference bundles ``(name, dtype, zero, block_mm, vadd)`` per semiring
(/root/reference/pkg/src/paco/matmul.py:34-57).  Here ``block_mm`` and
``vadd`` are device operations (``paco_mm`` / ``paco_fold``) instead of
NumPy calls; ``dtype`` and ``zero`` keep the reference's meaning (element type
of C and the fill value of temporaries).

Reference semirings, same semantics bit for bit:

* ``SEMIRING_INT``      int64 (+,x), two's-complement wrap (matmul.py:53)
* ``SEMIRING_F64``      float64 (+,x)                        (matmul.py:54)
* ``SEMIRING_MINPLUS``  int64 (min,+), zero 2^62, wrapping add (matmul.py:29,55)

B200-native additions for the BASELINE configs:

* ``SEMIRING_MINPLUS_SAT`` (min,+) on int32 lanes, domain [0, 2^30],
  INF = 2^30, saturating (cfg2).  Equals the reference (min,+) followed by
  ``min(C, 2^30)`` on that domain.
* ``SEMIRING_MAXPLUS``   (max,+) on int32 lanes, domain [-2^30, 2^30),
  -INF = -2^30, saturating (cfg4).  Equals ``-minplus(-A, -B)`` of the
  reference on that domain.
* ``SEMIRING_F32``       float32 (+,x) on the tensor cores as 3xTF32 (hi/lo split,
  ~fp32 accuracy; Strassen leaves, cfg5).  ``SEMIRING_F32_SIMT`` is the FFMA
  (CUDA-core) kernel of the same semiring.
* ``SEMIRING_BF16``      bf16 inputs, float32 accumulate and C, tcgen05 (cfg3).
"""

from __future__ import annotations

import numpy as np

from . import _native as nat

MINPLUS_INF = np.int64(2**62)
TROPICAL_INF = 2**30


class Semiring:
    """Element algebra plus the device kernels that implement it."""

    def __init__(self, name: str, dtype, zero, kernel_id: int, in_dtype=None, *,
                 narrow_kernel_id: int | None = None, narrow_in_dtype=None):
        self.name = name
        self.dtype = np.dtype(dtype) if dtype != "bfloat16" else dtype
        self.zero = zero
        self.kernel_id = kernel_id
        self.in_dtype = in_dtype if in_dtype is not None else self.dtype
        # int32 operands of the int64 ring run the i32 x i32 -> i64 kernel
        self.narrow_kernel_id = narrow_kernel_id
        self.narrow_in_dtype = narrow_in_dtype

    def __repr__(self) -> str:
        return f"Semiring({self.name!r})"

    def block_mm(self, C, A, B) -> None:
        """C <- C (+) A (x) B in place (device or host arrays)."""
        from .mm import mm_seq

        mm_seq(A, B, C, self)

    def vadd(self, x, y):
        """Elementwise (+) into a new array (device fold kernel)."""
        from .mm import semiring_vadd

        return semiring_vadd(self, x, y)


SEMIRING_INT = Semiring("int", np.int64, np.int64(0), nat.SR_INT_I64,
                        narrow_kernel_id=nat.SR_INT_I32_I64, narrow_in_dtype=np.dtype(np.int32))
SEMIRING_F64 = Semiring("f64", np.float64, 0.0, nat.SR_F64)
SEMIRING_MINPLUS = Semiring("minplus", np.int64, MINPLUS_INF, nat.SR_MINPLUS_I64)

SEMIRING_MINPLUS_SAT = Semiring("minplus_sat", np.int32, np.int32(TROPICAL_INF), nat.SR_MINPLUS_SAT32)
SEMIRING_MAXPLUS = Semiring("maxplus", np.int32, np.int32(-TROPICAL_INF), nat.SR_MAXPLUS_SAT32)
SEMIRING_F32 = Semiring("f32", np.float32, np.float32(0.0), nat.SR_F32_TC)
SEMIRING_F32_SIMT = Semiring("f32_simt", np.float32, np.float32(0.0), nat.SR_F32)
SEMIRING_BF16 = Semiring("bf16", np.float32, np.float32(0.0), nat.SR_BF16_F32, in_dtype="bfloat16")

# internal: SEMIRING_MINPLUS's image on u32 lanes (operands range-checked into
# [0, 2^31), no clamp; mm.py narrows to it and widens the result back)
SEMIRING_MINPLUS_U32 = Semiring("minplus_u32", np.uint32, np.uint32(0xFFFFFFFF), nat.SR_MINPLUS_U32)

# reference registry (matmul.py:57) plus the B200 additions
SEMIRINGS = {s.name: s for s in (SEMIRING_INT, SEMIRING_F64, SEMIRING_MINPLUS)}
ALL_SEMIRINGS = dict(SEMIRINGS, **{s.name: s for s in (
    SEMIRING_MINPLUS_SAT, SEMIRING_MAXPLUS, SEMIRING_F32, SEMIRING_F32_SIMT, SEMIRING_BF16)})
