"""ctypes front of oracle/semiring_ref.c -- TEST INFRASTRUCTURE ONLY.

``mm(sr, A, B, C)`` computes C (+)= A (x) B on the host with the plain-C
restatement of the reference's defining sums (matmul.py:400-414), in place,
for C-contiguous NumPy arrays.  OpenMP uses every host core unless
``threads`` is given.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

SR_INT_I64, SR_INT_I32_I64, SR_F64, SR_MINPLUS_I64 = 0, 1, 2, 3
SR_MINPLUS_SAT32, SR_MAXPLUS_SAT32, SR_F32 = 4, 5, 6

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "build", "liboracle.so")
_lib = None

_IN = {SR_INT_I64: np.int64, SR_INT_I32_I64: np.int32, SR_F64: np.float64, SR_MINPLUS_I64: np.int64,
       SR_MINPLUS_SAT32: np.int32, SR_MAXPLUS_SAT32: np.int32, SR_F32: np.float32}
_OUT = {SR_INT_I64: np.int64, SR_INT_I32_I64: np.int64, SR_F64: np.float64, SR_MINPLUS_I64: np.int64,
        SR_MINPLUS_SAT32: np.int32, SR_MAXPLUS_SAT32: np.int32, SR_F32: np.float32}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            import subprocess
            import sys
            root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
            subprocess.run([sys.executable, "-c",
                            "import __graft_entry__ as g; g.build_oracle()"], cwd=root, check=True)
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.oracle_mm_rows_simple.restype = ctypes.c_int
        _lib.oracle_mm_rows_simple.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                               ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                               ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
        _lib.oracle_mm_rows.restype = ctypes.c_int
        _lib.oracle_mm_rows.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                        ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
    return _lib


def mm(sr: int, A: np.ndarray, B: np.ndarray, C: np.ndarray, threads: int | None = None,
       simple: bool = False) -> np.ndarray:
    """C (+)= A (x) B in place; ``simple`` forces the plain loop (no cache blocking)."""
    n, k = A.shape
    k2, m = B.shape
    assert k == k2 and C.shape == (n, m), (A.shape, B.shape, C.shape)
    A = np.ascontiguousarray(A, dtype=_IN[sr])
    B = np.ascontiguousarray(B, dtype=_IN[sr])
    assert C.dtype == _OUT[sr] and C.flags["C_CONTIGUOUS"], (C.dtype, C.flags)
    if threads is not None:
        os.environ["OMP_NUM_THREADS"] = str(threads)
    fn = lib().oracle_mm_rows_simple if simple else lib().oracle_mm_rows
    rc = fn(sr, A.ctypes.data, A.strides[0] // A.itemsize, B.ctypes.data,
                              B.strides[0] // B.itemsize, C.ctypes.data, C.strides[0] // C.itemsize,
                              n, m, k, 0, n)
    assert rc == 0, f"oracle rc={rc}"
    return C


def mm_rows(sr: int, A: np.ndarray, B: np.ndarray, C_rows: np.ndarray, rows) -> np.ndarray:
    """Oracle rows ``rows`` of C (+)= A (x) B into ``C_rows`` (len(rows) x m)."""
    return mm(sr, np.ascontiguousarray(A[np.asarray(rows)]), B, C_rows)
