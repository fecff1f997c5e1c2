"""ctypes binding of libpaco_b200.so (the C ABI in include/paco_b200.h).

The library is built in-tree by ``__graft_entry__.build()``.  There is no
fallback: if the shared object is missing every compute entry point raises.
ctypes releases the GIL for the duration of each call, so the per-worker
threads of ``execute_plan(mode="parallel")`` enqueue concurrently.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .plan import PlanError

LIB_PATH = os.environ.get("PACO_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpaco_b200.so")

# semiring ids (include/paco_b200.h)
SR_INT_I64 = 0
SR_INT_I32_I64 = 1
SR_F64 = 2
SR_MINPLUS_I64 = 3
SR_MINPLUS_SAT32 = 4
SR_MAXPLUS_SAT32 = 5
SR_F32 = 6
SR_BF16_F32 = 7
SR_F32_TC = 8
SR_MINPLUS_U32 = 9
SR_COUNT = 10

DT_F32, DT_F64, DT_I64 = 0, 1, 2

# kernel families of paco_kernel_timing_read
KT_SIMT_MM, KT_TC_GEMM, KT_TF32_SPLIT, KT_LINCOMB, KT_ELEMENTWISE = 0, 1, 2, 3, 4

MM_OVERWRITE = 1
MM_ATOMIC = 2
MM_REMOTE = 4
MM_PACO_PLAN = 8
MM_SYS = 16
FOLD_RESET = 1
FOLD_ATOMIC = 2
TROPICAL_INF = 1 << 30
MAX_PIECES = 640

OK, ERR_ARG, ERR_CUDA, ERR_UNSUPPORTED = 0, -1, -2, -3

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_int = ctypes.c_int

# name -> (restype, argtypes); every symbol the header declares
SIGNATURES = {
    "paco_mm": (_int, [_int, _vp, _int, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _i64,
                       ctypes.POINTER(ctypes.c_int32), _int, _int]),
    "paco_mm_tile_shape": (_int, [_int] + [ctypes.POINTER(_int)] * 4),
    "paco_plan_one_piece": (_int, [_i64, _i64, _i64, _int, ctypes.POINTER(_i64)]),
    "paco_plan_cta": (_int, [_int, _i64, _i64, _i64, _int, ctypes.POINTER(ctypes.c_int32)]),
    "paco_cta_grid": (_int, [_int, _i64, _i64, _i64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_i64)]),
    "paco_cta_grid_tail": (_int, [_int, _i64, _i64, _i64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_i64)]),
    "paco_fold": (_int, [_int, _vp, _int, _vp, _i64, _vp, _i64, _i64, _i64, _int]),
    "paco_fill": (_int, [_int, _vp, _int, _vp, _i64, _i64, _i64]),
    "paco_mm_naive": (_int, [_int, _vp, _int, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _i64]),
    "paco_lincomb": (_int, [_int, _vp, _int, _vp, _i64, _i64, _i64, _int,
                            ctypes.POINTER(_vp), ctypes.POINTER(_i64),
                            ctypes.POINTER(ctypes.c_int32), _int]),
    "paco_lincomb_multi": (_int, [_int, _vp, _i64, _i64, _int, ctypes.POINTER(_vp), ctypes.POINTER(_i64), _int,
                                  ctypes.POINTER(_vp), ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_int32)]),
    "paco_mm_batch": (_int, [_int, _vp, _int, _int, ctypes.c_void_p]),
    "paco_tf32_split": (_int, [_int, _vp, _int, ctypes.POINTER(_vp), ctypes.POINTER(_i64),
                               ctypes.POINTER(ctypes.c_int32), _i64, _i64, _int, _vp, _vp, _i64]),
    "paco_mm_tf32x3": (_int, [_int, _vp, _int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64,
                              ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64, ctypes.POINTER(_vp), _i64, _i64,
                              _i64, _i64, _int]),
    "paco_mm_tf32x3_multi": (_int, [_int, _vp, _int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64,
                                    ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64, ctypes.POINTER(ctypes.c_int32),
                                    ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_int32), _i64, _i64, _i64, _i64]),
    "paco_narrow_i64": (_int, [_int, _vp, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _int, _vp]),
    "paco_widen_u32_i64": (_int, [_int, _vp, _vp, _i64, _vp, _i64, _i64, _i64]),
    "paco_narrow_minplus_inf": (_int, [_int, _vp, _vp, _i64, _vp, _i64, _i64, _i64, _vp]),
    "paco_widen_minplus_i64": (_int, [_int, _vp, _vp, _i64, _vp, _i64, _i64, _i64, _int]),
    "paco_host_copy2d": (_int, [_vp, _i64, _vp, _i64, _i64, _i64, _int]),
    "paco_mm_tf32x3_fused": (_int, [_int, _vp, _int, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(_vp),
                                    ctypes.POINTER(ctypes.c_int32), _i64, ctypes.POINTER(ctypes.c_int32),
                                    ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_int32), _i64,
                                    ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_int32),
                                    _i64, _i64, _i64, _i64]),
    "paco_mm_tf32x3_fused_a": (_int, [_int, _vp, _int, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(_vp),
                                      ctypes.POINTER(ctypes.c_int32), _i64, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                      _i64, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(_vp),
                                      ctypes.POINTER(ctypes.c_int32), _i64, _i64, _i64, _i64]),
    "paco_tf32b2_split": (_int, [_int, _vp, _int, ctypes.POINTER(_vp), ctypes.POINTER(_i64),
                                 ctypes.POINTER(ctypes.c_int32), _i64, _i64, _int, _vp, _vp, _vp, _i64]),
    "paco_mm_tf32b2_multi": (_int, [_int, _vp, _int] + [ctypes.POINTER(_vp)] * 3 + [_i64] +
                             [ctypes.POINTER(_vp)] * 3 + [_i64, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(_vp),
                                                          ctypes.POINTER(ctypes.c_int32), _i64, _i64, _i64, _i64]),
    "paco_lincomb_split": (_int, [_int, _vp, _i64, _i64, _int, ctypes.POINTER(_vp), ctypes.POINTER(_i64), _int,
                                  ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_i64),
                                  ctypes.POINTER(ctypes.c_int32)]),
    "paco_mm_bf16x3_multi": (_int, [_int, _vp, _int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64,
                                    ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64, ctypes.POINTER(ctypes.c_int32),
                                    ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_int32), _i64, _i64, _i64, _i64]),
    "paco_strassen_split49": (_int, [_int, _vp, _int, _vp, _i64, _i64, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                     _i64]),
    "paco_mm_bf16x3_multi_bn": (_int, [_int, _vp, _int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64,
                                       ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64, ctypes.POINTER(ctypes.c_int32),
                                       ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_int32), _i64, _i64, _i64, _i64]),
    "paco_transpose": (_int, [_int, _vp, _int, _vp, _i64, _vp, _i64, _i64, _i64]),
    "paco_copy2d": (_int, [_int, _vp, _vp, _i64, _vp, _i64, _i64, _i64]),
    "paco_host_register": (_int, [_vp, ctypes.c_size_t]),
    "paco_host_unregister": (_int, [_vp]),
    "paco_device_alloc": (_int, [_int, ctypes.c_size_t, ctypes.POINTER(_vp)]),
    "paco_device_free": (_int, [_int, _vp]),
    "paco_ipc_handle": (_int, [_int, _vp, _vp]),
    "paco_ipc_open": (_int, [_int, _vp, ctypes.POINTER(_vp)]),
    "paco_ipc_close": (_int, [_int, _vp]),
    "paco_enable_peer": (_int, [_int, _int]),
    "paco_alu_probe": (_int, [_int, _vp, _int, _int, ctypes.POINTER(ctypes.c_double),
                              ctypes.POINTER(ctypes.c_double)]),
    "paco_debug_trace": (_int, [_vp]),
    "paco_kernel_timing": (_int, [_int]),
    "paco_kernel_timing_read": (_int, [_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64)]),
    "paco_last_error": (ctypes.c_char_p, []),
    "paco_abi_version": (_int, []),
}

_lock = threading.Lock()
_lib = None


class NativeError(RuntimeError):
    """CUDA-side failure reported by the C ABI."""


def load() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeError(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                    " -- there is no CPU fallback")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.paco_abi_version() != 1:
                raise NativeError("libpaco_b200.so ABI version mismatch; rebuild")
            _lib = lib
    return _lib


def check(rc: int) -> None:
    """Map C status codes to the reference's exception types."""
    if rc == OK:
        return
    msg = load().paco_last_error().decode(errors="replace")
    if rc == ERR_ARG:
        raise PlanError(msg) if "piece" in msg or "worker" in msg else ValueError(msg)
    if rc == ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise NativeError(msg)


def tile_shape(sr: int) -> tuple[int, int, int, int]:
    vals = [_int() for _ in range(4)]
    check(load().paco_mm_tile_shape(sr, *[ctypes.byref(v) for v in vals]))
    return tuple(v.value for v in vals)


def plan_one_piece(n: int, m: int, k: int, p: int) -> list[tuple[int, ...]]:
    """Native MM-1-Piece geometry: p rows of (i0, j0, l0, n, m, k)."""
    buf = (_i64 * (6 * p))()
    check(load().paco_plan_one_piece(n, m, k, p, buf))
    return [tuple(buf[6 * i:6 * i + 6]) for i in range(p)]


class MMProblem(ctypes.Structure):
    """``paco_mm_problem`` of include/paco_b200.h."""

    _fields_ = [("A", ctypes.c_void_p), ("lda", ctypes.c_int64), ("B", ctypes.c_void_p), ("ldb", ctypes.c_int64),
                ("C", ctypes.c_void_p), ("ldc", ctypes.c_int64), ("n", ctypes.c_int64), ("m", ctypes.c_int64),
                ("k", ctypes.c_int64), ("flags", ctypes.c_int32)]


MAX_BATCH = 64


def mm_batch(device: int, stream: int, sr: int, problems: list) -> None:
    """One paco_mm_batch launch per MAX_BATCH problems; each problem is
    (A_ptr, lda, B_ptr, ldb, C_ptr, ldc, n, m, k, flags)."""
    lib = load()
    for i in range(0, len(problems), MAX_BATCH):
        chunk = problems[i:i + MAX_BATCH]
        arr = (MMProblem * len(chunk))(*[MMProblem(*p) for p in chunk])
        check(lib.paco_mm_batch(device, stream, sr, len(chunk), ctypes.cast(arr, ctypes.c_void_p)))


def cta_grid(sr: int, n: int, m: int, k: int) -> tuple[int, int]:
    """(k split, CTA count) of paco_mm's default tile-grid plan."""
    s, ctas = ctypes.c_int(), _i64()
    check(load().paco_cta_grid(sr, n, m, k, ctypes.byref(s), ctypes.byref(ctas)))
    return s.value, ctas.value


GRID_BAND = 8  # cta_plan.cuh kGridBand


def grid_pieces(sr: int, n: int, m: int, k: int) -> list[tuple[int, ...]]:
    """The default tile-grid plan as (ti0, tj0, tl0, tn, tm, tk) rows, CTA order
    (C tiles in row-block bands of GRID_BAND, column by column inside a band;
    the partial last SM-wave's tiles split ``paco_cta_grid_tail`` ways in k)."""
    bm, bn, kq, _ = tile_shape(sr)
    s, ctas = cta_grid(sr, n, m, k)
    tail, head = ctypes.c_int(), _i64()
    check(load().paco_cta_grid_tail(sr, n, m, k, ctypes.byref(tail), ctypes.byref(head)))
    tail, head = tail.value, head.value
    tn_, tm_, ku = -(-n // bm), -(-m // bn), -(-k // kq)
    out = []
    for idx in range(ctas):
        if tail > 1 and idx >= head:
            tile, part = head + (idx - head) // tail, (idx - head) % tail
            s = tail
        else:
            tile, part = divmod(idx, s)
        r0 = (tile // (GRID_BAND * tm_)) * GRID_BAND
        rows = min(GRID_BAND, tn_ - r0)
        v = tile - r0 * tm_
        l0 = part * ku // s
        out.append((r0 + v % rows, v // rows, l0, 1, 1, (part + 1) * ku // s - l0))
    return out


def plan_cta(sr: int, n: int, m: int, k: int, p: int) -> list[tuple[int, ...]]:
    """The library's default CTA-level plan: p rows of (ti0, tj0, tl0, tn, tm, tk)."""
    buf = (ctypes.c_int32 * (6 * p))()
    check(load().paco_plan_cta(sr, n, m, k, p, buf))
    return [tuple(buf[6 * i:6 * i + 6]) for i in range(p)]


def pieces_array(pieces):
    """Flatten [(ti0, tj0, tl0, tn, tm, tk), ...] into a ctypes int32 array."""
    if not pieces:
        return None, 0
    if len(pieces) > MAX_PIECES:
        raise PlanError(f"{len(pieces)} CTA pieces exceed PACO_MAX_PIECES={MAX_PIECES}")
    flat = [int(v) for pc in pieces for v in pc]
    return (ctypes.c_int32 * len(flat))(*flat), len(pieces)


class kernel_timing:
    """Context manager: live CUDA-event timing of the library's own launches.

    ``with kernel_timing() as kt: ...`` then ``kt.read(KT_TC_GEMM)`` ->
    (summed ms, launches) of that kernel family inside the block."""

    def __enter__(self):
        check(load().paco_kernel_timing(1))
        return self

    def __exit__(self, *exc):
        check(load().paco_kernel_timing(0))

    @staticmethod
    def read(family: int) -> tuple[float, int]:
        ms, cnt = ctypes.c_double(), _i64()
        check(load().paco_kernel_timing_read(family, ctypes.byref(ms), ctypes.byref(cnt)))
        return ms.value, cnt.value
