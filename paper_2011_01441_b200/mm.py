"""Semiring MM entry points with the reference's signatures, run on B200.

* ``mm_seq``      -- matmul.py:342-366: C <- C (+) A (x) B on one device.  The
  reference recursion (halve the longest axis down to 32^3 NumPy leaves,
  matmul.py:369-397) is replaced by one sm_100a launch whose CTAs each own a
  piece of the CTA-level plan (default: one C tile per CTA with a cost-model
  k split; the balanced PACO cuboid plan on request, PACO_MM_PACO_PLAN).
  Pinned host operands are streamed through a k-first / rows-last
  H2D-compute-D2H pipeline.
* ``mm_execute``  -- matmul.py:417-462: binds a plan to device work.  COMPUTE
  tasks launch ``paco_mm`` on sub-views; REDUCE tasks launch ``paco_fold``
  (t (+)= temp; temp = zero).  Plan workers map to (device, stream) pairs.
* ``mm_oracle``   -- matmul.py:400-414: defining sums, one thread per element.

Inputs may be NumPy arrays (staged to the device and C written back in place,
as the reference mutates C) or CUDA tensors (used in place).
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _native as nat
from .cuboid import DEFAULT_BASE, Cuboid, temp_shape
from .device import Output, View, is_host, pick_device, stage_in, torch_dtype
from .engine import execute_plan
from .plan import COMPUTE, REDUCE, CostReport, Plan, PlanError
from .semiring import SEMIRING_INT, SEMIRING_MINPLUS, SEMIRING_MINPLUS_U32, Semiring


def _dtype_of(x):
    if isinstance(x, np.ndarray):
        return x.dtype
    if isinstance(x, torch.Tensor):
        return x.dtype
    raise TypeError(f"unsupported array type {type(x).__name__}")


def _is_i32(x) -> bool:
    dt = _dtype_of(x)
    return dt == np.int32 or dt == torch.int32


def kernel_for(semiring: Semiring, A, B) -> tuple[int, object]:
    """(kernel id, operand dtype) for this semiring and these operands."""
    if semiring.narrow_kernel_id is not None and _is_i32(A) and _is_i32(B):
        return semiring.narrow_kernel_id, semiring.narrow_in_dtype
    return semiring.kernel_id, semiring.in_dtype


# --- the reference's own int64 semirings on 32-bit kernels ----------------------
# SEMIRING_INT and SEMIRING_MINPLUS keep int64 storage (matmul.py:45-55), but a
# 64-bit add+min or multiply-add is 4-6 ALU instructions per term.  When every
# operand fits 32 bits the product is computed on 32-bit lanes with the same
# result bit for bit: (+,x) on int32 x int32 -> int64 (IMAD.WIDE, wrapping
# int64 accumulation, as NumPy's); (min,+) on u32 lanes, either with the INF
# sentinel kept exact (paco_narrow_minplus_inf: finite operands in [0, 2^30 - 2]
# and INF = 2^62, whose sums -- including the reference's INF + INF wrap to
# -2^63 -- map to an order-preserving u32 code) or, failing that, for operands
# in [0, 2^31) (a + b <= 2^32 - 2: no wrap).  The product is formed from the
# semiring zero and min-ed into the int64 C by paco_widen_minplus_i64.  The
# range checks run on the device while narrowing; any other value (negatives,
# big finite values next to INF) keeps the int64 kernel.
NARROW_MIN_TERMS = 1 << 22   # below this the 64-bit kernel is cheaper than a narrowing pass + flag read
_NARROW_RANGE = {"int": (-(2**31), 2**31 - 1), "minplus": (0, 2**31 - 1)}


def _is_i64(x) -> bool:
    dt = _dtype_of(x)
    return dt == np.int64 or dt == torch.int64


def _narrowable(semiring: Semiring, A, B, C, n: int, m: int, k: int) -> bool:
    return (semiring in (SEMIRING_INT, SEMIRING_MINPLUS) and _is_i64(A) and _is_i64(B) and _is_i64(C)
            and float(n) * m * k >= NARROW_MIN_TERMS)


def _narrow_dev(x: torch.Tensor, lo: int, hi: int, saturate: bool, flag: torch.Tensor, st) -> torch.Tensor:
    """int32 image of a device int64 matrix (paco_narrow_i64); range misses set ``flag``."""
    out = torch.empty(tuple(x.shape), dtype=torch.int32, device=x.device)
    xv, ov = View.of(x), View.of(out)
    nat.check(nat.load().paco_narrow_i64(xv.device, st.cuda_stream, xv.ptr, xv.ld, ov.ptr, ov.ld, xv.rows, xv.cols,
                                         lo, hi, int(saturate), flag.data_ptr()))
    return out


def _narrow_inf(x: torch.Tensor, flag: torch.Tensor, st) -> torch.Tensor:
    """u32 code of a SEMIRING_MINPLUS operand with INF kept (paco_narrow_minplus_inf)."""
    out = torch.empty(tuple(x.shape), dtype=torch.int32, device=x.device)
    xv, ov = View.of(x), View.of(out)
    nat.check(nat.load().paco_narrow_minplus_inf(xv.device, st.cuda_stream, xv.ptr, xv.ld, ov.ptr, ov.ld, xv.rows,
                                                 xv.cols, flag.data_ptr()))
    return out


class _Narrowed:
    """Device operands of a narrowed product and how to put C back (int64)."""

    def __init__(self, semiring: Semiring, A, B, C, dev: int, st, overwrite: bool):
        self.a64 = stage_in(A, np.int64, dev)
        self.b64 = stage_in(B, np.int64, dev)
        self.out = Output(C, np.int64, dev, load=not overwrite)
        if overwrite:
            launch_fill(semiring.kernel_id, st, View.of(self.out.dev))
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.minplus = semiring is SEMIRING_MINPLUS
        self.inf = False
        self.r = None
        if self.minplus:
            # INF-keeping code first (distance matrices hold the 2^62 sentinel);
            # plain [0, 2^31) operands without INF as the second try
            self.a32 = _narrow_inf(self.a64, flag, st)
            self.b32 = _narrow_inf(self.b64, flag, st)
            self.inf = int(flag.item()) == 0
            if not self.inf:
                flag.zero_()
                lo, hi = _NARROW_RANGE["minplus"]
                self.a32 = _narrow_dev(self.a64, lo, hi, False, flag, st)
                self.b32 = _narrow_dev(self.b64, lo, hi, False, flag, st)
            # the product from the u32 zero, min-ed into the int64 C by finish()
            self.r = torch.empty(tuple(self.out.dev.shape), dtype=torch.int32, device=dev)
            launch_fill(nat.SR_MINPLUS_U32, st, View.of(self.r))
        else:
            lo, hi = _NARROW_RANGE["int"]
            self.a32 = _narrow_dev(self.a64, lo, hi, False, flag, st)
            self.b32 = _narrow_dev(self.b64, lo, hi, False, flag, st)
        self.ok = self.inf or int(flag.item()) == 0   # one 4-byte read: the range verdict

    @property
    def semiring(self) -> Semiring:
        return SEMIRING_MINPLUS_U32 if self.minplus else SEMIRING_INT

    @property
    def c(self) -> torch.Tensor:
        return self.r if self.minplus else self.out.dev

    def finish(self, st) -> None:
        if self.minplus:
            r, c = View.of(self.r), View.of(self.out.dev)
            nat.check(nat.load().paco_widen_minplus_i64(c.device, st.cuda_stream, r.ptr, r.ld, c.ptr, c.ld, c.rows,
                                                        c.cols, int(self.inf)))
        self.out.finish()


def launch_mm(kid: int, stream: torch.cuda.Stream, a: View, b: View, c: View, *,
              pieces=None, overwrite: bool = False, flags: int = 0, device: int | None = None) -> None:
    """One ``paco_mm`` call on views (no validation beyond the C ABI's).

    ``device`` is the GPU that runs the kernel (default: C's device; differs
    when C is peer memory, with ``flags`` carrying MM_REMOTE)."""
    arr, npieces = nat.pieces_array(pieces)
    nat.check(nat.load().paco_mm(
        c.device if device is None else device, stream.cuda_stream, kid, a.ptr, a.ld, b.ptr, b.ld,
        c.ptr, c.ld, c.rows, c.cols, a.cols, arr, npieces, flags | (nat.MM_OVERWRITE if overwrite else 0)))


def launch_fold(kid: int, stream: torch.cuda.Stream, dst: View, src: View, reset: bool, *,
                atomic: bool = False) -> None:
    """dst (+)= src (paco_fold); ``reset``: src = zero afterwards; ``atomic``: per-element
    atomics, safe while other kernels fold into dst."""
    flags = (nat.FOLD_RESET if reset else 0) | (nat.FOLD_ATOMIC if atomic else 0)
    nat.check(nat.load().paco_fold(dst.device, stream.cuda_stream, kid, dst.ptr, dst.ld,
                                   src.ptr, src.ld, dst.rows, dst.cols, flags))


def launch_fill(kid: int, stream: torch.cuda.Stream, dst: View) -> None:
    nat.check(nat.load().paco_fill(dst.device, stream.cuda_stream, kid, dst.ptr, dst.ld,
                                   dst.rows, dst.cols))


def _shape_check(A, B, C) -> tuple[int, int, int]:
    n, k = tuple(A.shape)
    k2, m = tuple(B.shape)
    if k != k2 or tuple(C.shape) != (n, m):
        raise ValueError(f"shape mismatch: A{tuple(A.shape)} B{tuple(B.shape)} C{tuple(C.shape)}")
    return n, m, k


def mm_seq(A, B, C, semiring: Semiring = SEMIRING_INT, base: int = DEFAULT_BASE, sim=None,
           ids: tuple[int, int, int] = (100, 101, 0), *, stream: torch.cuda.Stream | None = None,
           pieces=None, overwrite: bool = False, _narrow: bool = True) -> None:
    """C <- C (+) A (x) B on one B200 (matmul.py:342-366).

    ``base`` is accepted for signature compatibility: the leaf size of the
    reference recursion has no role once the CTA-level plan tiles the cuboid.
    ``pieces`` overrides the CTA-level plan (tile-unit cuboids);
    ``overwrite`` declares C == zero so the kernel does not read it.
    """
    n, m, k = _shape_check(A, B, C)
    if sim is not None:
        raise NotImplementedError("cache simulation is out of scope on B200; use ncu counters")
    kid, in_dt = kernel_for(semiring, A, B)
    dev = pick_device(A, B, C)
    with torch.cuda.device(dev):
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        if _narrow and _narrowable(semiring, A, B, C, n, m, k):
            with torch.cuda.stream(st):
                nw = _Narrowed(semiring, A, B, C, dev, st, overwrite)
                if nw.ok:
                    mm_seq(nw.a32, nw.b32, nw.c, nw.semiring, stream=st, pieces=pieces)
                else:  # some operand needs 64 bits: the int64 kernel on the staged operands
                    mm_seq(nw.a64, nw.b64, nw.out.dev, semiring, stream=st, pieces=pieces, _narrow=False)
                    nw.minplus = False
                nw.finish(st)
            return
        pinned = _pinned_host(A, in_dt) and _pinned_host(B, in_dt) and _pinned_host(C, semiring.dtype)
        if pieces is None and n >= 2 * _PIPE_MIN_ROWS and (pinned or (
                _numpy_host(A, in_dt) and _numpy_host(B, in_dt) and _numpy_host(C, semiring.dtype))):
            if k >= 4 * _PIPE_MIN_K:
                _kphased_host_mm(A, B, C, kid, dev, st, overwrite)
            elif pinned:
                _pipelined_host_mm(A, B, C, kid, semiring, dev, st, overwrite)
            else:
                _kphased_host_mm(A, B, C, kid, dev, st, overwrite, front_share=0.0)
            return
        with torch.cuda.stream(st):
            a = View.of(stage_in(A, in_dt, dev))
            b = View.of(stage_in(B, in_dt, dev))
            out = Output(C, semiring.dtype, dev, load=not overwrite)
            launch_mm(kid, st, a, b, View.of(out.dev), pieces=pieces, overwrite=overwrite)
            out.finish()


_PIPE_MIN_ROWS = 512
_PIPE_GRID = (4, 2)  # 2-D block grid for short k: measured best of 4x4/8x1/4x2/2x4/8x2 for 8192^3
_PIPE_MIN_K = 512
# k-phased schedule: first k chunk, growth factor, chunk cap, share of k in the
# row-blocked last phase, and its number of row blocks (tools/kp_sweep.py:
# within 0.3 % of the best of eight shapes on 8192^3)
_KP = (128, 2, 2048, 0.25, 16)
# staged (pageable NumPy) operands: every chunk costs a host copy before its
# DMA, so the chunks grow more slowly (growth <= compute rate / staging rate
# keeps the GPU fed) and each chunk's staging is cut into ~8 MiB row parts whose
# DMAs start while the next part is being copied
_KP_STAGED = (128, 1.5, 2048, 0.25, 16)
# last-phase row blocks: None = _KP[4] uniform blocks, else geometric decay toward the end
# (cfg2 end to end from NumPy: 32.02 ms at 0.6, 32.04-32.06 at 0.7, 32.21-32.24 uniform;
# tools/e2e_rows_ab.py)
_ROW_DECAY = 0.6
_ROW_CAP = 2048
_STAGE_PART_BYTES = 8 << 20


def _pinned_host(x, dtype) -> bool:
    return (isinstance(x, torch.Tensor) and not x.is_cuda and x.is_pinned() and x.is_contiguous()
            and x.dtype == torch_dtype(dtype))


def _numpy_host(x, dtype) -> bool:
    """A pageable NumPy matrix the pipeline can stage (unit column stride, exact dtype)."""
    return (isinstance(x, np.ndarray) and x.ndim == 2 and x.dtype == np.dtype(dtype) and x.dtype != object
            and (x.shape[1] <= 1 or x.strides[1] == x.itemsize) and x.dtype.itemsize in (4, 8))


# Participants of the native staging memcpy (paco_host_copy2d).  Measured on the
# 16-core GPU host (tools/e2e_numpy_timeline.py, cfg2 NumPy e2e): 4/6/8/12/16
# threads -> 53.7/42.5/36.6/33.9/34.1 ms per call
_HOST_THREADS = max(1, min(12, (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else 16) * 3 // 4))


def _host_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[...] = src for equal-shape 2-D row-major views (unit column stride),
    by the library's native parallel memcpy (paco_host_copy2d, GIL released)."""
    assert dst.shape == src.shape and dst.itemsize == src.itemsize, (dst.shape, src.shape)
    if dst.size == 0:
        return
    rows, cols = dst.shape
    nat.check(nat.load().paco_host_copy2d(dst.ctypes.data, dst.strides[0] if rows > 1 else cols * dst.itemsize,
                                          src.ctypes.data, src.strides[0] if rows > 1 else cols * src.itemsize,
                                          cols * dst.itemsize, rows, _HOST_THREADS))


# NumPy operands of the host pipeline are page-locked once and kept registered
# while their buffer lives (weakref.finalize unregisters before it is freed), so a
# caller that passes the same arrays again gets direct DMA instead of staging
REGISTER_HOST = True
_REGISTER_MIN_BYTES = 64 << 20
_registered: dict = {}   # base buffer address -> byte size


def _owner(x: np.ndarray) -> np.ndarray:
    while isinstance(x.base, np.ndarray):
        x = x.base
    return x


def _register_host(arrays) -> bool:
    """Page-lock the buffers behind these NumPy arrays (cached); False if the
    driver refuses (lock limits) -- the caller then stages through pinned copies."""
    import weakref

    if not REGISTER_HOST:
        return False
    lib = nat.load()
    for x in arrays:
        o = _owner(x)
        if o.base is not None or not o.flags["C_CONTIGUOUS"] and not o.flags["F_CONTIGUOUS"]:
            return False   # memory not owned by a NumPy array (e.g. a foreign buffer): do not pin it
        ptr, size = o.ctypes.data, o.nbytes
        if size < _REGISTER_MIN_BYTES:
            return False
        if _registered.get(ptr) == size:
            continue
        if lib.paco_host_register(ptr, size) != nat.OK:
            return False
        _registered[ptr] = size

        def _release(p=ptr):
            if _registered.pop(p, None) is not None:
                nat.load().paco_host_unregister(p)
        weakref.finalize(o, _release)
    return True


def _pinned_like(shape, dtype) -> torch.Tensor:
    """Pinned staging buffer (PyTorch's caching host allocator keeps it for the next call)."""
    return torch.empty(tuple(shape), dtype=torch_dtype(dtype), pin_memory=True)


def _copy2d(stream, dst: torch.Tensor, dr0: int, dc0: int, src: torch.Tensor, sr0: int, sc0: int,
            rows: int, cols: int) -> None:
    """Async 2-D block copy between row-major tensors (host pinned <-> device)."""
    es = dst.element_size()
    nat.check(nat.load().paco_copy2d(
        dst.device.index if dst.is_cuda else src.device.index, stream.cuda_stream,
        dst.data_ptr() + (dr0 * dst.stride(0) + dc0) * es, dst.stride(0) * es,
        src.data_ptr() + (sr0 * src.stride(0) + sc0) * es, src.stride(0) * es, cols * es, rows))


def _copy2d_raw(device: int, out: torch.Tensor, src_ptr: int, src_pitch: int) -> None:
    """out (contiguous, on ``device``) <- rows of raw device memory at src_ptr."""
    st = torch.cuda.current_stream(device)
    es = out.element_size()
    nat.check(nat.load().paco_copy2d(device, st.cuda_stream, out.data_ptr(), out.stride(0) * es, src_ptr,
                                     src_pitch, out.shape[1] * es, out.shape[0]))


def _pipelined_host_mm(A, B, C, kid: int, semiring: Semiring, dev: int, st, overwrite: bool) -> None:
    """Host (pinned) operands: overlap H2D, compute and D2H over a 2-D block grid.

    C is cut into R row blocks x J column blocks.  The H2D stream uploads B's
    column block j (needed by every row block), the row blocks of A on the
    first pass, and C's block (unless overwriting); the compute stream runs
    block (i, j) as soon as its inputs landed; the D2H stream returns C(i, j)
    while later blocks compute.  So only the first block's inputs and the last
    block's output are exposed.  The reference mutates C synchronously, so this
    returns after the last D2H.
    """
    n, k = tuple(A.shape)
    m = B.shape[1]
    R, J = _PIPE_GRID
    R = max(1, min(R, n // _PIPE_MIN_ROWS))
    J = max(1, min(J, m // _PIPE_MIN_ROWS))
    redges = [((n * i // R) // 128) * 128 for i in range(R)] + [n]
    cedges = [((m * j // J) // 128) * 128 for j in range(J)] + [m]
    h2d = torch.cuda.Stream(device=dev)
    d2h = torch.cuda.Stream(device=dev)
    h2d.wait_stream(st)
    a_d = torch.empty((n, k), dtype=A.dtype, device=dev)
    b_d = torch.empty((k, m), dtype=B.dtype, device=dev)
    c_d = torch.empty((n, m), dtype=C.dtype, device=dev)
    for t in (a_d, b_d, c_d):
        t.record_stream(h2d)
        t.record_stream(d2h)
    av, bv, cv = View.of(a_d), View.of(b_d), View.of(c_d)
    blocks = [(i, j) for j in range(J) for i in range(R)]
    landed = {}
    for (i, j) in blocks:
        r0, r1, c0, c1 = redges[i], redges[i + 1], cedges[j], cedges[j + 1]
        if i == 0:
            _copy2d(h2d, b_d, 0, c0, B, 0, c0, k, c1 - c0)
        if j == 0:
            _copy2d(h2d, a_d, r0, 0, A, r0, 0, r1 - r0, k)
        if not overwrite:
            _copy2d(h2d, c_d, r0, c0, C, r0, c0, r1 - r0, c1 - c0)
        ev = torch.cuda.Event()
        ev.record(h2d)
        landed[(i, j)] = ev
    for (i, j) in blocks:
        r0, r1, c0, c1 = redges[i], redges[i + 1], cedges[j], cedges[j + 1]
        if r1 <= r0 or c1 <= c0:
            continue
        st.wait_event(landed[(i, j)])
        launch_mm(kid, st, av.sub(r0, 0, r1 - r0, k), bv.sub(0, c0, k, c1 - c0),
                  cv.sub(r0, c0, r1 - r0, c1 - c0), overwrite=overwrite)
        done = torch.cuda.Event()
        done.record(st)
        d2h.wait_event(done)
        _copy2d(d2h, C, r0, c0, c_d, r0, c0, r1 - r0, c1 - c0)
    st.wait_stream(d2h)
    d2h.synchronize()


def _row_edges(n: int) -> list[int]:
    """Row blocks of the last phase.  Uniform: _KP[4] blocks.  Geometric
    (_ROW_DECAY): the blocks shrink by _ROW_DECAY toward the end, from at most
    _ROW_CAP rows down to 128, so block i's C download still hides behind block
    i + 1's compute while only the last, smallest download is exposed, with
    fewer, fuller launches at the front."""
    if _ROW_DECAY is None or n < 4 * 128:
        R = max(1, min(int(_KP[4]), n // _PIPE_MIN_ROWS))
        return [((n * i // R) // 128) * 128 for i in range(R)] + [n]
    n_al = n // 128 * 128  # blocks on tile boundaries; the last absorbs n % 128
    sizes, s_, tot = [], 128.0, 0
    while tot < n_al:
        b = min(n_al - tot, max(128, int(-(-s_ // 128)) * 128))
        sizes.append(b)
        tot += b
        s_ = min(float(_ROW_CAP), s_ / _ROW_DECAY)
    if len(sizes) > 1 and sizes[-1] < sizes[-2] // 2:  # fold a small remainder into the first block
        tail = sizes.pop()
        sizes[-1] += tail
    sizes[0] += n - n_al
    edges = [0]
    for b in reversed(sizes):
        edges.append(edges[-1] + b)
    return edges


def _kphased_edges(k: int, kp: tuple = _KP) -> tuple[list[int], int]:
    """k-chunk edges of the front phase (geometric growth from a small first
    chunk, capped) and the start of the row-blocked last phase."""
    first, growth, cap, share, _ = kp
    align = 128
    last = min(k - align, max(align, -(-int(k * share) // align) * align))
    front = k - last
    edges, pos, w = [0], 0, int(first)
    while pos < front:
        step = min(max(align, (w // align) * align), int(cap), front - pos)
        if front - pos - step < max(align, step // 2):
            step = front - pos
        pos += step
        edges.append(pos)
        w = int(w * growth)
    return edges, front


def _kphased_host_mm(A, B, C, kid: int, dev: int, st, overwrite: bool, front_share: float | None = None) -> None:
    """Host operands with a long k: overlap H2D, compute and D2H by cutting k
    first, rows last.

    Front phase: k chunks [l0, l1) of geometrically growing width; A[:, l0:l1]
    and B[l0:l1, :] go up on the H2D stream and the compute stream runs the
    whole C (+)= A[:, l0:l1] (x) B[l0:l1, :] as soon as they land (the first
    chunk overwrites; C's upload queues behind every chunk's, hidden by the
    front phase's compute, and is folded in with one (+) pass).  Last phase:
    the final k chunk row block by row block, each block's rows of C returned
    by the D2H stream while the next block computes.  So only the small first
    chunk's upload and the last row block's download are exposed.  The
    semiring's (+) is associative and commutative, so the result is the
    one-shot product (integer/tropical bit-identical; float within its
    summation tolerance).

    Pinned torch operands are DMA'd straight from host memory.  Pageable NumPy
    operands (the reference's own calling convention, matmul.py:342-366) are
    first copied chunk by chunk into pinned staging by the host thread pool --
    each chunk's upload is enqueued as soon as it is staged, so the staging of
    chunk i + 1 overlaps the DMA and compute of chunk i -- and C's row blocks
    are copied out of pinned staging while later blocks still compute.
    ``front_share`` (default the schedule's 0.75) = 0 skips the k chunks (short k).
    """
    n, k = tuple(A.shape)
    m = B.shape[1]
    staged = isinstance(A, np.ndarray)
    if staged and _register_host([A, B, C]):
        # page-locked in place: DMA straight from the NumPy buffers, as for pinned tensors
        A, B, C = torch.from_numpy(A), torch.from_numpy(B), torch.from_numpy(C)
        staged = False
    if front_share is not None and front_share <= 0:
        edges, front = [0], 0
    else:
        edges, front = _kphased_edges(k, _KP_STAGED if staged else _KP)
    redges = _row_edges(n)
    h2d = torch.cuda.Stream(device=dev)
    d2h = torch.cuda.Stream(device=dev)
    h2d.wait_stream(st)
    a_d = torch.empty((n, k), dtype=torch_dtype(A.dtype), device=dev)
    b_d = torch.empty((k, m), dtype=torch_dtype(B.dtype), device=dev)
    c_d = torch.empty((n, m), dtype=torch_dtype(C.dtype), device=dev)
    c_in = None if overwrite or front == 0 else torch.empty((n, m), dtype=torch_dtype(C.dtype), device=dev)
    for t in (a_d, b_d, c_d, c_in):
        if t is not None:
            t.record_stream(h2d)
            t.record_stream(d2h)
    if staged:  # whole-operand pinned staging, filled chunk by chunk
        a_s, b_s = _pinned_like(A.shape, A.dtype), _pinned_like(B.shape, B.dtype)
        c_s = _pinned_like(C.shape, C.dtype)
        a_sn, b_sn, c_sn = a_s.numpy(), b_s.numpy(), c_s.numpy()
        A_src, B_src, C_src = a_s, b_s, c_s
    else:
        A_src, B_src, C_src = A, B, C

    def upload(dst, r0, c0, rows, cols, src_t, src_np=None, host=None):
        if staged:  # row parts: part i's DMA runs while part i + 1 is staged
            parts = max(1, min(rows, rows * cols * host.itemsize // _STAGE_PART_BYTES))
            cuts = [r0 + rows * i // parts for i in range(parts + 1)]
            for a, b in zip(cuts[:-1], cuts[1:]):
                _host_copy(src_np[a:b, c0:c0 + cols], host[a:b, c0:c0 + cols])
                _copy2d(h2d, dst, a, c0, src_t, a, c0, b - a, cols)
        else:
            _copy2d(h2d, dst, r0, c0, src_t, r0, c0, rows, cols)
        ev = torch.cuda.Event()
        ev.record(h2d)
        return ev

    av, bv, cv = View.of(a_d), View.of(b_d), View.of(c_d)
    spans = list(zip(edges[:-1], edges[1:])) + [(front, k)]
    for idx, (l0, l1) in enumerate(spans):
        upload(a_d, 0, l0, n, l1 - l0, A_src, a_sn if staged else None, A)
        ev = upload(b_d, l0, 0, l1 - l0, m, B_src, b_sn if staged else None, B)
        if idx < len(spans) - 1:
            st.wait_event(ev)
            launch_mm(kid, st, av.sub(0, l0, n, l1 - l0), bv.sub(l0, 0, l1 - l0, m), cv, overwrite=idx == 0)
    last_ev = ev
    if front == 0:
        # no front phase: C is loaded first and the row blocks accumulate into it
        if not overwrite:
            st.wait_event(upload(c_d, 0, 0, n, m, C_src, c_sn if staged else None, C))
        else:
            launch_fill(kid, st, cv)
    elif c_in is not None:
        st.wait_event(upload(c_in, 0, 0, n, m, C_src, c_sn if staged else None, C))
        launch_fold(kid, st, cv, View.of(c_in), reset=False)
    st.wait_event(last_ev)
    outs = []
    for i in range(len(redges) - 1):
        r0, r1 = redges[i], redges[i + 1]
        if r1 <= r0:
            continue
        launch_mm(kid, st, av.sub(r0, front, r1 - r0, k - front), bv.sub(front, 0, k - front, m),
                  cv.sub(r0, 0, r1 - r0, m))
        done = torch.cuda.Event()
        done.record(st)
        d2h.wait_event(done)
        _copy2d(d2h, C_src, r0, 0, c_d, r0, 0, r1 - r0, m)
        if staged:
            back = torch.cuda.Event()
            back.record(d2h)
            outs.append((back, r0, r1))
    for back, r0, r1 in outs:  # copy each landed row block out while later ones compute
        back.synchronize()
        _host_copy(C[r0:r1], c_sn[r0:r1])
    st.wait_stream(d2h)
    d2h.synchronize()


def mm_oracle(A, B, semiring: Semiring = SEMIRING_INT):
    """Triple-loop ground truth on the device (matmul.py:400-414).

    One thread per C element folds the defining sum in l order; no tiling,
    shared memory or CTA plan, so it is independent of the fast kernels.
    Returns the same array kind as ``A``.
    """
    n, k = tuple(A.shape)
    _, m = tuple(B.shape)
    kid, in_dt = kernel_for(semiring, A, B)
    dev = pick_device(A, B)
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev)
        a = View.of(stage_in(A, in_dt, dev))
        b = View.of(stage_in(B, in_dt, dev))
        c = torch.empty((n, m), dtype=torch_dtype(semiring.dtype), device=dev)
        cv = View.of(c)
        launch_fill(kid, st, cv)
        nat.check(nat.load().paco_mm_naive(dev, st.cuda_stream, kid, a.ptr, a.ld, b.ptr, b.ld,
                                           cv.ptr, cv.ld, n, m, k))
    if isinstance(A, np.ndarray):
        return c.cpu().numpy()
    return c if isinstance(A, torch.Tensor) and A.is_cuda else c.cpu()


def semiring_vadd(semiring: Semiring, x, y):
    """Elementwise (+) of two equal-shape matrices into a new one."""
    if tuple(x.shape) != tuple(y.shape):
        raise ValueError(f"shape mismatch: {tuple(x.shape)} vs {tuple(y.shape)}")
    dev = pick_device(x, y)
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev)
        out = stage_in(x, semiring.dtype, dev).clone()
        yy = stage_in(y, semiring.dtype, dev)
        launch_fold(semiring.kernel_id, st, View.of(out), View.of(yy), reset=False)
    if isinstance(x, np.ndarray):
        return out.cpu().numpy()
    return out if isinstance(x, torch.Tensor) and x.is_cuda else out.cpu()


def fold_destinations(plan: Plan) -> dict[int, tuple[int, int, int]]:
    """Where each temporary finally lands: temp id -> (buffer 0, row offset, col offset).

    A REDUCE folds temp ``b`` into ``(out, oi, oj)`` (matmul.py:455-460); chains of
    nested k-cuts compose, ending in the caller's C (buffer 0).
    """
    via = {spec[0]: (spec[1], spec[2], spec[3]) for spec in plan.meta["reduces"].values()}
    dest: dict[int, tuple[int, int, int]] = {}

    def resolve(bid: int) -> tuple[int, int, int]:
        if bid == 0:
            return (0, 0, 0)
        if bid not in dest:
            tgt, oi, oj = via[bid]
            fb, fi, fj = resolve(tgt)
            dest[bid] = (fb, fi + oi, fj + oj)
        return dest[bid]

    for bid in plan.meta["temp_sizes"]:
        resolve(bid)
    return dest


_TC_KERNELS = (nat.SR_BF16_F32, nat.SR_F32_TC)
# test hook (set by tests/stage_all_check.py, never from the environment): every
# worker takes the remote-GPU path, "fused" (epilogue folds over NVLink) or
# "stage" (local block, one copy, staged atomic fold)
_REMOTE_ALL = ""


def mm_execute(plan: Plan, A, B, C, semiring: Semiring = SEMIRING_INT, mode: str = "serial_sim",
               sims: dict | None = None, *, devices: list[int] | None = None,
               fused_folds: bool | None = None, batch: bool | None = None, _narrow: bool = True) -> CostReport:
    """Run an MM plan on B200s (matmul.py:417-462).

    Worker ``w`` runs on ``devices[w % len(devices)]`` with its own stream
    (default: every worker on the current device, one stream each).  C and the
    temporaries live on the first device; A and B are replicated to every
    device used, and kernels on other devices reach C/temps through NVLink
    peer access.  ``mode`` keeps the reference meaning: ``serial_sim``
    enqueues tasks in plan order from this thread, ``parallel`` from one host
    thread per worker; the device result is identical.

    ``batch`` (default: on when every worker is on one device, the semiring
    runs on the SIMT kernel and the k-cut folds are fused): the plan's COMPUTE
    cuboids become ONE ``paco_mm_batch`` launch -- the GPU-level PACO plan is
    the CTA-level work list -- instead of one launch per task; any explicit
    REDUCE folds follow in plan order.
    """
    if sims is not None:
        raise NotImplementedError("cache simulation is out of scope on B200; use ncu counters")
    n, m, k = _shape_check(A, B, C)
    meta = plan.meta
    if (meta.get("n"), meta.get("m"), meta.get("k")) not in ((n, m, k), (None, None, None)):
        raise PlanError(f"plan built for {meta.get('n')}x{meta.get('m')}x{meta.get('k')}, "
                        f"operands are {n}x{m}x{k}")
    if _narrow and _narrowable(semiring, A, B, C, n, m, k):
        dev = devices[0] if devices else pick_device(A, B, C)
        with torch.cuda.device(dev):
            st = torch.cuda.current_stream(dev)
            nw = _Narrowed(semiring, A, B, C, dev, st, False)
            if nw.ok:
                report = mm_execute(plan, nw.a32, nw.b32, nw.c, nw.semiring, mode, devices=devices,
                                    fused_folds=fused_folds, batch=batch)
            else:
                report = mm_execute(plan, nw.a64, nw.b64, nw.out.dev, semiring, mode, devices=devices,
                                    fused_folds=fused_folds, batch=batch, _narrow=False)
                nw.minplus = False
            nw.finish(st)
        return report
    kid, in_dt = kernel_for(semiring, A, B)
    if devices is None:
        devices = [pick_device(A, B, C)]
    home = devices[0]
    dev_of = [devices[w % len(devices)] for w in range(plan.p)]
    used = sorted(set(dev_of))
    has_reduces = bool(meta["reduces"])
    if fused_folds is None:
        fused_folds = semiring.dtype.kind in "iu" if hasattr(semiring.dtype, "kind") else False
    if kid in _TC_KERNELS and any(d != home for d in used):
        fused_folds = False  # the tensor-core epilogue folds atomically only into local C
    fused_folds = fused_folds and has_reduces
    fold_dest = fold_destinations(plan) if fused_folds else {}
    if batch is None:
        batch = len(used) == 1 and kid not in _TC_KERNELS and (fused_folds or not has_reduces)
    batch = bool(batch) and len(used) == 1 and kid not in _TC_KERNELS
    batched: list = []     # COMPUTE problems, launched together after the plan walk
    deferred: list = []    # explicit REDUCE folds, run after the batch in plan order
    lib = nat.load()
    for d in used:
        if d != home:
            nat.check(lib.paco_enable_peer(d, home))

    with torch.cuda.device(home):
        stage = torch.cuda.current_stream(home)
        a_on = {d: View.of(stage_in(A, in_dt, d)) for d in used}
        b_on = {d: View.of(stage_in(B, in_dt, d)) for d in used}
        out = Output(C, semiring.dtype, home)
        c_view = View.of(out.dev)
        temps: dict[int, View] = {}
        for bid, size in ([] if fused_folds else meta["temp_sizes"].items()):
            shape = temp_shape(plan, bid) if size else (0, 1)
            t = torch.empty(shape, dtype=torch_dtype(semiring.dtype), device=home)
            temps[bid] = View.of(t)
            launch_fill(semiring.kernel_id, stage, temps[bid])
        staged = torch.cuda.Event()
        staged.record(stage)
        for d in used:
            if d != home:
                torch.cuda.current_stream(d).wait_event(staged)

        if batch:  # one launch on the staging stream: no worker streams to fork and join
            streams, fold_stream = [stage] * plan.p, stage
        else:
            streams = [torch.cuda.Stream(device=dev_of[w]) for w in range(plan.p)]
            for s in streams:
                s.wait_event(staged)
            fold_stream = torch.cuda.Stream(device=home)   # staged remote blocks fold here
            fold_stream.wait_event(staged)
        tdt = torch_dtype(semiring.dtype)
        events: list[torch.cuda.Event | None] = [None] * len(plan.tasks)
        reduces = meta["reduces"]
        t_begin = torch.cuda.Event(enable_timing=True)
        t_begin.record(stage)

        def buffer(bid: int) -> View:
            return c_view if bid == 0 else temps[bid]

        def runner(task) -> None:
            w = task.workers()[0]
            st = streams[w]
            if not batch:  # batched: nothing is launched here, the order is applied after the walk
                for d in task.deps:
                    st.wait_event(events[d])
            if task.kind == COMPUTE:
                cb: Cuboid = task.region
                dv = dev_of[w]
                if fused_folds:
                    fb, fi, fj = fold_dest.get(cb.out, (0, 0, 0))
                    out = c_view.sub(fi + cb.out_i0, fj + cb.out_j0, cb.n, cb.m)
                    flags = nat.MM_ATOMIC
                else:
                    out = buffer(cb.out).sub(cb.out_i0, cb.out_j0, cb.n, cb.m)
                    flags = 0
                av = a_on[dv].sub(cb.i0, cb.l0, cb.n, cb.k)
                bv = b_on[dv].sub(cb.l0, cb.j0, cb.k, cb.m)
                if batch:
                    batched.append((task.id, (av.ptr, av.ld, bv.ptr, bv.ld, out.ptr, out.ld, cb.n, cb.m, cb.k,
                                              flags)))
                    return
                remote = dv != home or bool(_REMOTE_ALL)
                staged = remote and (kid in _TC_KERNELS or _REMOTE_ALL == "stage")
                if remote and not staged:
                    # fused over NVLink: the kernel on the worker's GPU folds each finished
                    # tile into C on the home GPU with the semiring's (+) as per-element
                    # atomics (PACO_MM_REMOTE) -- the transfer overlaps the math tile by
                    # tile, no second pass (a k-cut partner may fold into the same block)
                    launch_mm(kid, st, av, bv, out, flags=nat.MM_ATOMIC | nat.MM_REMOTE, device=dv)
                elif staged:
                    # the tcgen05 kernels never address peer memory: the block is computed
                    # locally, shipped in one copy into a staging buffer on the home GPU
                    # and folded into its destination there with per-element atomics
                    with torch.cuda.device(dv):
                        loc = torch.empty((cb.n, cb.m), dtype=tdt, device=dv)
                        loc.record_stream(st)
                    launch_mm(kid, st, av, bv, View.of(loc), overwrite=True, device=dv)
                    stg = torch.empty((cb.n, cb.m), dtype=tdt, device=home)
                    stg.record_stream(st)
                    stg.record_stream(fold_stream)
                    _copy2d(st, stg, 0, 0, loc, 0, 0, cb.n, cb.m)
                    shipped = torch.cuda.Event()
                    shipped.record(st)
                    fold_stream.wait_event(shipped)
                    launch_fold(semiring.kernel_id, fold_stream, out, View.of(stg), False, atomic=True)
                    ev = torch.cuda.Event()
                    ev.record(fold_stream)
                    events[task.id] = ev
                    return
                else:
                    launch_mm(kid, st, av, bv, out, flags=flags, device=dv)
            elif task.kind == REDUCE and not fused_folds:
                bid, tgt, oi, oj, rn, rm = reduces[task.id]
                if batch:
                    deferred.append((task.id, buffer(tgt).sub(oi, oj, rn, rm), temps[bid]))
                    return
                launch_fold(semiring.kernel_id, st, buffer(tgt).sub(oi, oj, rn, rm),
                            temps[bid], reset=True)
            if not batch:
                ev = torch.cuda.Event()
                ev.record(st)
                events[task.id] = ev

        report = execute_plan(plan, runner, mode)
        if batch:  # the whole plan on one device: one launch, then the folds in plan order
            nat.mm_batch(home, stage.cuda_stream, kid, [p for _, p in sorted(batched)])
            for _, dst, src in sorted(deferred, key=lambda x: x[0]):
                launch_fold(semiring.kernel_id, stage, dst, src, reset=True)
        if not batch:
            for s in streams:
                stage.wait_stream(s)
            stage.wait_stream(fold_stream)
        t_end = torch.cuda.Event(enable_timing=True)
        t_end.record(stage)
        out.finish()
        t_end.synchronize()
        report.gpu_ms = t_begin.elapsed_time(t_end)
    return report


def measured_weights(devices: list[int], which: int = 0, iters: int = 20000) -> tuple[float, ...]:
    """Per-GPU throughput weights for ``mm_hetero_partition``.

    Runs the ALU issue-rate probe (``paco_alu_probe``: 0 = VIADDMNMX tropical
    term, 2 = FFMA) on every device and returns terms/clk/SM x the SM clock it
    ran at -- power-capped or thermally throttled GPUs get proportionally
    smaller cuboids.
    """
    out = []
    lib = nat.load()
    for d in devices:
        import ctypes

        tpc, mhz = ctypes.c_double(), ctypes.c_double()
        with torch.cuda.device(d):
            nat.check(lib.paco_alu_probe(d, None, which, iters, ctypes.byref(tpc), ctypes.byref(mhz)))
        out.append(tpc.value * mhz.value)
    return tuple(out)
