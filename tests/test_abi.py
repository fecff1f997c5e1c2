"""The C-ABI library loads on a CPU-only host and exports every declared symbol."""

import ctypes
import os
import re

import pytest

from paper_2011_01441_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "paco_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(paco_[a-z0-9_]+)\s*\(", text)))


def test_all_header_symbols_exported_and_bound():
    lib = nat.load()
    names = header_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(lib, name), name
        assert name in nat.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.paco_abi_version() == 1


def test_tile_shapes():
    for sr in range(nat.SR_COUNT):
        bm, bn, bk, cps = nat.tile_shape(sr)
        assert bm > 0 and bn > 0 and bk > 0 and cps >= 1


def test_argument_errors_without_device():
    lib = nat.load()
    rc = lib.paco_mm(0, None, 99, None, 0, None, 0, None, 0, 1, 1, 1, None, 0, 0)
    assert rc == nat.ERR_ARG and b"semiring" in lib.paco_last_error()
    rc = lib.paco_mm(0, None, nat.SR_F32, None, 4, None, 4, None, 4, 4, 4, 4, None, 0, 0)
    assert rc == nat.ERR_ARG and b"null" in lib.paco_last_error()
    rc = lib.paco_mm(0, None, nat.SR_F32, 16, 2, 16, 4, 16, 4, 4, 4, 4, None, 0, 0)
    assert rc == nat.ERR_ARG and b"leading dimension" in lib.paco_last_error()
    with pytest.raises(ValueError):
        nat.check(rc)
    with pytest.raises(nat.PlanError):
        nat.plan_one_piece(1, 1, 1, 2)


@pytest.mark.parametrize("shape,cols", [((1, 1), (0, 1)), ((7, 5), (1, 4)), ((3000, 700), (13, 555)),
                                        ((8192, 2048), (128, 1152))])
def test_host_copy2d_parallel_staging(shape, cols):
    """paco_host_copy2d (the pageable -> pinned staging memcpy of the NumPy e2e
    path) copies strided 2-D views exactly, from 1 to 16 participants, repeatedly
    (the persistent pool is reused across calls)."""
    import numpy as np

    from paper_2011_01441_b200 import mm as MM
    rng = np.random.default_rng(shape[0])
    src = rng.integers(-2**31, 2**31 - 1, shape, dtype=np.int64).astype(np.int32)
    c0, c1 = cols
    for threads in (1, 3, 8, 16):
        dst = np.zeros(shape, np.int32)
        old = MM._HOST_THREADS
        MM._HOST_THREADS = threads
        try:
            for _ in range(3):
                MM._host_copy(dst[:, c0:c1], src[:, c0:c1])
        finally:
            MM._HOST_THREADS = old
        want = np.zeros(shape, np.int32)
        want[:, c0:c1] = src[:, c0:c1]
        assert np.array_equal(dst, want), threads


def test_host_copy2d_back_to_back_jobs():
    """Many short jobs back to back, each into a fresh destination: a pool
    worker that wakes after its job finished must not take part in the next
    one with the old job's pointers (which would leave a part of the new
    destination uncopied)."""
    import numpy as np

    from paper_2011_01441_b200 import mm as MM
    rng = np.random.default_rng(7)
    srcs = [rng.integers(0, 2**31 - 1, (256 + 64 * (i % 5), 1024 + 256 * (i % 3)), dtype=np.int64).astype(np.int32)
            for i in range(8)]
    old = MM._HOST_THREADS
    MM._HOST_THREADS = 12
    try:
        for it in range(400):
            src = srcs[it % len(srcs)]
            dst = np.zeros_like(src)
            MM._host_copy(dst, src)
            assert np.array_equal(dst, src), it
    finally:
        MM._HOST_THREADS = old
