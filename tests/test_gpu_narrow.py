"""The reference's own int64 semirings on the 32-bit kernels (range-checked narrowing).

SEMIRING_MINPLUS (int64, zero 2^62, matmul.py:29,49-50,55) and SEMIRING_INT
(int64, matmul.py:45-46,53) keep their int64 API; when every operand fits 32
bits mm_seq / mm_execute run the u32 (min,+) or int32 x int32 -> int64 kernel
and must give the int64 answer bit for bit -- and fall back to the int64
kernel on any operand outside the range (INF = 2^62 sentinels, negatives,
values >= 2^31).  Checked against the pinned CPU oracle and the reference's
golden vectors.
"""

import numpy as np
import pytest
import torch

from oracle import cref
from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200 import mm as MM

pytestmark = pytest.mark.gpu

ZERO = int(M.MINPLUS_INF)


@pytest.fixture
def always_narrow(monkeypatch):
    monkeypatch.setattr(MM, "NARROW_MIN_TERMS", 0)


def _spy(monkeypatch):
    """Record which kernel ids paco_mm / paco_mm_batch ran."""
    seen = []
    real_launch, real_batch = MM.launch_mm, MM.nat.mm_batch

    def launch(kid, *a, **kw):
        seen.append(kid)
        return real_launch(kid, *a, **kw)

    def batch(dev, st, kid, probs):
        seen.append(kid)
        return real_batch(dev, st, kid, probs)
    monkeypatch.setattr(MM, "launch_mm", launch)
    monkeypatch.setattr(MM.nat, "mm_batch", batch)
    return seen


def _want_minplus(A, B, C0):
    want = C0.copy()
    return cref.mm(cref.SR_MINPLUS_I64, A, B, want)


@pytest.mark.parametrize("shape", [(1, 1, 1), (37, 45, 29), (200, 130, 257), (513, 260, 300)])
def test_minplus_i64_narrowed_matches_oracle(always_narrow, monkeypatch, shape):
    n, m, k = shape
    rng = np.random.default_rng(11 + n)
    A = rng.integers(0, 2**31, (n, k), dtype=np.int64)
    B = rng.integers(0, 2**31, (k, m), dtype=np.int64)
    A[0, 0] = 2**31 - 1  # extreme sums: 2^32 - 2
    B[0, 0] = 2**31 - 1
    C0 = np.full((n, m), ZERO, np.int64)
    mask = rng.random((n, m)) < 0.2
    C0[mask] = rng.integers(0, 2**33, int(mask.sum()))  # finite C entries, some above 2^32 - 1
    C0.flat[::7] = rng.integers(0, 2**34, C0.flat[::7].shape)
    want = _want_minplus(A, B, C0)
    seen = _spy(monkeypatch)
    C = C0.copy()
    M.mm_seq(A, B, C, M.SEMIRING_MINPLUS)
    assert np.array_equal(C, want)
    assert seen and all(s == 9 for s in seen)  # PACO_SR_MINPLUS_U32


def test_minplus_i64_out_of_range_falls_back(always_narrow, monkeypatch, golden_cases):
    # the reference fixture holds 2^62 sentinels and a wrapping INF + INF: int64 kernel
    A, B, want = golden_cases["minplus_i64_A"], golden_cases["minplus_i64_B"], golden_cases["minplus_i64_C"]
    n, k = A.shape
    m = B.shape[1]
    seen = _spy(monkeypatch)
    C = np.full((n, m), ZERO, np.int64)
    M.mm_execute(M.mm_paco_partition(n, m, k, 3), A, B, C, M.SEMIRING_MINPLUS)
    assert np.array_equal(C, want)
    assert 9 not in seen
    # a negative operand also keeps the int64 kernel
    rng = np.random.default_rng(3)
    A2 = rng.integers(0, 1000, (40, 50), dtype=np.int64)
    B2 = rng.integers(0, 1000, (50, 60), dtype=np.int64)
    A2[5, 5] = -3
    C0 = np.full((40, 60), ZERO, np.int64)
    want2 = _want_minplus(A2, B2, C0)
    C2 = C0.copy()
    M.mm_seq(A2, B2, C2, M.SEMIRING_MINPLUS)
    assert np.array_equal(C2, want2)
    # and a negative C
    C3 = C0.copy()
    C3[0, 0] = -1
    want3 = _want_minplus(A2 * 0 + 7, B2, C3)
    M.mm_seq(A2 * 0 + 7, B2, C3, M.SEMIRING_MINPLUS)
    assert np.array_equal(C3, want3)


@pytest.mark.parametrize("p", [1, 3, 5, 7])
def test_minplus_i64_narrowed_plans(always_narrow, p):
    n, m, k = 300, 260, 515
    rng = np.random.default_rng(100 + p)
    A = rng.integers(0, 2**20, (n, k), dtype=np.int64)
    B = rng.integers(0, 2**20, (k, m), dtype=np.int64)
    C0 = np.full((n, m), ZERO, np.int64)
    want = _want_minplus(A, B, C0)
    for fused in (True, False):
        C = C0.copy()
        M.mm_execute(M.mm_one_piece_partition(n, m, k, p), A, B, C, M.SEMIRING_MINPLUS, fused_folds=fused)
        assert np.array_equal(C, want), (p, fused)
    C = C0.copy()
    M.mm_execute(M.mm_paco_partition(n, m, k, p), A, B, C, M.SEMIRING_MINPLUS)
    assert np.array_equal(C, want)


def test_minplus_i64_device_tensors_and_overwrite(always_narrow):
    n, m, k = 129, 257, 200
    rng = np.random.default_rng(5)
    A = rng.integers(0, 2**31, (n, k), dtype=np.int64)
    B = rng.integers(0, 2**31, (k, m), dtype=np.int64)
    want = _want_minplus(A, B, np.full((n, m), ZERO, np.int64))
    a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    c = torch.full((n, m), ZERO, dtype=torch.int64, device="cuda")
    M.mm_seq(a, b, c, M.SEMIRING_MINPLUS)
    assert np.array_equal(c.cpu().numpy(), want)
    c2 = torch.empty((n, m), dtype=torch.int64, device="cuda")  # garbage C, overwrite declared
    M.mm_seq(a, b, c2, M.SEMIRING_MINPLUS, overwrite=True)
    assert np.array_equal(c2.cpu().numpy(), want)


def test_int64_ring_narrowed_wraps_like_numpy(always_narrow, monkeypatch, golden_cases):
    # extreme int32 values: products 2^62, sums wrap int64 exactly like NumPy
    n, m, k = 70, 90, 130
    rng = np.random.default_rng(9)
    A = rng.choice(np.array([-(2**31), 2**31 - 1, -1, 0, 1, 12345], np.int64), (n, k))
    B = rng.choice(np.array([-(2**31), 2**31 - 1, 7, -7], np.int64), (k, m))
    C0 = rng.integers(-(2**62), 2**62, (n, m), dtype=np.int64)
    with np.errstate(over="ignore"):
        want = C0 + A @ B
    seen = _spy(monkeypatch)
    C = C0.copy()
    M.mm_seq(A, B, C, M.SEMIRING_INT)
    assert np.array_equal(C, want)
    assert seen and all(s == 1 for s in seen)  # PACO_SR_INT_I32_I64
    # the reference's cfg1 plan on int64 operands (narrowed) matches its golden C
    g = golden_cases
    plan = M.mm_paco_partition(384, 320, 256, 3)
    C = np.zeros((384, 320), np.int64)
    M.mm_execute(plan, g["cfg1_A"].astype(np.int64), g["cfg1_B"].astype(np.int64), C, M.SEMIRING_INT)
    assert np.array_equal(C, g["cfg1_C"])
    # golden wrapping int64 fixture: operands beyond int32 -> int64 kernel, same answer
    seen.clear()
    C = g["int_wrap_C0"].copy()
    n, k = g["int_wrap_A"].shape
    m = g["int_wrap_B"].shape[1]
    M.mm_seq(g["int_wrap_A"], g["int_wrap_B"], C, M.SEMIRING_INT)
    assert np.array_equal(C, g["int_wrap_C"])
    assert 1 not in seen


def _inf_operands(rng, n, m, k, p_inf=0.2, hi=2**30 - 2):
    A = rng.integers(0, hi + 1, (n, k), dtype=np.int64)
    B = rng.integers(0, hi + 1, (k, m), dtype=np.int64)
    A[rng.random(A.shape) < p_inf] = ZERO
    B[rng.random(B.shape) < p_inf] = ZERO
    return A, B


@pytest.mark.parametrize("shape", [(1, 1, 1), (37, 45, 29), (200, 130, 257), (513, 260, 300)])
def test_minplus_i64_inf_kept_on_u32(always_narrow, monkeypatch, shape):
    """INF = 2^62 sentinels stay on the u32 kernel: one-INF terms give the
    reference's 2^62 + f, an all-INF row against an all-INF column its int64
    wrap INF + INF = -2^63 -- bit for bit."""
    n, m, k = shape
    rng = np.random.default_rng(21 + n)
    A, B = _inf_operands(rng, n, m, k)
    A[0, 0] = 2**30 - 2  # extreme finite sums
    B[0, 0] = 2**30 - 2
    if n > 2 and m > 2:
        A[1, :] = ZERO          # row 1: every term has an INF on the A side ...
        B[:, 2] = ZERO          # ... and column 2 every term on the B side: C[1, 2] = INF + INF wrap
        A[2, :] = ZERO          # row 2 against a finite column: C[2, 0] = 2^62 + min_l B[l, 0]
        B[:, 0] = rng.integers(0, 2**30 - 1, k)
    C0 = np.full((n, m), ZERO, np.int64)
    mask = rng.random((n, m)) < 0.2
    C0[mask] = rng.integers(-(2**40), 2**63 - 1, int(mask.sum()))  # any int64 C, negatives included
    want = _want_minplus(A, B, C0)
    seen = _spy(monkeypatch)
    C = C0.copy()
    M.mm_seq(A, B, C, M.SEMIRING_MINPLUS)
    assert np.array_equal(C, want)
    assert seen and all(s == 9 for s in seen)  # PACO_SR_MINPLUS_U32
    if n > 2 and m > 2:
        assert C[1, 2] == np.iinfo(np.int64).min
        assert C[2, 0] == min(C0[2, 0], ZERO + int(B[:, 0].min()))


@pytest.mark.parametrize("p", [3, 5, 7])
def test_minplus_i64_inf_plans(always_narrow, monkeypatch, p):
    n, m, k = 300, 260, 515
    rng = np.random.default_rng(300 + p)
    A, B = _inf_operands(rng, n, m, k, p_inf=0.5)
    C0 = np.full((n, m), ZERO, np.int64)
    want = _want_minplus(A, B, C0)
    seen = _spy(monkeypatch)
    for fused in (True, False):
        C = C0.copy()
        M.mm_execute(M.mm_one_piece_partition(n, m, k, p), A, B, C, M.SEMIRING_MINPLUS, fused_folds=fused)
        assert np.array_equal(C, want), (p, fused)
    assert seen and all(s == 9 for s in seen)


def test_minplus_i64_inf_ranges(always_narrow, monkeypatch):
    rng = np.random.default_rng(77)
    n, m, k = 90, 70, 110
    # finite values up to 2^31 - 1 without INF: the plain u32 code (second narrowing try)
    A = rng.integers(2**30, 2**31, (n, k), dtype=np.int64)
    B = rng.integers(0, 2**31, (k, m), dtype=np.int64)
    C0 = np.full((n, m), ZERO, np.int64)
    want = _want_minplus(A, B, C0)
    seen = _spy(monkeypatch)
    C = C0.copy()
    M.mm_seq(A, B, C, M.SEMIRING_MINPLUS)
    assert np.array_equal(C, want) and seen and all(s == 9 for s in seen)
    # INF next to a finite value >= 2^30 - 1: no u32 code holds both -> int64 kernel, same answer
    A2, B2 = _inf_operands(rng, n, m, k)
    A2[3, 3] = 2**30 - 1
    want2 = _want_minplus(A2, B2, C0)
    seen.clear()
    C2 = C0.copy()
    M.mm_seq(A2, B2, C2, M.SEMIRING_MINPLUS)
    assert np.array_equal(C2, want2) and 9 not in seen
    # a device-side run with overwrite: garbage C, INF operands
    a, b = torch.from_numpy(A2 * 0 + B2[:1, :1].item()).cuda(), torch.from_numpy(B2).cuda()
    A3, B3 = _inf_operands(rng, n, m, k)
    want3 = _want_minplus(A3, B3, C0)
    c = torch.empty((n, m), dtype=torch.int64, device="cuda")
    M.mm_seq(torch.from_numpy(A3).cuda(), torch.from_numpy(B3).cuda(), c, M.SEMIRING_MINPLUS, overwrite=True)
    assert np.array_equal(c.cpu().numpy(), want3)
    del a, b
