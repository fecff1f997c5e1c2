"""GPU parity of PACO-Strassen against the CPU restatement.

Integer ring: exact equality with the NumPy product / oracle Strassen.
float32: relative Frobenius error <= 1e-4 against the float64 oracle Strassen
(BASELINE cfg5 tolerance), at reduced size and at the full n=16384.
"""

import numpy as np
import pytest
import torch

from oracle import paco_numpy as PN
from paper_2011_01441_b200 import strassen as S

pytestmark = pytest.mark.gpu


def test_known_answers():
    assert S.strassen_seq(np.array([[3]], np.int64), np.array([[-4]], np.int64), 1).tolist() == [[-12]]
    rng = np.random.default_rng(1)
    B4 = rng.integers(-9, 10, (4, 4)).astype(np.int64)
    assert np.array_equal(S.strassen_seq(np.eye(4, dtype=np.int64), B4, 4, base=1), B4)
    A8, B8 = rng.integers(-9, 10, (8, 8)).astype(np.int64), rng.integers(-9, 10, (8, 8)).astype(np.int64)
    assert np.array_equal(S.strassen_seq(A8, B8, 8, base=1), A8 @ B8)


@pytest.mark.parametrize("n,base", [(16, 2), (64, 8), (100, 16), (256, 32), (256, 64)])
def test_integer_ring_exact(n, base):
    rng = np.random.default_rng(n + base)
    A = rng.integers(-50, 50, (n, n)).astype(np.int64)
    B = rng.integers(-50, 50, (n, n)).astype(np.int64)
    assert np.array_equal(S.strassen_seq(A, B, n, base=base), A @ B)


@pytest.mark.parametrize("p", [1, 2, 3, 5, 7, 10, 13])
def test_execute_plans_integer_exact(p):
    rng = np.random.default_rng(p)
    n = 256
    A = rng.integers(-30, 30, (n, n)).astype(np.int64)
    B = rng.integers(-30, 30, (n, n)).astype(np.int64)
    for plan in (S.strassen_paco_partition(n, p, base=16),
                 S.strassen_const_pieces_partition(n, p, S.SuperRoundCfg(2), base=16)):
        for mode in ("serial_sim", "parallel"):
            C = S.strassen_execute(plan, A, B, mode)
            assert np.array_equal(C, A @ B), (p, mode, plan.meta["variant"])


@pytest.mark.parametrize("p", [5, 8])
def test_execute_split_leftover(p):
    """Leftover leaves cut into p cuboids with k-cut folds: exact on the int64
    ring, 1e-4 on fp32 (3xTF32 leaf pieces), serial and parallel."""
    rng = np.random.default_rng(10 + p)
    n = 512
    A = rng.integers(-30, 30, (n, n)).astype(np.int64)
    B = rng.integers(-30, 30, (n, n)).astype(np.int64)
    plan = S.strassen_paco_partition(n, p, base=64, split_leftover=True)
    assert "split" in plan.meta["variant"]
    for mode in ("serial_sim", "parallel"):
        C = S.strassen_execute(plan, A, B, mode)
        assert np.array_equal(C, A @ B), (p, mode)
    Af = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    Bf = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    Cf = S.strassen_execute(plan, Af, Bf, "parallel")
    ref = Af.astype(np.float64) @ Bf.astype(np.float64)
    assert np.linalg.norm(Cf - ref) <= 1e-4 * np.linalg.norm(ref)


def test_f32_two_levels_vs_oracle():
    rng = np.random.default_rng(1005)
    n = 2048
    A = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    B = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    C = S.strassen_seq(A, B, n, base=n // 4)
    ref = PN.strassen(A.astype(np.float64), B.astype(np.float64), 2)
    err = np.linalg.norm(C.astype(np.float64) - ref) / np.linalg.norm(ref)
    assert err <= 1e-4, err


def test_cfg5_full_size_vs_oracle():
    """BASELINE cfg5: n=16384, 2 levels (49 leaves of 4096^3), fp32, rel Frobenius <= 1e-4."""
    rng = np.random.default_rng(1005)
    n = 16384
    A = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    B = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    c = S.strassen_seq(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), n, base=n // 4)
    C = c.cpu().numpy()
    del c
    torch.cuda.empty_cache()
    ref = PN.strassen(A.astype(np.float64), B.astype(np.float64), 2)
    err = np.linalg.norm(C.astype(np.float64) - ref) / np.linalg.norm(ref)
    assert err <= 1e-4, err


@pytest.mark.parametrize("transpose", [False, True])
def test_tf32_split_fused_sum_and_presplit_mm(transpose):
    """paco_tf32_split forms x = sum(+-in) as a tf32 (hi, lo) pair (hi has 13
    zero low mantissa bits, |x - hi - lo| <= 2^-21 |x|), optionally transposed;
    paco_mm_tf32x3 on pre-split operands equals the 3xTF32 paco_mm."""
    import ctypes
    from paper_2011_01441_b200 import _native as nat
    lib = nat.load()
    g = torch.Generator(device="cuda").manual_seed(3)
    rows, cols = 300, 260   # ragged: exercises the scalar edges of the vector kernels
    X = [torch.rand(rows + 5, cols + 8, device="cuda", generator=g) * 2 - 1 for _ in range(2)]
    views = [x[2:2 + rows, 4:4 + cols] for x in X]
    want = (views[0] - views[1]).double()
    orow, ocol = (cols, rows) if transpose else (rows, cols)
    ldo = (ocol + 3) // 4 * 4
    hi = torch.empty(orow, ldo, device="cuda"); lo = torch.empty(orow, ldo, device="cuda")
    ins = (ctypes.c_void_p * 2)(*[v.data_ptr() for v in views])
    lds = (ctypes.c_int64 * 2)(*[v.stride(0) for v in views])
    coefs = (ctypes.c_int32 * 2)(1, -1)
    nat.check(lib.paco_tf32_split(0, None, 2, ins, lds, coefs, rows, cols, int(transpose),
                                  hi.data_ptr(), lo.data_ptr(), ldo))
    torch.cuda.synchronize()
    h, l = hi[:, :ocol], lo[:, :ocol]
    if transpose:
        h, l = h.t(), l.t()
    assert int((h.contiguous().view(torch.int32) & 0x1FFF).abs().max()) == 0
    err = (h.double() + l.double() - want).abs()
    assert float((err - want.abs() * 2.0**-21).max()) <= 0
    # pre-split MM: C = S x T with S = X0 - X1 (n x k), T^T given transposed
    n, k, m = rows, cols, 200
    Y = torch.rand(k, m, device="cuda", generator=g) * 2 - 1
    ah = torch.empty(n, (k + 3) // 4 * 4, device="cuda"); al = torch.empty_like(ah)
    nat.check(lib.paco_tf32_split(0, None, 2, ins, lds, coefs, n, k, 0, ah.data_ptr(), al.data_ptr(), ah.stride(0)))
    bth = torch.empty(m, (k + 3) // 4 * 4, device="cuda"); btl = torch.empty_like(bth)
    yin = (ctypes.c_void_p * 1)(Y.data_ptr()); yld = (ctypes.c_int64 * 1)(Y.stride(0)); one = (ctypes.c_int32 * 1)(1)
    nat.check(lib.paco_tf32_split(0, None, 1, yin, yld, one, k, m, 1, bth.data_ptr(), btl.data_ptr(), bth.stride(0)))
    # a batch of 3: the same product into three C's (one tile queue), C[1] accumulating
    Cs = [torch.zeros(n, m, device="cuda") for _ in range(3)]
    Cs[1].fill_(1.0)
    arr = lambda xs: (ctypes.c_void_p * 3)(*xs)
    nat.check(lib.paco_mm_tf32x3(0, None, 3, arr([ah.data_ptr()] * 3), arr([al.data_ptr()] * 3), ah.stride(0),
                                 arr([bth.data_ptr()] * 3), arr([btl.data_ptr()] * 3), bth.stride(0),
                                 arr([c.data_ptr() for c in Cs]), Cs[0].stride(0), n, m, k, 0))
    torch.cuda.synchronize()
    ref = want @ Y.double()
    for q, C in enumerate(Cs):
        got = C.double() - (1.0 if q == 1 else 0.0)
        assert float((got - ref).norm() / ref.norm()) < 1e-5, q


@pytest.mark.parametrize("n,base", [(1000, 128), (777, 200), (33, 8)])
def test_f32_non_power_of_two(n, base):
    """fp32 Strassen on a zero-padded non-power-of-two n (3xTF32 leaves, fused
    leaf-level splits where the sizes allow), seq and a split-leftover plan."""
    rng = np.random.default_rng(n)
    A = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    B = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    C = S.strassen_seq(A, B, n, base=base)
    assert C.shape == (n, n)
    assert np.linalg.norm(C - ref) <= 1e-4 * np.linalg.norm(ref)
    C2 = S.strassen_execute(S.strassen_paco_partition(n, 6, base=base, split_leftover=True), A, B, "parallel")
    assert np.linalg.norm(C2 - ref) <= 1e-4 * np.linalg.norm(ref)


def test_tf32x3_multi_signed_destinations():
    """paco_mm_tf32x3_multi: product q folded with sign into each of its 1..4
    destinations (the fused Strassen C combination); destinations shared by two
    products receive both contributions; ragged n x m x k."""
    import ctypes
    from paper_2011_01441_b200 import _native as nat
    lib = nat.load()
    g = torch.Generator(device="cuda").manual_seed(5)
    n, m, k = 260, 200, 300
    kp = (k + 3) // 4 * 4
    prods, ops = [], []
    for _ in range(2):
        S = torch.rand(n, k, device="cuda", generator=g) * 2 - 1
        T = torch.rand(k, m, device="cuda", generator=g) * 2 - 1
        ah = torch.empty(n, kp, device="cuda"); al = torch.empty_like(ah)
        bh = torch.empty(m, kp, device="cuda"); bl = torch.empty_like(bh)
        one = (ctypes.c_int32 * 1)(1)
        nat.check(lib.paco_tf32_split(0, None, 1, (ctypes.c_void_p * 1)(S.data_ptr()),
                                      (ctypes.c_int64 * 1)(S.stride(0)), one, n, k, 0, ah.data_ptr(), al.data_ptr(), kp))
        nat.check(lib.paco_tf32_split(0, None, 1, (ctypes.c_void_p * 1)(T.data_ptr()),
                                      (ctypes.c_int64 * 1)(T.stride(0)), one, k, m, 1, bh.data_ptr(), bl.data_ptr(), kp))
        prods.append(S.double() @ T.double())
        ops.append((ah, al, bh, bl))
    mp = (m + 3) // 4 * 4
    D = [torch.zeros(n, mp, device="cuda") for _ in range(4)]
    D[3].fill_(2.0)
    # product 0 -> D0 (+), D1 (-), D2 (+), D3 (-); product 1 -> D1 (+), D3 (+)
    plan = [[(0, 1), (1, -1), (2, 1), (3, -1)], [(1, 1), (3, 1)]]
    ndst = (ctypes.c_int32 * 2)(*[len(p) for p in plan])
    dst = (ctypes.c_void_p * 8)()
    sign = (ctypes.c_int32 * 8)()
    for q, p in enumerate(plan):
        for d, (i, sg) in enumerate(p):
            dst[4 * q + d] = D[i].data_ptr()
            sign[4 * q + d] = sg
    arr = lambda j: (ctypes.c_void_p * 2)(*[o[j].data_ptr() for o in ops])
    nat.check(lib.paco_mm_tf32x3_multi(0, None, 2, arr(0), arr(1), kp, arr(2), arr(3), kp, ndst, dst, sign, mp,
                                       n, m, k))
    torch.cuda.synchronize()
    want = [prods[0], -prods[0] + prods[1], prods[0], 2.0 - prods[0] + prods[1]]
    for i in range(4):
        got = D[i][:, :m].double()
        assert float((got - want[i]).norm() / want[i].norm()) < 1e-5, i
