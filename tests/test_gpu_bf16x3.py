"""The bf16x3 Strassen leaf format: paco_lincomb_split (signed sums written as
bf16 hi / lo planes) and paco_mm_bf16x3_multi (hi*hi + hi*lo + lo*hi on
tcgen05 kind::f16 CTA pairs, signed multi-destination epilogue).

The split is checked bit-exactly against torch's own bf16 rounding of the same
fp32 sums; the products against float64 products of the fp32 operands (the
format keeps ~16 significant bits of each operand, so the product error is
in the 1e-5 class, well inside cfg5's 1e-4 Frobenius budget); the Strassen
path end to end against the f64 product at cfg5's half size."""

import ctypes

import pytest
import torch

from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200 import strassen as S

pytestmark = pytest.mark.gpu


def _split(lib, st, q, rows):
    """paco_lincomb_split of the coefficient rows over the input views q."""
    n, m = q[0].shape
    his = [torch.full((n, m + 8), float("nan"), device="cuda").bfloat16()[:, :m] for _ in rows]
    los = [torch.full((n, m + 8), float("nan"), device="cuda").bfloat16()[:, :m] for _ in rows]
    nat.check(lib.paco_lincomb_split(0, st, n, m, len(q), (ctypes.c_void_p * len(q))(*[x.data_ptr() for x in q]),
                                     (ctypes.c_int64 * len(q))(*[x.stride(0) for x in q]), len(rows),
                                     (ctypes.c_void_p * len(rows))(*[h.data_ptr() for h in his]),
                                     (ctypes.c_void_p * len(rows))(*[x.data_ptr() for x in los]),
                                     (ctypes.c_int64 * len(rows))(*[h.stride(0) for h in his]),
                                     (ctypes.c_int32 * (len(rows) * len(q)))(*[c for r in rows for c in r])))
    return his, los


@pytest.mark.parametrize("shape", [(64, 64), (257, 1032), (4096, 4096)])
def test_lincomb_split_exact(shape):
    """Each output is hi = bf16_rn(x), lo = bf16_rn(x - hi) of the fp32 signed sum x,
    bit-identical to torch's rounding; one-term rows are split copies."""
    n, m = shape
    lib = nat.load()
    st = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(n + m)
    big = torch.randn(2 * n, 2 * m + 8, device="cuda", generator=g)
    q = [big[:n, :m], big[:n, m:2 * m], big[n:, :m], big[n:, m:2 * m]]
    rows = [[1, 0, 0, 1], [0, 0, 1, 1], [1, 0, 0, 0], [0, 0, 0, 1], [1, 1, 0, 0], [-1, 0, 1, 0], [0, 1, 0, -1]]
    his, los = _split(lib, st, q, rows)
    torch.cuda.synchronize()
    for h, lo, r in zip(his, los, rows):
        x = sum(c * v for c, v in zip(r, q) if c)
        hi_ref = x.bfloat16()
        lo_ref = (x - hi_ref.float()).bfloat16()
        assert torch.equal(h.view(torch.int16), hi_ref.view(torch.int16))
        assert torch.equal(lo.view(torch.int16), lo_ref.view(torch.int16))
        # the pair reproduces x to ~2^-17 relative
        rec = h.double() + lo.double()
        assert float(((rec - x.double()).abs() / x.double().abs().clamp_min(1e-30)).max()) <= 2.0 ** -16


def test_lincomb_split_eight_inputs():
    """Eight inputs (two level-0 blocks' quadrants): a leaf node's operands straight
    from the level-0 blocks, e.g. (A00 + A11)'s sub-quadrant sums."""
    n = m = 520
    lib = nat.load()
    st = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(8, n, m, device="cuda", generator=g)
    q = [x[i] for i in range(8)]
    rows = [[1, 0, 0, 1, -1, 0, 0, -1], [0, 0, 1, 1, 0, 0, 1, 1], [1, 0, 0, 0, 1, 0, 0, 0],
            [0, 0, 0, 1, 0, 0, 0, -1], [1, 1, 0, 0, 1, 1, 0, 0], [-1, 0, 1, 0, -1, 0, 1, 0], [0, 1, 0, -1, 0, 0, 0, 0]]
    his, los = _split(lib, st, q, rows)
    torch.cuda.synchronize()
    for h, lo, r in zip(his, los, rows):
        want = sum(c * v.double() for c, v in zip(r, q) if c)
        rec = h.double() + lo.double()
        assert float((rec - want).abs().max() / want.abs().max()) <= 2.0 ** -15


@pytest.mark.parametrize("bnat", [False, True])
@pytest.mark.parametrize("shape", [(2048, 2048, 512, 4), (2000, 1800, 336, 7), (256, 256, 32, 1), (384, 200, 72, 2)])
def test_bf16x3_pair_kernel_accuracy(shape, bnat):
    """Products vs float64 of the fp32 operands: two signed destinations per
    product, ragged extents (TMA zero fill at tile edges), count 1..7; B given
    as B^T (K-major tiles) or in its own k x m layout (bnat: MN-major tiles)."""
    n, m, k, cnt = shape
    lib = nat.load()
    st = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(k + cnt)
    a = [(torch.rand(n, k, device="cuda", generator=g) * 2 - 1) for _ in range(cnt)]
    b = [(torch.rand(m, k, device="cuda", generator=g) * 2 - 1) for _ in range(cnt)]
    sa = [_split(lib, st, [x], [[1]]) for x in a]
    sb = [_split(lib, st, [x.t().contiguous() if bnat else x], [[1]]) for x in b]
    lda, ldb = sa[0][0][0].stride(0), sb[0][0][0].stride(0)
    arr = lambda xs: (ctypes.c_void_p * cnt)(*[x.data_ptr() for x in xs])  # noqa: E731
    C = [torch.zeros(n, m, device="cuda") for _ in range(2)]
    ndst = (ctypes.c_int32 * cnt)(*[2] * cnt)
    dst = (ctypes.c_void_p * (4 * cnt))()
    sign = (ctypes.c_int32 * (4 * cnt))()
    ref = [torch.zeros(n, m, dtype=torch.float64, device="cuda") for _ in range(2)]
    for q in range(cnt):
        dst[4 * q], dst[4 * q + 1] = C[q % 2].data_ptr(), C[(q + 1) % 2].data_ptr()
        sign[4 * q], sign[4 * q + 1] = 1, (-1 if q % 2 else 1)
        p = a[q].double() @ b[q].double().t()
        ref[q % 2] += p
        ref[(q + 1) % 2] += -p if q % 2 else p
    fn = lib.paco_mm_bf16x3_multi_bn if bnat else lib.paco_mm_bf16x3_multi
    nat.check(fn(0, st, cnt, arr([x[0][0] for x in sa]), arr([x[1][0] for x in sa]), lda,
                 arr([x[0][0] for x in sb]), arr([x[1][0] for x in sb]), ldb, ndst, dst, sign, m, n, m, k))
    torch.cuda.synchronize()
    for i in range(2):
        if cnt == 1 and i == 1:
            continue
        assert float((C[i].double() - ref[i]).norm() / ref[i].norm()) < 2e-5, i


def test_bf16x3_rejects_misaligned():
    lib = nat.load()
    st = torch.cuda.current_stream().cuda_stream
    x = torch.zeros(256, 40, dtype=torch.bfloat16, device="cuda")
    c = torch.zeros(256, 256, device="cuda")
    one = lambda p: (ctypes.c_void_p * 1)(p)  # noqa: E731
    rc = lib.paco_mm_bf16x3_multi(0, st, 1, one(x.data_ptr() + 2), one(x.data_ptr()), 40, one(x.data_ptr()),
                                  one(x.data_ptr()), 40, (ctypes.c_int32 * 1)(1), one(c.data_ptr()),
                                  (ctypes.c_int32 * 4)(1), 256, 256, 256, 32)
    assert rc != 0


@pytest.mark.parametrize("direct,natural,onepass", [(True, True, True), (True, True, False), (True, False, False),
                                                    (False, False, False)])
def test_strassen_bf16x3_vs_tf32b2(monkeypatch, direct, natural, onepass):
    """cfg5's shape at half size (8192, 2 levels): the bf16x3 leaves (default: leaf
    operands of a side in one pass, or per node straight from the level-0 blocks, B
    in its own layout or transposed; or from level-1 fp32 sums) and the tf32 + 2 x
    bf16 leaves all within 1e-4 of the f64 product."""
    monkeypatch.setattr(S, "B3_DIRECT", direct)
    monkeypatch.setattr(S, "B3_NATURAL", natural)
    monkeypatch.setattr(S, "B3_ONEPASS", onepass)
    n, base = 8192, 2048
    g = torch.Generator(device="cuda").manual_seed(8)
    a = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    b = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    rows = torch.arange(0, n, 61, device="cuda")
    ref = a[rows].double() @ b.double()
    err = {}
    for b3 in (True, False):
        monkeypatch.setattr(S, "LEAF_BF16X3", b3)
        c = S.strassen_seq(a, b, n, base=base)
        err[b3] = float((c[rows].double() - ref).norm() / ref.norm())
    assert err[True] < 1e-4 and err[False] < 1e-4, err


def test_strassen_into_b3n_signed_placements():
    """strassen_into on a leaf-level node and on a node whose children are
    leaf-level, B in its own layout, folded +/- into two C blocks."""
    from paper_2011_01441_b200.device import View
    for n, base in ((4096, 2048), (8192, 2048)):
        g = torch.Generator(device="cuda").manual_seed(n)
        a = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
        b = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
        C = torch.rand(n, 2 * n, device="cuda", generator=g)
        C0 = C.clone()
        st = torch.cuda.current_stream()
        assert S._b3n_ok(n, base, [(None, 1), (None, -1)]) == (n == 4096)
        dests = [(View.of(C[:, :n]), 1)] if n == 8192 else [(View.of(C[:, :n]), 1), (View.of(C[:, n:]), -1)]
        assert S.strassen_into(View.of(a), View.of(b), dests, base, st)
        rows = torch.arange(0, n, 61, device="cuda")
        ref = a[rows].double() @ b.double()
        for half, sg in ((0, 1), (1, -1))[:len(dests)]:
            got = C[rows, half * n:(half + 1) * n].double() - C0[rows, half * n:(half + 1) * n].double()
            err = float((got - sg * ref).norm() / ref.norm())
            assert err <= 1e-4, (n, half, err)


@pytest.mark.parametrize("side", [0, 1])
def test_strassen_split49(side):
    """paco_strassen_split49: leaf (r, r') = formula r over the quadrants and r' over
    their sub-quadrants, as bf16 hi / lo planes (hi + lo within 2^-15 of the f64 sum)."""
    h = 264
    n = 4 * h
    lib = nat.load()
    st = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(side)
    big = torch.rand(n, n + 8, device="cuda", generator=g) * 2 - 1
    x = big[:, :n]
    planes = torch.full((2, 49, h, h + 8), float("nan"), device="cuda").bfloat16()
    his = (ctypes.c_void_p * 49)(*[planes[0, o].data_ptr() for o in range(49)])
    los = (ctypes.c_void_p * 49)(*[planes[1, o].data_ptr() for o in range(49)])
    nat.check(lib.paco_strassen_split49(0, st, side, x.data_ptr(), x.stride(0), h, his, los, h + 8))
    torch.cuda.synchronize()
    names = ("00", "01", "10", "11")
    tab = S.T_TERMS if side else S.S_TERMS
    blk = lambda q1, q2: x[(names.index(q1) >> 1) * 2 * h + (names.index(q2) >> 1) * h:][:h, (names.index(q1) & 1) * 2 * h + (names.index(q2) & 1) * h:][:, :h]  # noqa: E731
    for r in range(1, 8):
        for r2 in range(1, 8):
            want = sum(c1 * c2 * blk(q1, q2).double() for c1, q1 in tab[r] for c2, q2 in tab[r2])
            o = 7 * (r - 1) + r2 - 1
            got = planes[0, o, :, :h].double() + planes[1, o, :, :h].double()
            assert float((got - want).abs().max()) <= 2.0 ** -15 * float(want.abs().max()), (r, r2)


def test_strassen_split49_rejects_bad_arguments():
    lib = nat.load()
    st = torch.cuda.current_stream().cuda_stream
    x = torch.zeros(4 * 64, 4 * 64, device="cuda")
    p = torch.zeros(64, 64, dtype=torch.bfloat16, device="cuda")
    planes = (ctypes.c_void_p * 49)(*([p.data_ptr()] * 49))
    assert lib.paco_strassen_split49(0, st, 2, x.data_ptr(), 256, 64, planes, planes, 64) != 0      # side
    assert lib.paco_strassen_split49(0, st, 0, x.data_ptr() + 4, 256, 64, planes, planes, 64) != 0  # misaligned
    assert lib.paco_strassen_split49(0, st, 0, x.data_ptr(), 256, 60, planes, planes, 64) != 0      # h % 8
