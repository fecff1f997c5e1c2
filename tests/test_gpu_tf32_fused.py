"""The fused-formation 3xTF32 kernel (paco_mm_tf32x3_fused) and paco_transpose.

Each problem's operands are signed sums of 1-2 raw fp32 views formed inside
the GEMM (Strassen's S_r and T_r^T); checked against float64 products of the
same sums, with ragged extents (TMA zero fill at the tile edges), both term
counts, negative terms and up to four signed destinations."""

import ctypes

import numpy as np
import pytest
import torch

from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200 import strassen as S

pytestmark = pytest.mark.gpu


def _call(probs, n, m, k, ldc):
    c = len(probs)
    nta, ntb = (ctypes.c_int32 * c)(), (ctypes.c_int32 * c)()
    at, bt = (ctypes.c_void_p * (2 * c))(), (ctypes.c_void_p * (2 * c))()
    asg, bsg = (ctypes.c_int32 * (2 * c))(), (ctypes.c_int32 * (2 * c))()
    ndst, dst, sign = (ctypes.c_int32 * c)(), (ctypes.c_void_p * (4 * c))(), (ctypes.c_int32 * (4 * c))()
    lda = ldb = None
    for q, (aterms, bterms, dests) in enumerate(probs):
        nta[q], ntb[q], ndst[q] = len(aterms), len(bterms), len(dests)
        for t, (sg, x) in enumerate(aterms):
            at[2 * q + t], asg[2 * q + t], lda = x.data_ptr(), sg, x.stride(0)
        for t, (sg, x) in enumerate(bterms):
            bt[2 * q + t], bsg[2 * q + t], ldb = x.data_ptr(), sg, x.stride(0)
        for d, (sg, x) in enumerate(dests):
            dst[4 * q + d], sign[4 * q + d] = x.data_ptr(), sg
    nat.check(nat.load().paco_mm_tf32x3_fused(0, torch.cuda.current_stream().cuda_stream, c, nta, at, asg, lda, ntb,
                                              bt, bsg, ldb, ndst, dst, sign, ldc, n, m, k))


@pytest.mark.parametrize("shape", [(128, 256, 16), (300, 520, 100), (1024, 768, 1040), (129, 252, 33)])
def test_fused_terms_signs_destinations(shape):
    n, m, k = shape
    g = torch.Generator(device="cuda").manual_seed(n + m + k)
    kp = (k + 3) // 4 * 4   # 16-byte row pitch
    mp = (m + 3) // 4 * 4

    def mat(r):
        return (torch.rand(r, kp, device="cuda", generator=g) * 2 - 1)[:, :k] if kp != k else \
            torch.rand(r, k, device="cuda", generator=g) * 2 - 1
    probs, wants = [], []
    C = [torch.zeros(n, mp, device="cuda") for _ in range(3)]
    ref = [torch.zeros(n, m, dtype=torch.float64, device="cuda") for _ in range(3)]
    specs = [((1,), (1,), ((1, 0),)), ((1, 1), (1, -1), ((1, 1), (-1, 2))), ((-1, 1), (1, 1), ((1, 0), (1, 2))),
             ((1, -1), (-1,), ((-1, 0), (1, 1), (1, 2)))]
    for asg, bsg, dsts in specs:
        aterms = [(s, mat(n)) for s in asg]
        bterms = [(s, mat(m)) for s in bsg]
        a = sum(s * x.double() for s, x in aterms)
        b = sum(s * x.double() for s, x in bterms)
        prod = a @ b.t()
        for s, d in dsts:
            ref[d] += s * prod
        probs.append((aterms, bterms, [(s, C[d]) for s, d in dsts]))
    _call(probs, n, m, k, mp)
    torch.cuda.synchronize()
    for d in range(3):
        got = C[d][:, :m].double()
        err = float((got - ref[d]).norm() / ref[d].norm())
        assert err < 1e-5, (d, err)
        if mp > m:
            assert bool((C[d][:, m:] == 0).all())   # nothing past the row end


def test_fused_rejects_bad_arguments():
    lib = nat.load()
    x = torch.zeros(64, 64, device="cuda")
    one = (ctypes.c_int32 * 1)(1)
    three = (ctypes.c_int32 * 1)(3)
    p = (ctypes.c_void_p * 2)(x.data_ptr(), x.data_ptr())
    sg = (ctypes.c_int32 * 2)(1, 1)
    d = (ctypes.c_void_p * 4)(x.data_ptr(), 0, 0, 0)
    s4 = (ctypes.c_int32 * 4)(1, 1, 1, 1)
    st = torch.cuda.current_stream().cuda_stream
    assert lib.paco_mm_tf32x3_fused(0, st, 1, three, p, sg, 64, one, p, sg, 64, one, d, s4, 64, 64, 64, 64) == nat.ERR_ARG
    mis = (ctypes.c_void_p * 2)(x.data_ptr() + 4, x.data_ptr())
    assert lib.paco_mm_tf32x3_fused(0, st, 1, one, mis, sg, 64, one, p, sg, 64, one, d, s4, 64, 60, 60, 60) == \
        nat.ERR_UNSUPPORTED


@pytest.mark.parametrize("shape", [(1, 1), (33, 65), (4096, 1000), (70000, 40)])
def test_transpose(shape):
    r, c = shape
    x = torch.randn(r, c, device="cuda")
    out = torch.full((c, r + 3), float("nan"), device="cuda")
    nat.check(nat.load().paco_transpose(0, torch.cuda.current_stream().cuda_stream, 4, out.data_ptr(), r + 3,
                                        x.data_ptr(), c, r, c))
    assert torch.equal(out[:, :r], x.t())
    assert bool(torch.isnan(out[:, r:]).all())


@pytest.mark.parametrize("n,base", [(512, 128), (2048, 512), (4096, 1024)])
def test_strassen_fused_producer_matches_split_path(n, base, monkeypatch):
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    b = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    ref = a.double() @ b.double()
    calls = []
    real = S._leaf_level_fused
    monkeypatch.setattr(S, "_leaf_level_fused", lambda *x: calls.append(1) or real(*x))
    monkeypatch.setattr(S, "LEAF_BF16X3", False)   # the 3xTF32 paths under test
    monkeypatch.setattr(S, "FUSED_PRODUCER", True)
    c1 = S.strassen_seq(a, b, n, base=base)
    assert calls, "fused-producer leaves not used"
    monkeypatch.setattr(S, "FUSED_PRODUCER", False)
    c2 = S.strassen_seq(a, b, n, base=base)
    e1 = float((c1.double() - ref).norm() / ref.norm())
    e2 = float((c2.double() - ref).norm() / ref.norm())
    assert e1 < 1e-5 and e2 < 1e-5, (e1, e2)
    # same sums, same hi/lo split, same MMAs: the two paths agree to fp32 rounding
    assert float((c1 - c2).norm() / c2.norm()) < 1e-6


def test_fused_rounding_bit_identical_to_split_path():
    """One product, one destination (a single fold: deterministic): the fused
    kernel's in-smem formation + integer tf32 rounding gives the split path's
    bits exactly (paco_tf32_split's cvt.rna.tf32 + paco_mm_tf32x3_multi)."""
    n = m = k = 512
    g = torch.Generator(device="cuda").manual_seed(77)
    a0, a1 = (torch.rand(n, k, device="cuda", generator=g) * 2 - 1 for _ in range(2))
    b0, b1 = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1 for _ in range(2))
    # include values whose tf32 rounding carries into the exponent and ties
    a0[0, :4] = torch.tensor([1.0 - 2 ** -24, 1.0 + 2 ** -11, -(1.0 + 3 * 2 ** -12), 2 ** -126], device="cuda")
    c_fused = torch.zeros(n, m, device="cuda")
    _call([([(1, a0), (-1, a1)], [(1, b0), (1, b1)], [(1, c_fused)])], n, m, k, m)
    lib = nat.load()
    st = torch.cuda.current_stream().cuda_stream
    ah, al = torch.empty(n, k, device="cuda"), torch.empty(n, k, device="cuda")
    bh, bl = torch.empty(m, k, device="cuda"), torch.empty(m, k, device="cuda")
    for (x0, x1, s1, hi, lo) in ((a0, a1, -1, ah, al), (b0, b1, 1, bh, bl)):
        ins = (ctypes.c_void_p * 2)(x0.data_ptr(), x1.data_ptr())
        lds = (ctypes.c_int64 * 2)(k, k)
        co = (ctypes.c_int32 * 2)(1, s1)
        nat.check(lib.paco_tf32_split(0, st, 2, ins, lds, co, x0.shape[0], k, 0, hi.data_ptr(), lo.data_ptr(), k))
    c_split = torch.zeros(n, m, device="cuda")
    one = lambda t: (ctypes.c_void_p * 1)(t.data_ptr())  # noqa: E731
    nat.check(lib.paco_mm_tf32x3_multi(0, st, 1, one(ah), one(al), k, one(bh), one(bl), k, (ctypes.c_int32 * 1)(1),
                                       (ctypes.c_void_p * 4)(c_split.data_ptr(), 0, 0, 0),
                                       (ctypes.c_int32 * 4)(1, 1, 1, 1), m, n, m, k))
    torch.cuda.synchronize()
    assert torch.equal(c_fused, c_split)


@pytest.mark.parametrize("shape", [(2048, 2048, 256, 4), (2000, 1800, 333, 8)])
def test_cta_pair_kernel_multi_destination(shape):
    """Batches big enough for the CTA-pair 3xTF32 kernel (tcgen05 cta_group::2:
    M = 256 per pair, each CTA holding half of B^T), ragged extents, two signed
    destinations per product; vs the float64 products."""
    n, m, k, cnt = shape
    lib = nat.load()
    st = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(n + cnt)
    kp = (k + 3) // 4 * 4
    a = [(torch.rand(n, kp, device="cuda", generator=g) * 2 - 1) for _ in range(cnt)]
    b = [(torch.rand(m, kp, device="cuda", generator=g) * 2 - 1) for _ in range(cnt)]
    for x in a + b:
        x[:, k:] = 0
    hl = []
    for x in a + b:
        h, lo = torch.empty_like(x), torch.empty_like(x)
        nat.check(lib.paco_tf32_split(0, st, 1, (ctypes.c_void_p * 1)(x.data_ptr()), (ctypes.c_int64 * 1)(kp),
                                      (ctypes.c_int32 * 1)(1), x.shape[0], k, 0, h.data_ptr(), lo.data_ptr(), kp))
        hl.append((h, lo))
    arr = lambda xs: (ctypes.c_void_p * cnt)(*[x.data_ptr() for x in xs])  # noqa: E731
    C = [torch.zeros(n, m, device="cuda") for _ in range(2)]
    ndst = (ctypes.c_int32 * cnt)(*[2] * cnt)
    dst = (ctypes.c_void_p * (4 * cnt))()
    sign = (ctypes.c_int32 * (4 * cnt))()
    ref = [torch.zeros(n, m, dtype=torch.float64, device="cuda") for _ in range(2)]
    for q in range(cnt):
        dst[4 * q], dst[4 * q + 1] = C[q % 2].data_ptr(), C[(q + 1) % 2].data_ptr()
        sign[4 * q], sign[4 * q + 1] = 1, (-1 if q % 2 else 1)
        p = a[q][:, :k].double() @ b[q][:, :k].double().t()
        ref[q % 2] += p
        ref[(q + 1) % 2] += -p if q % 2 else p
    nat.check(lib.paco_mm_tf32x3_multi(0, st, cnt, arr([x[0] for x in hl[:cnt]]), arr([x[1] for x in hl[:cnt]]), kp,
                                       arr([x[0] for x in hl[cnt:]]), arr([x[1] for x in hl[cnt:]]), kp, ndst, dst,
                                       sign, m, n, m, k))
    torch.cuda.synchronize()
    for i in range(2):
        assert float((C[i].double() - ref[i]).norm() / ref[i].norm()) < 1e-5, i


def test_strassen_pair_leaves_fused_a(monkeypatch):
    """8192 / base 2048: leaf batches of 7 x 64 pair tiles (>= 222) run on CTA pairs,
    S_r formed inside the kernel (FUSED_A) or split beforehand; both vs f64, and the
    two paths agree to fp32 rounding (same sums, same rounding, same MMAs)."""
    n, base = 8192, 2048
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    b = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    rows = torch.arange(0, n, 97, device="cuda")
    ref = a[rows].double() @ b.double()
    out = {}
    for fuse_a in (True, False):
        monkeypatch.setattr(S, "FUSED_A", fuse_a)
        c = S.strassen_seq(a, b, n, base=base)
        assert float((c[rows].double() - ref).norm() / ref.norm()) < 1e-4, fuse_a
        out[fuse_a] = c
    assert float((out[True] - out[False]).norm() / out[False].norm()) < 1e-6


@pytest.mark.parametrize("shape", [(2048, 2048, 512, 4), (2000, 1800, 333, 8)])
def test_tf32b2_pair_kernel_accuracy(shape):
    """The tf32 + 2 x bf16 format (paco_tf32b2_split + paco_mm_tf32b2_multi): hi*hi
    on tf32, hi*lo + lo*hi on bf16 MMAs, two signed destinations per product.
    Accuracy vs the f64 products must stay in the 3xTF32 class (<= 2x its error,
    and < 1e-5 absolute relative error), far inside cfg5's 1e-4."""
    n, m, k, cnt = shape
    lib = nat.load()
    st = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(k + cnt)
    kp = (k + 7) // 8 * 8   # 16-byte bf16 rows
    a = [(torch.rand(n, kp, device="cuda", generator=g) * 2 - 1) for _ in range(cnt)]
    b = [(torch.rand(m, kp, device="cuda", generator=g) * 2 - 1) for _ in range(cnt)]
    for x in a + b:
        x[:, k:] = 0

    def split3(x):
        hi = torch.zeros_like(x)
        h16 = torch.zeros(x.shape, dtype=torch.bfloat16, device="cuda")
        l16 = torch.zeros(x.shape, dtype=torch.bfloat16, device="cuda")
        nat.check(lib.paco_tf32b2_split(0, st, 1, (ctypes.c_void_p * 1)(x.data_ptr()), (ctypes.c_int64 * 1)(kp),
                                        (ctypes.c_int32 * 1)(1), x.shape[0], k, 0, hi.data_ptr(), h16.data_ptr(),
                                        l16.data_ptr(), kp))
        return hi, h16, l16
    sa, sb = [split3(x) for x in a], [split3(x) for x in b]
    # the format itself: hi is tf32 (13 low bits zero), hi + lo reproduces x to bf16(lo)'s precision
    hi0 = sa[0][0]
    assert int((hi0.view(torch.int32) & 0x1FFF).abs().sum()) == 0
    rec = hi0[:, :k].double() + sa[0][2][:, :k].double()
    assert float((rec - a[0][:, :k].double()).abs().max()) <= 2.0 ** -19
    arr = lambda xs: (ctypes.c_void_p * cnt)(*[x.data_ptr() for x in xs])  # noqa: E731
    C = [torch.zeros(n, m, device="cuda") for _ in range(2)]
    ndst = (ctypes.c_int32 * cnt)(*[2] * cnt)
    dst = (ctypes.c_void_p * (4 * cnt))()
    sign = (ctypes.c_int32 * (4 * cnt))()
    ref = [torch.zeros(n, m, dtype=torch.float64, device="cuda") for _ in range(2)]
    for q in range(cnt):
        dst[4 * q], dst[4 * q + 1] = C[q % 2].data_ptr(), C[(q + 1) % 2].data_ptr()
        sign[4 * q], sign[4 * q + 1] = 1, (-1 if q % 2 else 1)
        p = a[q][:, :k].double() @ b[q][:, :k].double().t()
        ref[q % 2] += p
        ref[(q + 1) % 2] += -p if q % 2 else p
    nat.check(lib.paco_mm_tf32b2_multi(0, st, cnt, arr([x[0] for x in sa]), arr([x[1] for x in sa]),
                                       arr([x[2] for x in sa]), kp, arr([x[0] for x in sb]), arr([x[1] for x in sb]),
                                       arr([x[2] for x in sb]), kp, ndst, dst, sign, m, n, m, k))
    torch.cuda.synchronize()
    for i in range(2):
        assert float((C[i].double() - ref[i]).norm() / ref[i].norm()) < 1e-5, i


@pytest.mark.parametrize("cv,raw", [(False, False), (True, False), (True, True)])
def test_strassen_tf32b2_vs_3xtf32(monkeypatch, cv, raw):
    """cfg5's shape at half size (8192, 2 levels): the tf32 + 2 x bf16 leaves vs the
    3xTF32 leaves -- both within 1e-4 of the f64 product, and the tf32b2 error no
    more than 1.5x the 3xTF32 one (Strassen's fp32 formation dominates both)."""
    n, base = 8192, 2048
    g = torch.Generator(device="cuda").manual_seed(8)
    a = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    b = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    rows = torch.arange(0, n, 61, device="cuda")
    ref = a[rows].double() @ b.double()
    err = {}
    monkeypatch.setattr(S, "LEAF_BF16X3", False)   # the formats under test, not the bf16x3 default
    monkeypatch.setattr(S, "TF32B2_CONVERT", cv)
    monkeypatch.setattr(S, "TF32B2_RAW", raw)
    for b2 in (True, False):
        monkeypatch.setattr(S, "TF32B2", b2)
        c = S.strassen_seq(a, b, n, base=base)
        err[b2] = float((c[rows].double() - ref).norm() / ref.norm())
    assert err[True] < 1e-4 and err[False] < 1e-4, err
    assert err[True] <= 1.5 * err[False], err


@pytest.mark.parametrize("shape", [(64, 64), (257, 1028), (4096, 4096)])
def test_lincomb_multi(shape):
    """paco_lincomb_multi: several signed sums of the same inputs in one pass
    (Strassen's S1, S2, S5, S6, S7 from four quadrants), exact vs torch."""
    n, m = shape
    lib = nat.load()
    g = torch.Generator(device="cuda").manual_seed(n)
    big = torch.randn(2 * n, 2 * m + 8, device="cuda", generator=g)   # quadrant views with a padded pitch
    q = [big[:n, :m], big[:n, m:2 * m], big[n:, :m], big[n:, m:2 * m]]
    rows = [[1, 0, 0, 1], [0, 0, 1, 1], [1, 1, 0, 0], [-1, 0, 1, 0], [0, 1, 0, -1]]
    outs = [torch.full((n, m + 4), float("nan"), device="cuda")[:, :m] for _ in rows]
    nat.check(lib.paco_lincomb_multi(0, torch.cuda.current_stream().cuda_stream, n, m, 4,
                                     (ctypes.c_void_p * 4)(*[x.data_ptr() for x in q]),
                                     (ctypes.c_int64 * 4)(*[x.stride(0) for x in q]), len(rows),
                                     (ctypes.c_void_p * len(rows))(*[o.data_ptr() for o in outs]),
                                     (ctypes.c_int64 * len(rows))(*[o.stride(0) for o in outs]),
                                     (ctypes.c_int32 * 20)(*[c for r in rows for c in r])))
    torch.cuda.synchronize()
    for o, r in zip(outs, rows):
        want = sum(c * x for c, x in zip(r, q) if c)
        assert torch.equal(o, want)
