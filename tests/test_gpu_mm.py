"""GPU parity of the sm_100a semiring kernels against the reference's own results.

Every test calls through the public API (-> C ABI -> CUDA) and compares with
(a) golden fixtures produced by the reference itself (tests/golden/), and
(b) the CPU oracle (oracle/semiring_ref.c) on seeded inputs.  Integer and
tropical semirings must match bit for bit; floating point within the stated
relative tolerance.
"""

import numpy as np
import pytest
import torch

from oracle import cref
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

pytestmark = pytest.mark.gpu

INF = 2**30


def tropical(rng, shape, lo, hi, inf_frac=0.0, inf=INF):
    x = rng.integers(lo, hi, shape, dtype=np.int32)
    if inf_frac:
        x[rng.random(shape) < inf_frac] = inf
    return x


# ---------------------------------------------------------------- golden vectors

def test_cfg1_full_paco_p3_matches_reference(golden_cases):
    A, B, want = golden_cases["cfg1_A"], golden_cases["cfg1_B"], golden_cases["cfg1_C"]
    plan = M.mm_paco_partition(384, 320, 256, 3)
    for mode in ("serial_sim", "parallel"):
        C = np.zeros((384, 320), np.int64)
        rep = M.mm_execute(plan, A, B, C, M.SEMIRING_INT, mode=mode)
        assert np.array_equal(C, want), mode
        assert rep.work_total == 384 * 320 * 256 + sum(
            t.cost_work for t in plan.tasks if t.kind == "reduce")
    # int64 operands take the wide int64 kernel: same answer
    C = np.zeros((384, 320), np.int64)
    M.mm_execute(plan, A.astype(np.int64), B.astype(np.int64), C, M.SEMIRING_INT)
    assert np.array_equal(C, want)


def test_minplus_sat_golden(golden_cases):
    for tag in ("minplus_sat", "minplus_inf"):
        A, B, want = golden_cases[f"{tag}_A"], golden_cases[f"{tag}_B"], golden_cases[f"{tag}_C"]
        n, k = A.shape
        m = B.shape[1]
        for p in (1, 3, 5, 7):
            C = np.full((n, m), INF, np.int32)
            M.mm_execute(M.mm_one_piece_partition(n, m, k, p), A, B, C, M.SEMIRING_MINPLUS_SAT)
            assert np.array_equal(C, want), (tag, p)
        C = np.full((n, m), INF, np.int32)
        M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT)
        assert np.array_equal(C, want), tag


def test_maxplus_golden(golden_cases):
    A, B, want = golden_cases["maxplus_A"], golden_cases["maxplus_B"], golden_cases["maxplus_C"]
    n, k = A.shape
    m = B.shape[1]
    for p in (1, 2, 3, 5, 7, 8):
        C = np.full((n, m), -INF, np.int32)
        M.mm_execute(M.mm_one_piece_partition(n, m, k, p), A, B, C, M.SEMIRING_MAXPLUS)
        assert np.array_equal(C, want), p


def test_reference_minplus_int64_with_wrap(golden_cases):
    A, B, want = golden_cases["minplus_i64_A"], golden_cases["minplus_i64_B"], golden_cases["minplus_i64_C"]
    n, k = A.shape
    m = B.shape[1]
    C = np.full((n, m), M.MINPLUS_INF, np.int64)
    M.mm_execute(M.mm_paco_partition(n, m, k, 3), A, B, C, M.SEMIRING_MINPLUS)
    assert np.array_equal(C, want)


def test_int64_ring_wraps_like_numpy(golden_cases):
    g = golden_cases
    C = g["int_wrap_C0"].copy()
    n, k = g["int_wrap_A"].shape
    m = g["int_wrap_B"].shape[1]
    M.mm_execute(M.mm_one_piece_partition(n, m, k, 5), g["int_wrap_A"], g["int_wrap_B"], C, M.SEMIRING_INT)
    assert np.array_equal(C, g["int_wrap_C"])


def test_f64_golden(golden_cases):
    g = golden_cases
    C = g["f64_C0"].copy()
    n, k = g["f64_A"].shape
    m = g["f64_B"].shape[1]
    M.mm_execute(M.mm_one_piece_partition(n, m, k, 3), g["f64_A"], g["f64_B"], C, M.SEMIRING_F64)
    np.testing.assert_allclose(C, g["f64_C"], rtol=1e-12, atol=1e-12)


def test_bf16_golden(golden_cases):
    g = golden_cases
    a = torch.from_numpy(g["bf16_A"]).cuda().to(torch.bfloat16)
    b = torch.from_numpy(g["bf16_B"]).cuda().to(torch.bfloat16)
    # the fixture operands are exactly bf16-representable
    assert torch.equal(a.float().cpu(), torch.from_numpy(g["bf16_A"]))
    c = torch.zeros(a.shape[0], b.shape[1], device="cuda")
    M.mm_seq(a, b, c, M.SEMIRING_BF16)
    ref = g["bf16_C"]
    err = np.linalg.norm(c.cpu().numpy().astype(np.float64) - ref) / np.linalg.norm(ref)
    assert err <= 1e-2  # BASELINE cfg3 tolerance; fp32 accumulation gives ~1e-7
    assert err < 1e-5


# ---------------------------------------------------------------- oracle sweeps

SHAPES = [(1, 1, 1), (1, 7, 3), (5, 1, 9), (3, 4, 1), (31, 33, 35), (128, 128, 32),
          (129, 127, 33), (200, 300, 257), (257, 129, 1000), (64, 1024, 48), (1030, 70, 520)]


@pytest.mark.parametrize("shape", SHAPES)
def test_minplus_sat_vs_oracle(shape):
    n, m, k = shape
    rng = np.random.default_rng(n * 7 + m * 3 + k)
    A = tropical(rng, (n, k), 0, 2**20, 0.1)
    B = tropical(rng, (k, m), 0, 2**20, 0.1)
    C0 = tropical(rng, (n, m), 0, 2**21, 0.5)
    want = cref.mm(cref.SR_MINPLUS_SAT32, A, B, C0.copy())
    C = C0.copy()
    M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT)
    assert np.array_equal(C, want)


@pytest.mark.parametrize("shape", SHAPES)
def test_maxplus_vs_oracle(shape):
    n, m, k = shape
    rng = np.random.default_rng(n * 5 + m * 11 + k)
    A = tropical(rng, (n, k), -2**20, 2**20, 0.05, -INF)
    B = tropical(rng, (k, m), -2**20, 2**20, 0.05, -INF)
    C0 = np.full((n, m), -INF, np.int32)
    want = cref.mm(cref.SR_MAXPLUS_SAT32, A, B, C0.copy())
    C = C0.copy()
    M.mm_seq(A, B, C, M.SEMIRING_MAXPLUS)
    assert np.array_equal(C, want)


@pytest.mark.parametrize("shape", SHAPES)
def test_int32_to_int64_vs_oracle(shape):
    n, m, k = shape
    rng = np.random.default_rng(n + m + k)
    A = rng.integers(-2**31, 2**31, (n, k), dtype=np.int64).astype(np.int32)
    B = rng.integers(-2**31, 2**31, (k, m), dtype=np.int64).astype(np.int32)
    C0 = rng.integers(-2**62, 2**62, (n, m), dtype=np.int64)
    want = cref.mm(cref.SR_INT_I32_I64, A, B, C0.copy())
    C = C0.copy()
    M.mm_seq(A, B, C, M.SEMIRING_INT)
    assert np.array_equal(C, want)


@pytest.mark.parametrize("shape", SHAPES[:8] + [(1000, 513, 777)])
@pytest.mark.parametrize("sr", ["tc", "simt"])
def test_f32_vs_oracle(shape, sr):
    """float32 (+,x): 3xTF32 tensor cores and FFMA, relative Frobenius <= 1e-5 vs f64."""
    n, m, k = shape
    rng = np.random.default_rng(n * 3 + k)
    A = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    B = rng.uniform(-1, 1, (k, m)).astype(np.float32)
    C0 = rng.uniform(-1, 1, (n, m)).astype(np.float32)
    C = C0.copy()
    M.mm_seq(A, B, C, M.SEMIRING_F32 if sr == "tc" else M.SEMIRING_F32_SIMT)
    ref = A.astype(np.float64) @ B.astype(np.float64) + C0
    assert np.linalg.norm(C - ref) <= 1e-5 * np.linalg.norm(ref)


def test_unaligned_views_and_ldc():
    """Sub-views at odd offsets take the element-granular load path."""
    rng = np.random.default_rng(5)
    big_a = torch.from_numpy(tropical(rng, (301, 403), 0, 2**20, 0.1)).cuda()
    big_b = torch.from_numpy(tropical(rng, (411, 299), 0, 2**20, 0.1)).cuda()
    big_c = torch.full((305, 307), INF, dtype=torch.int32, device="cuda")
    a = big_a[3:203, 5:390]      # 200 x 385, misaligned base
    b = big_b[7:392, 1:258]      # 385 x 257
    c = big_c[1:201, 9:266]      # 200 x 257
    want = cref.mm(cref.SR_MINPLUS_SAT32, a.cpu().numpy(), b.cpu().numpy(), c.cpu().numpy().copy())
    M.mm_seq(a, b, c, M.SEMIRING_MINPLUS_SAT)
    assert np.array_equal(c.cpu().numpy(), want)
    # untouched border of C stays INF
    assert int(big_c[0].min()) == INF and int(big_c[:, :9].min()) == INF


def test_cta_plan_overrides_and_ksplit_atomics():
    """Explicit CTA-level pieces, including k-split pieces folded by atomics."""
    rng = np.random.default_rng(11)
    n, m, k = 256, 384, 320
    A = tropical(rng, (n, k), 0, 2**20, 0.1)
    B = tropical(rng, (k, m), 0, 2**20, 0.1)
    want = cref.mm(cref.SR_MINPLUS_SAT32, A, B, np.full((n, m), INF, np.int32))
    bm, bn, bk, _ = nat.tile_shape(nat.SR_MINPLUS_SAT32)
    nt, mt, kt = -(-n // bm), -(-m // bn), -(-k // bk)
    for p in (1, 2, 3, 5, 7, 13, 20):
        plan = M.mm_one_piece_partition(nt, mt, kt, p)
        pieces = [(c.region.i0, c.region.j0, c.region.l0, c.region.n, c.region.m, c.region.k)
                  for c in plan.compute_tasks()]
        C = np.full((n, m), INF, np.int32)
        M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT, pieces=pieces)
        assert np.array_equal(C, want), p


def test_overwrite_mode_does_not_read_c():
    rng = np.random.default_rng(12)
    A = tropical(rng, (130, 70), 0, 2**20)
    B = tropical(rng, (70, 90), 0, 2**20)
    want = cref.mm(cref.SR_MINPLUS_SAT32, A, B, np.full((130, 90), INF, np.int32))
    c = torch.full((130, 90), -123, dtype=torch.int32, device="cuda")  # garbage C
    M.mm_seq(A, B, c, M.SEMIRING_MINPLUS_SAT, overwrite=True)
    assert np.array_equal(c.cpu().numpy(), want)


def test_empty_k_and_empty_output():
    A = np.zeros((4, 0), np.int32)
    B = np.zeros((0, 5), np.int32)
    C = np.full((4, 5), 7, np.int32)
    M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT)
    assert (C == 7).all()
    C = np.zeros((0, 5), np.int32)
    M.mm_seq(np.zeros((0, 3), np.int32), np.zeros((3, 5), np.int32), C, M.SEMIRING_MINPLUS_SAT)
    for sem, dt in ((M.SEMIRING_F32, torch.float32), (M.SEMIRING_BF16, torch.bfloat16),
                    (M.SEMIRING_INT, torch.int64), (M.SEMIRING_MAXPLUS, torch.int32)):
        a = torch.zeros((6, 0), dtype=dt, device="cuda")
        b = torch.zeros((0, 9), dtype=dt, device="cuda")
        c = torch.full((6, 9), 3, dtype=torch.float32 if dt.is_floating_point else dt, device="cuda")
        M.mm_seq(a, b, c, sem)
        assert bool((c == 3).all()), sem.name
        M.mm_seq(a, b, c, sem, overwrite=True)       # C = zero of the semiring
        assert bool((c == sem.zero).all()), sem.name


def test_device_oracle_matches_cpu_oracle():
    rng = np.random.default_rng(13)
    A = tropical(rng, (70, 90), 0, 2**20, 0.2)
    B = tropical(rng, (90, 50), 0, 2**20, 0.2)
    want = cref.mm(cref.SR_MINPLUS_SAT32, A, B, np.full((70, 50), INF, np.int32))
    assert np.array_equal(M.mm_oracle(A, B, M.SEMIRING_MINPLUS_SAT), want)
    A64 = rng.integers(-100, 100, (33, 44))
    B64 = rng.integers(-100, 100, (44, 55))
    assert np.array_equal(M.mm_oracle(A64, B64, M.SEMIRING_INT), A64 @ B64)


def test_shape_mismatch_raises_value_error():
    with pytest.raises(ValueError, match="shape mismatch"):
        M.mm_seq(np.zeros((3, 4), np.int32), np.zeros((5, 6), np.int32), np.zeros((3, 6), np.int64))


def test_paco_plans_every_p_minplus_i64():
    rng = np.random.default_rng(21)
    n, m, k = 70, 50, 90
    A = rng.integers(0, 1000, (n, k), dtype=np.int64)
    B = rng.integers(0, 1000, (k, m), dtype=np.int64)
    want = cref.mm(cref.SR_MINPLUS_I64, A, B, np.full((n, m), M.MINPLUS_INF, np.int64))
    for p in (1, 2, 3, 5, 7, 12, 13):
        for plan in (M.mm_paco_partition(n, m, k, p), M.mm_one_piece_partition(n, m, k, p)):
            C = np.full((n, m), M.MINPLUS_INF, np.int64)
            M.mm_execute(plan, A, B, C, M.SEMIRING_MINPLUS, mode="parallel")
            assert np.array_equal(C, want), (p, plan.meta["variant"])


@pytest.mark.parametrize("paco_plan", [False, True])
def test_device_derived_cta_plan_matches_host_plan(paco_plan):
    """Each CTA derives its piece on device; it must equal the host's plan
    (tile grid: paco_cta_grid; PACO_MM_PACO_PLAN: paco_plan_cta)."""
    lib = nat.load()
    rng = np.random.default_rng(31)
    # (3963, 1007, 1024): 248 ragged tiles, the last 100 split 4 ways in k (tail split)
    for (n, m, k) in [(1000, 700, 900), (300, 4000, 129), (2048, 2048, 2048), (200, 150, 3000), (3963, 1007, 1024)]:
        A = torch.from_numpy(tropical(rng, (n, k), 0, 2**20)).cuda()
        B = torch.from_numpy(tropical(rng, (k, m), 0, 2**20)).cuda()
        C = torch.full((n, m), INF, dtype=torch.int32, device="cuda")
        tr = torch.zeros(10 * 8192, dtype=torch.int64, device="cuda")
        nat.check(lib.paco_debug_trace(tr.data_ptr()))
        try:
            launch_mm(nat.SR_MINPLUS_SAT32, torch.cuda.current_stream(), View.of(A), View.of(B), View.of(C),
                        flags=nat.MM_PACO_PLAN if paco_plan else 0)
            torch.cuda.synchronize()
        finally:
            nat.check(lib.paco_debug_trace(None))
        t = tr.view(-1, 10).cpu().numpy()
        t = t[t[:, 2] > 0]
        host = (nat.plan_cta(nat.SR_MINPLUS_SAT32, n, m, k, len(t)) if paco_plan
                else nat.grid_pieces(nat.SR_MINPLUS_SAT32, n, m, k))
        assert [tuple(r) for r in t[:, 4:10]] == [tuple(h) for h in host]
        want = cref.mm(cref.SR_MINPLUS_SAT32, A.cpu().numpy(), B.cpu().numpy(), np.full((n, m), INF, np.int32))
        assert np.array_equal(C.cpu().numpy(), want)


def test_pinned_host_pipeline_matches_oracle():
    """Pinned host operands take the overlapped H2D/compute/D2H path."""
    rng = np.random.default_rng(41)
    n, m, k = 1500, 700, 333
    A = torch.from_numpy(tropical(rng, (n, k), 0, 2**20, 0.1)).pin_memory()
    B = torch.from_numpy(tropical(rng, (k, m), 0, 2**20, 0.1)).pin_memory()
    C0 = tropical(rng, (n, m), 0, 2**21, 0.3)
    C = torch.from_numpy(C0.copy()).pin_memory()
    M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT)
    want = cref.mm(cref.SR_MINPLUS_SAT32, A.numpy(), B.numpy(), C0.copy())
    assert np.array_equal(C.numpy(), want)
    C2 = torch.full((n, m), 12345, dtype=torch.int32).pin_memory()
    M.mm_seq(A, B, C2, M.SEMIRING_MINPLUS_SAT, overwrite=True)
    want2 = cref.mm(cref.SR_MINPLUS_SAT32, A.numpy(), B.numpy(), np.full((n, m), INF, np.int32))
    assert np.array_equal(C2.numpy(), want2)


def test_numpy_host_pipeline_short_k_matches_oracle(monkeypatch):
    """Pageable NumPy operands with a short k: staged row-blocked pipeline."""
    from paper_2011_01441_b200 import mm as MMmod
    calls = []
    real = MMmod._kphased_host_mm
    monkeypatch.setattr(MMmod, "_kphased_host_mm", lambda *a, **kw: calls.append(kw) or real(*a, **kw))
    rng = np.random.default_rng(42)
    n, m, k = 1500, 700, 333
    A = tropical(rng, (n, k), 0, 2**20, 0.1)
    B = tropical(rng, (k, m), 0, 2**20, 0.1)
    C0 = tropical(rng, (n, m), 0, 2**21, 0.3)
    for overwrite in (False, True):
        C = C0.copy() if not overwrite else np.full((n, m), 12345, np.int32)
        M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT, overwrite=overwrite)
        want = cref.mm(cref.SR_MINPLUS_SAT32, A, B, C0.copy() if not overwrite else np.full((n, m), INF, np.int32))
        assert np.array_equal(C, want), overwrite
    assert len(calls) == 2 and all(c.get("front_share") == 0.0 for c in calls)


@pytest.mark.parametrize("sr", ["minplus", "maxplus", "int", "f32", "bf16"])
@pytest.mark.parametrize("overwrite", [False, True])
@pytest.mark.parametrize("host", ["pinned", "numpy"])
def test_host_k_phased_pipeline(sr, overwrite, host, monkeypatch):
    """Long-k host operands -- pinned torch tensors, or pageable NumPy arrays staged
    through pinned buffers by host threads -- take the k-first / rows-last
    pipeline; same C as the oracle."""
    if host == "numpy" and sr == "bf16":
        pytest.skip("NumPy has no bfloat16")
    from paper_2011_01441_b200 import mm as MMmod
    rng = np.random.default_rng(43)
    n, m, k = 1100, 650, 2600
    assert MMmod._kphased_edges(k)[1] < k
    if sr in ("minplus", "maxplus"):
        lo, hi = (0, 2**20) if sr == "minplus" else (-2**20, 2**20)
        A = tropical(rng, (n, k), lo, hi, 0.1 if sr == "minplus" else 0.0)
        B = tropical(rng, (k, m), lo, hi, 0.1 if sr == "minplus" else 0.0)
        C0 = tropical(rng, (n, m), lo, 2**21, 0.3 if sr == "minplus" else 0.0)
        sem, cid = ((M.SEMIRING_MINPLUS_SAT, cref.SR_MINPLUS_SAT32) if sr == "minplus"
                    else (M.SEMIRING_MAXPLUS, cref.SR_MAXPLUS_SAT32))
        zero = INF if sr == "minplus" else -INF
    elif sr == "int":
        A = rng.integers(-50, 50, (n, k)).astype(np.int64)
        B = rng.integers(-50, 50, (k, m)).astype(np.int64)
        C0 = rng.integers(-1000, 1000, (n, m)).astype(np.int64)
        sem, cid, zero = M.SEMIRING_INT, cref.SR_INT_I64, 0
    else:
        A = rng.uniform(-1, 1, (n, k)).astype(np.float32)
        B = rng.uniform(-1, 1, (k, m)).astype(np.float32)
        if sr == "bf16":
            A = torch.from_numpy(A).to(torch.bfloat16).float().numpy()
            B = torch.from_numpy(B).to(torch.bfloat16).float().numpy()
        C0 = rng.uniform(-1, 1, (n, m)).astype(np.float32)
        sem, zero = (M.SEMIRING_F32 if sr == "f32" else M.SEMIRING_BF16), 0.0
    if overwrite:
        C0 = np.full((n, m), zero, C0.dtype)
    calls = []
    real = MMmod._kphased_host_mm
    monkeypatch.setattr(MMmod, "_kphased_host_mm", lambda *a, **kw: calls.append(1) or real(*a, **kw))
    if sr == "int":
        monkeypatch.setattr(MMmod, "NARROW_MIN_TERMS", 1 << 62)  # the int64 kernel's own pipeline
    if host == "numpy":
        Ah, Bh = A.copy(), B.copy()
        C = np.full(C0.shape, 7, C0.dtype) if overwrite else C0.copy()
    else:
        Ah, Bh = torch.from_numpy(A), torch.from_numpy(B)
        if sr == "bf16":
            Ah, Bh = Ah.to(torch.bfloat16), Bh.to(torch.bfloat16)
        Ah, Bh = Ah.pin_memory(), Bh.pin_memory()
        C = torch.full(C0.shape, 7, dtype=torch.from_numpy(C0).dtype).pin_memory() if overwrite \
            else torch.from_numpy(C0.copy()).pin_memory()
    M.mm_seq(Ah, Bh, C, sem, overwrite=overwrite)
    got = C if host == "numpy" else C.numpy()
    assert calls, "host pipeline not taken"
    if sr in ("f32", "bf16"):
        want = C0.astype(np.float64) + A.astype(np.float64) @ B.astype(np.float64)
        err = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert err <= (1e-5 if sr == "f32" else 1e-5), err   # exact-bf16 inputs, f32 accumulation
    else:
        want = cref.mm(cid, A, B, C0.copy())
        assert np.array_equal(got, want)


@pytest.mark.parametrize("fused", [True, False])
def test_fused_and_explicit_folds_agree(fused):
    """k-cut plans: epilogue-fused folds (no temps) and explicit REDUCE folds give the reference C."""
    rng = np.random.default_rng(51)
    n, m, k = 150, 130, 700                      # k-heavy: every plan below cuts k
    A = tropical(rng, (n, k), 0, 2**20, 0.1)
    B = tropical(rng, (k, m), 0, 2**20, 0.1)
    C0 = tropical(rng, (n, m), 0, 2**21, 0.5)
    want = cref.mm(cref.SR_MINPLUS_SAT32, A, B, C0.copy())
    for p in (2, 3, 5, 7, 8):
        for plan in (M.mm_one_piece_partition(n, m, k, p), M.mm_paco_partition(n, m, k, p, base=64)):
            assert plan.meta["reduces"], (p, plan.meta["variant"])
            C = C0.copy()
            M.mm_execute(plan, A, B, C, M.SEMIRING_MINPLUS_SAT, mode="parallel", fused_folds=fused)
            assert np.array_equal(C, want), (p, plan.meta["variant"], fused)
    # int64 ring (wide kernel, element atomics) and f64 (order-free within tolerance)
    A64 = rng.integers(-1000, 1000, (n, k)).astype(np.int64)
    B64 = rng.integers(-1000, 1000, (k, m)).astype(np.int64)
    C = np.zeros((n, m), np.int64)
    M.mm_execute(M.mm_paco_partition(n, m, k, 5, base=64), A64, B64, C, M.SEMIRING_INT, fused_folds=fused)
    assert np.array_equal(C, A64 @ B64)
    Af, Bf = rng.standard_normal((n, k)), rng.standard_normal((k, m))
    C = np.zeros((n, m))
    M.mm_execute(M.mm_one_piece_partition(n, m, k, 7), Af, Bf, C, M.SEMIRING_F64, fused_folds=fused)
    np.testing.assert_allclose(C, Af @ Bf, rtol=1e-11, atol=1e-9)


def test_hetero_plan_from_measured_weights():
    """Throughput-weighted one-piece plan (matmul.py:303-339) driven by the live ALU probe."""
    w = M.measured_weights([0, 0, 0])
    assert len(w) == 3 and all(x > 0 for x in w)
    rng = np.random.default_rng(61)
    n, m, k = 300, 200, 260
    A = tropical(rng, (n, k), 0, 2**20, 0.1)
    B = tropical(rng, (k, m), 0, 2**20, 0.1)
    want = cref.mm(cref.SR_MINPLUS_SAT32, A, B, np.full((n, m), INF, np.int32))
    for weights in (w, (3.0, 1.0, 1.0), (1.0, 2.0)):
        C = np.full((n, m), INF, np.int32)
        M.mm_execute(M.mm_hetero_partition(n, m, k, weights), A, B, C, M.SEMIRING_MINPLUS_SAT, mode="parallel")
        assert np.array_equal(C, want), weights


@pytest.mark.parametrize("sr", ["f32", "bf16"])
def test_tensor_core_plans_on_concurrent_streams(sr):
    """Plan workers launch the tcgen05 kernels concurrently on their own streams;
    each launch's split/repack scratch is its own (regression: a shared
    per-device scratch raced under mode='parallel')."""
    rng = np.random.default_rng(77)
    n, m, k = 200, 150, 300
    A = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    B = rng.uniform(-1, 1, (k, m)).astype(np.float32)
    if sr == "bf16":
        a = torch.from_numpy(A).cuda().to(torch.bfloat16)
        b = torch.from_numpy(B).cuda().to(torch.bfloat16)
        A, B = a.float().cpu().numpy(), b.float().cpu().numpy()
        sem = M.SEMIRING_BF16
    else:
        a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        sem = M.SEMIRING_F32
    ref = A.astype(np.float64) @ B.astype(np.float64)
    for p in (3, 5, 7):
        for plan in (M.mm_paco_partition(n, m, k, p, base=16), M.mm_one_piece_partition(n, m, k, p)):
            for _ in range(3):
                C = torch.zeros((n, m), device="cuda")
                M.mm_execute(plan, a, b, C, sem, mode="parallel")
                got = C.cpu().numpy().astype(np.float64)
                assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref), (p, plan.meta["variant"])


@pytest.mark.parametrize("sr", ["f32", "bf16"])
@pytest.mark.parametrize("offs", [(0, 1, 1), (3, 5, 7), (1, 0, 2)])
def test_tensor_core_misaligned_views(sr, offs):
    """tcgen05 operands / C whose first element is not 16-byte aligned are
    repacked through scratch (TMA boxes must start 16-byte aligned)."""
    ri, rl, rj = offs
    g = torch.Generator(device="cuda").manual_seed(sum(offs))
    dt = torch.float32 if sr == "f32" else torch.bfloat16
    big_a = (torch.rand(300, 300, device="cuda", generator=g) * 2 - 1).to(dt)
    big_b = (torch.rand(300, 300, device="cuda", generator=g) * 2 - 1).to(dt)
    big_c = torch.rand(300, 300, device="cuda", generator=g)
    n, k, m = 139, 96, 171
    a, b = big_a[ri:ri + n, rl:rl + k], big_b[rl:rl + k, rj:rj + m]
    c = big_c[ri:ri + n, rj:rj + m]
    c0 = c.clone()
    M.mm_seq(a, b, c, M.SEMIRING_F32 if sr == "f32" else M.SEMIRING_BF16)
    ref = c0.double() + a.double() @ b.double()
    assert float((c.double() - ref).norm() / ref.norm()) < 1e-5
    outside = big_c.clone()
    outside[ri:ri + n, rj:rj + m] = 0
    assert torch.count_nonzero(outside[ri:ri + n, :rj]) == rj * n  # neighbours untouched


@pytest.mark.parametrize("fused", [None, False])
def test_plan_as_one_batched_launch(fused):
    """mm_execute on one device runs the plan's COMPUTE cuboids as one
    paco_mm_batch launch (explicit REDUCE folds after it): same C as per-task
    launches and as the oracle, for one-piece and multi-piece plans."""
    rng = np.random.default_rng(61)
    n, m, k = 333, 290, 701
    A = tropical(rng, (n, k), 0, 2**20, 0.1)
    B = tropical(rng, (k, m), 0, 2**20, 0.1)
    C0 = tropical(rng, (n, m), 0, 2**21, 0.3)
    want = cref.mm(cref.SR_MINPLUS_SAT32, A, B, C0.copy())
    for p in (3, 5, 8, 13):
        for plan in (M.mm_one_piece_partition(n, m, k, p), M.mm_paco_partition(n, m, k, p, base=32)):
            for batch in (True, False):
                C = C0.copy()
                M.mm_execute(plan, A, B, C, M.SEMIRING_MINPLUS_SAT, mode="parallel", fused_folds=fused,
                             batch=batch)
                assert np.array_equal(C, want), (p, plan.meta["variant"], batch)
    # int (+,x) with k-cuts, int32 operands -> int64
    Ai = rng.integers(-100, 100, (n, k)).astype(np.int32)
    Bi = rng.integers(-100, 100, (k, m)).astype(np.int32)
    C = np.zeros((n, m), np.int64)
    M.mm_execute(M.mm_paco_partition(n, m, k, 7, base=32), Ai, Bi, C, M.SEMIRING_INT, fused_folds=fused)
    assert np.array_equal(C, Ai.astype(np.int64) @ Bi.astype(np.int64))


@pytest.mark.parametrize("style", ["fused", "stage"])
def test_remote_worker_paths(style):
    """mm_execute's paths for workers on another GPU -- fused (the epilogue folds
    into the home C with atomics) and staged (local block -> one copy -> atomic
    fold) -- forced on for every worker of the single test GPU
    (mm._REMOTE_ALL, in a fresh process)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, os.path.join(here, "stage_all_check.py"), style], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "stage-all ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_tensor_core_call_from_fresh_thread():
    """The first CUDA call of a new host thread may be a tcgen05 paco_mm (its
    tensor maps use the driver API, which needs the primary context current on
    that thread -- use_device() makes it so)."""
    import threading
    a = torch.randn(300, 200, device="cuda").to(torch.bfloat16)
    b = torch.randn(200, 260, device="cuda").to(torch.bfloat16)
    c = torch.zeros(300, 260, device="cuda")
    torch.cuda.synchronize()
    errs = []

    def work():
        try:
            nat.check(nat.load().paco_mm(0, None, nat.SR_BF16_F32, a.data_ptr(), a.stride(0), b.data_ptr(),
                                         b.stride(0), c.data_ptr(), c.stride(0), 300, 260, 200, None, 0,
                                         nat.MM_OVERWRITE))
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    t = threading.Thread(target=work)
    t.start()
    t.join()
    torch.cuda.synchronize()
    assert not errs, errs
    ref = a.double() @ b.double()
    assert float((c.double() - ref).norm() / ref.norm()) < 1e-5


@pytest.mark.parametrize("warm", [False, True])
def test_tensor_core_launches_in_cuda_graph(warm):
    """tcgen05 launches captured into a CUDA graph (first use of the stream
    inside the capture, or after eager launches on it) replay correctly, and
    back-to-back launches on one stream reuse the self-resetting tile counters
    (different shapes / group counts in a row)."""
    g = torch.Generator(device="cuda").manual_seed(5)
    shapes = [(1000, 256, 1024), (777, 96, 300), (4096, 512, 2048)]   # (n, k, m): resident and streaming kinds
    ops = []
    for n, k, m in shapes:
        a = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
        b = torch.randn(k, m, device="cuda", generator=g).to(torch.bfloat16)
        ops.append((a, b, torch.zeros(n, m, device="cuda"), a.double() @ b.double()))
    st = torch.cuda.Stream()

    def run():
        for a, b, c, _ in ops:
            launch_mm(nat.SR_BF16_F32, st, View.of(a), View.of(b), View.of(c), overwrite=True)

    with torch.cuda.stream(st):
        if warm:
            for _ in range(3):
                run()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=st):
            run()
        for _ in range(3):
            for _, _, c, _ in ops:
                c.zero_()
            graph.replay()
            st.synchronize()
            for _, _, c, ref in ops:
                assert float((c.double() - ref).norm() / ref.norm()) < 1e-5
        run()   # eager again on the same stream after the replays
        st.synchronize()
    for _, _, c, ref in ops:
        assert float((c.double() - ref).norm() / ref.norm()) < 1e-5


def test_numpy_operands_registered_once(monkeypatch):
    """Large NumPy operands are page-locked on first use (paco_host_register) and
    DMA'd in place by later calls; the registration is dropped when the array is
    freed; results equal the staged path's and the oracle's."""
    import gc

    from paper_2011_01441_b200 import mm as MMmod
    monkeypatch.setattr(MMmod, "_REGISTER_MIN_BYTES", 0)
    rng = np.random.default_rng(44)
    n, m, k = 1100, 650, 2600
    A = tropical(rng, (n, k), 0, 2**20, 0.1)
    B = tropical(rng, (k, m), 0, 2**20, 0.1)
    C0 = tropical(rng, (n, m), 0, 2**21, 0.3)
    want = cref.mm(cref.SR_MINPLUS_SAT32, A, B, C0.copy())
    C = C0.copy()
    before = len(MMmod._registered)
    for _ in range(2):
        C[...] = C0
        M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT)
        assert np.array_equal(C, want)
    assert len(MMmod._registered) == before + 3
    monkeypatch.setattr(MMmod, "REGISTER_HOST", False)   # the staged path gives the same C
    C2 = C0.copy()
    M.mm_seq(A, B, C2, M.SEMIRING_MINPLUS_SAT)
    assert np.array_equal(C2, want)
    del A, B, C
    gc.collect()
    assert len(MMmod._registered) == before + 0
