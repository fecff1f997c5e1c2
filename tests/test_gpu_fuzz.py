"""Seeded fuzz of the whole MM path against the CPU oracle.

Random shapes (ragged, 1..600 per axis), every semiring family, every GPU-level
plan variant (one-piece / multi-piece PACO / hetero, p = 1..9), both executor
modes, fused and explicit k-cut folds, and three operand kinds (NumPy, CUDA
tensors at odd offsets inside larger buffers, pinned host tensors through
mm_seq).  Integer / tropical results must be bit-exact; f32 / f64 within the
tolerances of tests/test_gpu_mm.py.
"""

import numpy as np
import pytest
import torch

from oracle import cref
from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200.plan import PlanError

pytestmark = pytest.mark.gpu
INF = 2**30

FAMILIES = {
    # name: (semiring, oracle id, operand dtype, C dtype, draw)
    "minplus_sat": (M.SEMIRING_MINPLUS_SAT, cref.SR_MINPLUS_SAT32, np.int32, np.int32, "trop"),
    "maxplus": (M.SEMIRING_MAXPLUS, cref.SR_MAXPLUS_SAT32, np.int32, np.int32, "trop-neg"),
    "int_i32": (M.SEMIRING_INT, cref.SR_INT_I32_I64, np.int32, np.int64, "small"),
    "int_i64": (M.SEMIRING_INT, cref.SR_INT_I64, np.int64, np.int64, "small"),
    "minplus_i64": (M.SEMIRING_MINPLUS, cref.SR_MINPLUS_I64, np.int64, np.int64, "trop64"),
    "f64": (M.SEMIRING_F64, cref.SR_F64, np.float64, np.float64, "unit"),
    "f32": (M.SEMIRING_F32, cref.SR_F32, np.float32, np.float32, "unit"),
}


def draw(rng, kind, shape, dt):
    if kind == "trop":
        x = rng.integers(0, 2**20, shape).astype(dt)
        x[rng.random(shape) < 0.15] = INF
        return x
    if kind == "trop-neg":
        x = rng.integers(-2**20, 2**20, shape).astype(dt)
        x[rng.random(shape) < 0.15] = -INF
        return x
    if kind == "trop64":
        return rng.integers(0, 2**40, shape).astype(dt)
    if kind == "small":
        return rng.integers(-1000, 1000, shape).astype(dt)
    return rng.uniform(-1, 1, shape).astype(dt)


def c_init(rng, name, shape):
    sr, _, _, cdt, kind = FAMILIES[name]
    if rng.random() < 0.3:
        return np.full(shape, sr.zero, cdt)
    if kind == "trop":
        return draw(rng, "trop", shape, cdt)
    if kind == "trop-neg":
        return draw(rng, "trop-neg", shape, cdt)
    return draw(rng, kind, shape, cdt)


def check(name, got, want, ctx):
    if name in ("f32", "f64"):
        ref = want.astype(np.float64)
        tol = 1e-5 if name == "f32" else 1e-12
        den = max(np.linalg.norm(ref), 1e-30)
        assert np.linalg.norm(got.astype(np.float64) - ref) <= tol * den, ctx
    else:
        assert np.array_equal(got, want), ctx


def make_plan(rng, n, m, k):
    p = int(rng.integers(1, 10))
    v = rng.choice(["one", "paco", "hetero"])
    if v == "one" or n * m * k < 8 * p:
        return M.mm_one_piece_partition(n, m, k, p), "one", p
    if v == "paco":
        return M.mm_paco_partition(n, m, k, p, base=int(rng.choice([8, 16, 32, 64]))), "paco", p
    w = tuple(float(x) for x in rng.uniform(0.5, 2.0, p))
    return M.mm_hetero_partition(n, m, k, w), "hetero", p


@pytest.mark.parametrize("block", range(6))
def test_fuzz_mm_execute(block):
    rng = np.random.default_rng(9000 + block)
    names = list(FAMILIES)
    for case in range(30):
        name = names[int(rng.integers(len(names)))]
        sr, cid, dt, cdt, kind = FAMILIES[name]
        n, m, k = (int(x) for x in rng.integers(1, 600, 3))
        A, B = draw(rng, kind, (n, k), dt), draw(rng, kind, (k, m), dt)
        C0 = c_init(rng, name, (n, m))
        want = cref.mm(cid, A, B, C0.copy())
        try:
            plan, variant, p = make_plan(rng, n, m, k)
        except PlanError:
            continue
        mode = "parallel" if rng.random() < 0.5 else "serial_sim"
        fused = None if rng.random() < 0.7 else False
        if rng.random() < 0.5:  # numpy in, numpy out
            C = C0.copy()
            M.mm_execute(plan, A, B, C, sr, mode=mode, fused_folds=fused)
            got = C
        else:  # CUDA views at odd offsets inside larger buffers
            oi, oj, ol = (int(x) for x in rng.integers(0, 5, 3))
            bigA = torch.zeros((n + oi + 3, k + ol + 5), dtype=torch.from_numpy(A).dtype, device="cuda")
            bigB = torch.zeros((k + ol + 2, m + oj + 7), dtype=torch.from_numpy(B).dtype, device="cuda")
            bigC = torch.zeros((n + oi + 1, m + oj + 3), dtype=torch.from_numpy(C0).dtype, device="cuda")
            a = bigA[oi:oi + n, ol:ol + k]
            b = bigB[ol:ol + k, oj:oj + m]
            c = bigC[oi:oi + n, oj:oj + m]
            a.copy_(torch.from_numpy(A))
            b.copy_(torch.from_numpy(B))
            c.copy_(torch.from_numpy(C0))
            M.mm_execute(plan, a, b, c, sr, mode=mode, fused_folds=fused)
            got = c.cpu().numpy()
            assert int(torch.count_nonzero(bigC[:oi])) == 0 if oi else True
        check(name, got, want, (name, n, m, k, variant, p, mode, fused))


@pytest.mark.parametrize("block", range(3))
def test_fuzz_mm_seq_pinned_and_plain(block):
    """mm_seq on pinned host tensors (k-first or 2-D pipeline when large enough)
    and on plain CPU tensors / NumPy, all semiring families."""
    rng = np.random.default_rng(9100 + block)
    for case in range(16):
        name = list(FAMILIES)[int(rng.integers(len(FAMILIES)))]
        sr, cid, dt, cdt, kind = FAMILIES[name]
        big = rng.random() < 0.5
        n = int(rng.integers(1024, 1500)) if big else int(rng.integers(1, 400))
        m = int(rng.integers(1, 700))
        k = int(rng.integers(2048, 2700)) if big and rng.random() < 0.5 else int(rng.integers(1, 500))
        A, B = draw(rng, kind, (n, k), dt), draw(rng, kind, (k, m), dt)
        C0 = c_init(rng, name, (n, m))
        want = cref.mm(cid, A, B, C0.copy())
        overwrite = bool((C0 == sr.zero).all())
        Ah, Bh = torch.from_numpy(A), torch.from_numpy(B)
        Ch = torch.from_numpy(C0.copy())
        if rng.random() < 0.7:
            Ah, Bh, Ch = Ah.pin_memory(), Bh.pin_memory(), Ch.pin_memory()
        M.mm_seq(Ah, Bh, Ch, sr, overwrite=overwrite)
        check(name, Ch.numpy(), want, (name, n, m, k))
