"""BASELINE configs at FULL size on the GPU, checked against the CPU oracle.

cfg2 (8192^3 min-plus) and cfg4 (16384^3 max-plus) are compared with the
pinned CPU oracle on EVERY element of C (np.array_equal on the whole matrix;
the oracle's cache-blocked tropical path does the 5.5e11 / 4.4e12 terms in
seconds / about half a minute on the host cores).  On top, size-independent
properties the domain offers: every PACO plan of the same product --
GPU-level one-piece with k-cut folds -- must give the bit-identical C
(min/max are associative, commutative and idempotent), and C is a fixed point
of C (+)= A (x) B.  Seeds/distributions follow SURVEY.md 8(d).
"""

import numpy as np
import pytest
import torch

from oracle import cref
from paper_2011_01441_b200 import matmul as M

pytestmark = pytest.mark.gpu
INF = 2**30


def cfg2_inputs():
    rng = np.random.default_rng(1002)
    n = 8192
    A = rng.integers(0, 2**20, (n, n), dtype=np.int32)
    A[rng.random(A.shape) < 0.10] = INF
    B = rng.integers(0, 2**20, (n, n), dtype=np.int32)
    B[rng.random(B.shape) < 0.10] = INF
    return A, B


def cfg4_inputs():
    rng = np.random.default_rng(1004)
    n = 16384
    A = rng.integers(-2**20, 2**20, (n, n), dtype=np.int32)
    B = rng.integers(-2**20, 2**20, (n, n), dtype=np.int32)
    return A, B


def oracle_c(sr, A, B, zero):
    """The whole oracle C = zero (+) A (x) B on the host cores."""
    return cref.mm(sr, A, B, np.full((A.shape[0], B.shape[1]), zero, np.int32))


def test_cfg2_minplus_8192_full():
    A, B = cfg2_inputs()
    a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    c = torch.full((8192, 8192), INF, dtype=torch.int32, device="cuda")
    M.mm_seq(a, b, c, M.SEMIRING_MINPLUS_SAT)
    C = c.cpu().numpy()
    assert np.array_equal(C, oracle_c(cref.SR_MINPLUS_SAT32, A, B, INF))
    # GPU-level PACO plans with k-cut MIN folds (p=5: 1 fold, p=7: 3 folds) agree bit for bit
    for p in (3, 5, 7):
        c2 = torch.full((8192, 8192), INF, dtype=torch.int32, device="cuda")
        M.mm_execute(M.mm_one_piece_partition(8192, 8192, 8192, p), a, b, c2, M.SEMIRING_MINPLUS_SAT,
                     mode="parallel")
        assert torch.equal(c, c2), p
    # fixed point: min(C, A (x) B) == C
    M.mm_seq(a, b, c, M.SEMIRING_MINPLUS_SAT)
    assert np.array_equal(c.cpu().numpy(), C)
    assert (C <= INF).all() and (C >= 0).all()


def test_cfg4_maxplus_16384_full_all_p():
    A, B = cfg4_inputs()
    a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    c = torch.full((16384, 16384), -INF, dtype=torch.int32, device="cuda")
    M.mm_seq(a, b, c, M.SEMIRING_MAXPLUS)
    C = c.cpu().numpy()
    assert np.array_equal(C, oracle_c(cref.SR_MAXPLUS_SAT32, A, B, -INF))
    for p in (1, 2, 3, 4, 5, 7, 8):
        c2 = torch.full((16384, 16384), -INF, dtype=torch.int32, device="cuda")
        M.mm_execute(M.mm_one_piece_partition(16384, 16384, 16384, p), a, b, c2, M.SEMIRING_MAXPLUS,
                     mode="parallel")
        assert torch.equal(c, c2), p


def test_cfg3_bf16_full_vs_f64():
    rng = np.random.default_rng(1003)
    A = rng.standard_normal((65536, 256), dtype=np.float32)
    B = rng.standard_normal((256, 1024), dtype=np.float32)
    a = torch.from_numpy(A).cuda().to(torch.bfloat16)
    b = torch.from_numpy(B).cuda().to(torch.bfloat16)
    c = torch.empty(65536, 1024, device="cuda")
    M.mm_seq(a, b, c, M.SEMIRING_BF16, overwrite=True)
    ref = a.double().cpu().numpy() @ b.double().cpu().numpy()
    err = np.linalg.norm(c.cpu().numpy().astype(np.float64) - ref) / np.linalg.norm(ref)
    assert err <= 1e-2 and err < 1e-5, err


def test_c_beyond_2g_elements_minplus():
    """Maximum-size indexing: a 49152 x 49152 int32 C (2.4e9 elements, 9.7 GB --
    element offsets beyond 2^31) through the tile-grid plan and the PACO cuboid
    plan; sampled rows (including the last) bit-exact vs the oracle."""
    from paper_2011_01441_b200 import _native as nat
    from paper_2011_01441_b200.device import View
    from paper_2011_01441_b200.mm import launch_mm
    rng = np.random.default_rng(77)
    n, k = 49152, 160
    A = rng.integers(0, 2**20, (n, k), dtype=np.int32)
    B = rng.integers(0, 2**20, (k, n), dtype=np.int32)
    a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    rows = np.array([0, 1, 12345, 30000, n - 2, n - 1])
    want = cref.mm_rows(cref.SR_MINPLUS_SAT32, A, B, np.full((len(rows), n), INF, np.int32), rows)
    for flags in (0, nat.MM_PACO_PLAN):
        c = torch.full((n, n), INF, dtype=torch.int32, device="cuda")
        launch_mm(nat.SR_MINPLUS_SAT32, torch.cuda.current_stream(), View.of(a), View.of(b), View.of(c),
                  flags=flags)
        got = c[torch.from_numpy(rows).cuda()].cpu().numpy()
        assert np.array_equal(got, want), flags
        del c
        torch.cuda.empty_cache()


def test_c_beyond_2g_elements_bf16():
    """The tcgen05 path at the same scale: 49152 x 49152 fp32 C from bf16 operands."""
    n, k = 49152, 128
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(k, n, device="cuda", generator=g).to(torch.bfloat16)
    c = torch.empty(n, n, device="cuda")
    M.mm_seq(a, b, c, M.SEMIRING_BF16, overwrite=True)
    rows = torch.tensor([0, 777, 40000, n - 1], device="cuda")
    ref = a[rows].double() @ b.double()
    assert float((c[rows].double() - ref).norm() / ref.norm()) < 1e-5
