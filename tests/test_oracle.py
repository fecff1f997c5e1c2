"""Pin the CPU oracle (test infrastructure) to the reference's own results.

oracle/semiring_ref.c and oracle/paco_numpy.py restate the reference's
arithmetic; before either is trusted as a checker it must reproduce every
golden vector the reference produced (tests/golden/mm_cases.npz).
"""

import numpy as np
import pytest

from oracle import cref
from oracle import paco_numpy as PN
from paper_2011_01441_b200 import matmul as M

INF = 2**30


def test_c_oracle_pins(golden_cases):
    g = golden_cases
    C = np.zeros((384, 320), np.int64)
    assert np.array_equal(cref.mm(cref.SR_INT_I32_I64, g["cfg1_A"], g["cfg1_B"], C), g["cfg1_C"])
    C = np.zeros((384, 320), np.int64)
    assert np.array_equal(cref.mm(cref.SR_INT_I64, g["cfg1_A"].astype(np.int64),
                                  g["cfg1_B"].astype(np.int64), C), g["cfg1_C"])
    for tag in ("minplus_sat", "minplus_inf"):
        A, B = g[f"{tag}_A"], g[f"{tag}_B"]
        C = np.full((A.shape[0], B.shape[1]), INF, np.int32)
        assert np.array_equal(cref.mm(cref.SR_MINPLUS_SAT32, A, B, C), g[f"{tag}_C"]), tag
    A, B = g["maxplus_A"], g["maxplus_B"]
    C = np.full((A.shape[0], B.shape[1]), -INF, np.int32)
    assert np.array_equal(cref.mm(cref.SR_MAXPLUS_SAT32, A, B, C), g["maxplus_C"])
    A, B = g["minplus_i64_A"], g["minplus_i64_B"]
    C = np.full((A.shape[0], B.shape[1]), M.MINPLUS_INF, np.int64)
    assert np.array_equal(cref.mm(cref.SR_MINPLUS_I64, A, B, C), g["minplus_i64_C"])
    C = g["int_wrap_C0"].copy()
    assert np.array_equal(cref.mm(cref.SR_INT_I64, g["int_wrap_A"], g["int_wrap_B"], C), g["int_wrap_C"])
    C = g["f64_C0"].copy()
    np.testing.assert_allclose(cref.mm(cref.SR_F64, g["f64_A"], g["f64_B"], C), g["f64_C"], rtol=1e-12)


@pytest.mark.parametrize("shape", [(1, 1, 1), (5, 17, 3), (6, 16, 256), (7, 33, 257), (100, 517, 300),
                                   (97, 1025, 600)])
def test_c_oracle_blocked_tropical_equals_plain_loop(shape, golden_cases):
    """The cache-blocked 32-bit tropical path (used for the whole-C full-size checks)
    gives the plain loop's bits on ragged shapes, with and without INF entries."""
    n, m, k = shape
    rng = np.random.default_rng(n * 7 + m)
    for sr, lo, hi, zero in ((cref.SR_MINPLUS_SAT32, 0, 2**20, INF), (cref.SR_MAXPLUS_SAT32, -2**20, 2**20, -INF)):
        A = rng.integers(lo, hi, (n, k), dtype=np.int32)
        B = rng.integers(lo, hi, (k, m), dtype=np.int32)
        if sr == cref.SR_MINPLUS_SAT32:
            A[rng.random(A.shape) < 0.1] = INF
            B[rng.random(B.shape) < 0.1] = INF
        C0 = rng.integers(lo, hi, (n, m), dtype=np.int32)
        C0[rng.random(C0.shape) < 0.3] = zero
        assert np.array_equal(cref.mm(sr, A, B, C0.copy()), cref.mm(sr, A, B, C0.copy(), simple=True)), (sr, shape)
    for tag in ("minplus_sat", "minplus_inf"):  # and the blocked path alone reproduces the goldens
        A, B = golden_cases[f"{tag}_A"], golden_cases[f"{tag}_B"]
        C = np.full((A.shape[0], B.shape[1]), INF, np.int32)
        assert np.array_equal(cref.mm(cref.SR_MINPLUS_SAT32, A, B, C, simple=True), golden_cases[f"{tag}_C"])


def test_numpy_port_pins(golden_cases):
    g = golden_cases
    plan = M.mm_paco_partition(384, 320, 256, 3)
    C = np.zeros((384, 320), np.int64)
    PN.mm_execute_serial(plan, g["cfg1_A"].astype(np.int64), g["cfg1_B"].astype(np.int64), C, "int")
    assert np.array_equal(C, g["cfg1_C"])
    C = np.zeros((384, 320), np.int64)  # the threaded (mode="parallel") restatement: same C
    PN.mm_execute_parallel(plan, g["cfg1_A"].astype(np.int64), g["cfg1_B"].astype(np.int64), C, "int")
    assert np.array_equal(C, g["cfg1_C"])
    A, B = g["minplus_sat_A"], g["minplus_sat_B"]
    assert np.array_equal(PN.minplus_sat(A, B, np.full((A.shape[0], B.shape[1]), INF, np.int32)),
                          g["minplus_sat_C"])
    A, B = g["maxplus_A"], g["maxplus_B"]
    assert np.array_equal(PN.maxplus(A, B, np.full((A.shape[0], B.shape[1]), -INF, np.int32)),
                          g["maxplus_C"])
    A, B = g["minplus_i64_A"], g["minplus_i64_B"]
    C = np.full((A.shape[0], B.shape[1]), M.MINPLUS_INF, np.int64)
    with np.errstate(over="ignore"):
        PN.mm_execute_serial(M.mm_paco_partition(*A.shape[:1], B.shape[1], A.shape[1], 3), A, B, C,
                             "minplus")
    assert np.array_equal(C, g["minplus_i64_C"])


def test_saturating_identity_on_domain():
    """minplus_sat == clamp(reference minplus) and maxplus == -minplus(-A,-B) on the domain."""
    rng = np.random.default_rng(0)
    A = rng.integers(0, 2**30, (23, 31), dtype=np.int32)
    A[rng.random(A.shape) < 0.3] = INF
    B = rng.integers(0, 2**30, (31, 17), dtype=np.int32)
    B[rng.random(B.shape) < 0.3] = INF
    C = np.full((23, 17), INF, np.int32)
    assert np.array_equal(cref.mm(cref.SR_MINPLUS_SAT32, A, B, C.copy()), PN.minplus_sat(A, B, C))
    A = rng.integers(-2**30, 2**30, (23, 31), dtype=np.int32)
    B = rng.integers(-2**30, 2**30, (31, 17), dtype=np.int32)
    C = np.full((23, 17), -INF, np.int32)
    assert np.array_equal(cref.mm(cref.SR_MAXPLUS_SAT32, A, B, C.copy()), PN.maxplus(A, B, C))


# --- Strassen restatement: SPEC.md:494-498, 526 known answers ----------------

def test_strassen_known_answers():
    a, b = np.array([[3]]), np.array([[-4]])
    assert PN.strassen(a, b, 1).tolist() == [[-12]]
    rng = np.random.default_rng(4)
    B4 = rng.integers(-9, 10, (4, 4))
    assert np.array_equal(PN.strassen(np.eye(4, dtype=np.int64), B4, 2), B4)
    A8, B8 = rng.integers(-9, 10, (8, 8)), rng.integers(-9, 10, (8, 8))
    assert np.array_equal(PN.strassen(A8, B8, 3), A8 @ B8)
    for n in (16, 64, 256):
        A, B = rng.integers(-50, 50, (n, n)), rng.integers(-50, 50, (n, n))
        assert np.array_equal(PN.strassen(A, B, 2), A @ B)


def test_strassen_float_close():
    rng = np.random.default_rng(5)
    A, B = rng.uniform(-1, 1, (128, 128)), rng.uniform(-1, 1, (128, 128))
    C = PN.strassen(A, B, 2)
    assert np.linalg.norm(C - A @ B) / np.linalg.norm(A @ B) < 1e-13
